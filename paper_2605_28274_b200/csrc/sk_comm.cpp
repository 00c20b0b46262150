// sk_comm.cpp -- NCCL (run-time loaded) and local-group transports, see sk_comm.h.
#include "sk_comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

namespace sk {
namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// NCCL, resolved with dlopen/dlsym
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) {
      err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* nm) {
      void* p = dlsym(api.h, nm);
      if (!p) err = std::string("NCCL symbol missing: ") + nm;
      return p;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  });
  if (!err.empty()) throw std::runtime_error(err);
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t st) override {
    nccl_ok(nccl().AllGather(send, recv, (size_t)count, ncclFloat64, comm, st), "ncclAllGather");
  }
  void allgatherv(const double* send, double* recv, const int64_t* counts, const int64_t* displs,
                  cudaStream_t st) override {
    NcclApi& a = nccl();
    nccl_ok(a.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < size; ++r) {
      if (counts[rank] > 0) nccl_ok(a.Send(send, (size_t)counts[rank], ncclFloat64, r, comm, st), "ncclSend");
      if (counts[r] > 0) nccl_ok(a.Recv(recv + displs[r], (size_t)counts[r], ncclFloat64, r, comm, st), "ncclRecv");
    }
    nccl_ok(a.GroupEnd(), "ncclGroupEnd");
  }
  void halo(const Halo* h, int nh, cudaStream_t st) override {
    NcclApi& a = nccl();
    nccl_ok(a.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < nh; ++i) {
      if (h[i].count == 0) continue;
      if (rank > 0) {
        nccl_ok(a.Send(h[i].send_lo, (size_t)h[i].count, ncclFloat64, rank - 1, comm, st), "ncclSend");
        nccl_ok(a.Recv(h[i].recv_lo, (size_t)h[i].count, ncclFloat64, rank - 1, comm, st), "ncclRecv");
      }
      if (rank < size - 1) {
        nccl_ok(a.Send(h[i].send_hi, (size_t)h[i].count, ncclFloat64, rank + 1, comm, st), "ncclSend");
        nccl_ok(a.Recv(h[i].recv_hi, (size_t)h[i].count, ncclFloat64, rank + 1, comm, st), "ncclRecv");
      }
    }
    nccl_ok(a.GroupEnd(), "ncclGroupEnd");
  }
  const char* kind() const override { return "nccl"; }
};

// ---------------------------------------------------------------------------
// Local group: ranks are host threads; collectives are D2D copies behind
// host barriers (each rank's stream is drained before it publishes).
// ---------------------------------------------------------------------------
struct LocalGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<const double*> a, b;
  std::vector<const Comm::Halo*> halos;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalComm : Comm {
  std::shared_ptr<LocalGroup> g;
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t st) override {
    cuda_ok(cudaStreamSynchronize(st), "local allgather");
    g->a[rank] = send;
    g->barrier();
    for (int r = 0; r < size; ++r)
      cuda_ok(cudaMemcpyAsync(recv + r * count, g->a[r], sizeof(double) * count, cudaMemcpyDeviceToDevice, st),
              "local allgather copy");
    cuda_ok(cudaStreamSynchronize(st), "local allgather");
    g->barrier();
  }
  void allgatherv(const double* send, double* recv, const int64_t* counts, const int64_t* displs,
                  cudaStream_t st) override {
    cuda_ok(cudaStreamSynchronize(st), "local allgatherv");
    g->a[rank] = send;
    g->barrier();
    for (int r = 0; r < size; ++r)
      if (counts[r] > 0)
        cuda_ok(cudaMemcpyAsync(recv + displs[r], g->a[r], sizeof(double) * counts[r], cudaMemcpyDeviceToDevice, st),
                "local allgatherv copy");
    cuda_ok(cudaStreamSynchronize(st), "local allgatherv");
    g->barrier();
  }
  void halo(const Halo* h, int nh, cudaStream_t st) override {
    cuda_ok(cudaStreamSynchronize(st), "local halo");
    g->halos[rank] = h;
    g->barrier();
    for (int i = 0; i < nh; ++i) {
      if (h[i].count == 0) continue;
      const size_t bytes = sizeof(double) * h[i].count;
      if (rank > 0)
        cuda_ok(cudaMemcpyAsync(h[i].recv_lo, g->halos[rank - 1][i].send_hi, bytes, cudaMemcpyDeviceToDevice, st),
                "local halo copy");
      if (rank < size - 1)
        cuda_ok(cudaMemcpyAsync(h[i].recv_hi, g->halos[rank + 1][i].send_lo, bytes, cudaMemcpyDeviceToDevice, st),
                "local halo copy");
    }
    cuda_ok(cudaStreamSynchronize(st), "local halo");
    g->barrier();
  }
  const char* kind() const override { return "local"; }
};

}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_ok(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof id);
}

Comm* make_nccl_comm(const void* uid128, int nranks, int rank, int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::runtime_error("invalid NCCL rank / size");
  cuda_ok(cudaSetDevice(device), "cudaSetDevice");
  auto c = std::make_unique<NcclComm>();
  ncclUniqueId id;
  std::memcpy(&id, uid128, sizeof id);
  nccl_ok(nccl().CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  c->rank = rank;
  c->size = nranks;
  return c.release();
}

void make_local_group(int nranks, Comm** out) {
  if (nranks < 1) throw std::runtime_error("local group needs >= 1 rank");
  auto g = std::make_shared<LocalGroup>();
  g->n = nranks;
  g->a.assign(nranks, nullptr);
  g->b.assign(nranks, nullptr);
  g->halos.assign(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    auto* c = new LocalComm();
    c->g = g;
    c->rank = r;
    c->size = nranks;
    out[r] = c;
  }
}

}  // namespace sk
