// sk_comm.h -- collectives of the row-partitioned solve.
//
// The partitioned iteration needs exactly two exchange steps: an all-gather of
// the reduction-chunk nodes of each Gram pass (tens of doubles per rank) and a
// neighbour halo exchange of the newest basis block (one grid line / plane per
// boundary). Both are stream-ordered, so the device-resident loop keeps
// enqueueing without host round-trips.
//
// Two transports implement them:
//   * NCCL (one process per GPU, NVLink/NVSwitch): libnccl.so.2 is loaded at
//     run time (the one torch already mapped, or the system copy), so the
//     library itself has no link-time NCCL dependency.
//   * a local group: G ranks as G host threads of one process, collectives as
//     device-to-device copies between the ranks' buffers behind host barriers.
//     It runs the partitioned data path on a single GPU for the parity tests;
//     no kernel ever waits on another rank's kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace sk {

struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() {}
  // recv[r * count + i] = send_r[i] for every rank r
  virtual void allgather(const double* send, double* recv, int64_t count, cudaStream_t st) = 0;
  // rank r's send (counts[r] doubles) lands at recv + displs[r] on every rank
  virtual void allgatherv(const double* send, double* recv, const int64_t* counts, const int64_t* displs,
                          cudaStream_t st) = 0;
  // neighbour exchange, one group: send_lo -> rank-1 (its recv_hi), send_hi -> rank+1 (its recv_lo)
  struct Halo {
    const double* send_lo;
    const double* send_hi;
    double* recv_lo;
    double* recv_hi;
    int64_t count;
  };
  virtual void halo(const Halo* h, int nh, cudaStream_t st) = 0;
  virtual const char* kind() const = 0;
};

// throws std::runtime_error with a message on failure
void nccl_unique_id(void* out128);
Comm* make_nccl_comm(const void* uid128, int nranks, int rank, int device);
void make_local_group(int nranks, Comm** out);

}  // namespace sk
