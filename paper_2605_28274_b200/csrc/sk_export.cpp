// On-disk formats of a solve: history CSV, Matrix Market text and
// the binary sidecar. The text writers restate the reference's byte format:
//   write_history_csv            bench.cpp:179-193
//   write_matrix_market(Sparse)  matrix_market.cpp:148-161  ("coordinate real general")
//   write_matrix_market(Dense)   matrix_market.cpp:163-175  ("array real general")
//   write_value                  matrix_market.cpp:140-144  (snprintf "%.17g")
// Factors are streamed out of HBM in column chunks (sk_solution_copy_V_cols) and
// formatted on all host threads, then written in order, so the host never holds
// V or W whole and the file is byte-identical to the serial writer's.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sylkrylov_b200.h"

extern "C" void sk_internal_set_error(const char* msg);

namespace {

struct File {
  std::FILE* f = nullptr;
  std::string path;
  explicit File(const std::string& p) : path(p) { f = std::fopen(p.c_str(), "wb"); }
  ~File() {
    if (f) std::fclose(f);
  }
  bool write(const void* d, size_t n) { return std::fwrite(d, 1, n, f) == n; }
  bool write(const std::string& s) { return write(s.data(), s.size()); }
  bool close() {
    const int rc = std::fclose(f);
    f = nullptr;
    return rc == 0;
  }
};

sk_status io_error(const std::string& what) {
  sk_internal_set_error(what.c_str());
  return SK_ERR_IO;
}

int host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h, 64u));
}

// "%.17g\n" of v[0..count) appended to out
void format_values(const double* v, int64_t count, std::string& out) {
  char buf[40];
  out.reserve(out.size() + (size_t)count * 25);
  for (int64_t i = 0; i < count; ++i) {
    const int len = std::snprintf(buf, sizeof buf, "%.17g\n", v[i]);
    out.append(buf, (size_t)len);
  }
}

// formats count values on all host threads; pieces are written in order
bool write_values_parallel(File& f, const double* v, int64_t count) {
  const int T = (int)std::min<int64_t>(host_threads(), std::max<int64_t>(1, count / 65536));
  std::vector<std::string> parts((size_t)T);
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      const int64_t a = count * t / T, b = count * (t + 1) / T;
      format_values(v + a, b - a, parts[(size_t)t]);
    });
  for (auto& x : th) x.join();
  for (auto& p : parts)
    if (!f.write(p)) return false;
  return true;
}

using ColCopy = sk_status (*)(const sk_solution*, int64_t, int64_t, double*);

// rows x cols matrix whose column chunks come from copy(); text or binary body
sk_status write_streamed(const std::string& path, int64_t rows, int64_t cols, int32_t format,
                         const sk_solution* sol, ColCopy copy) {
  File f(path);
  if (!f.f) return io_error("cannot write " + path);
  bool ok = true;
  if (format == SK_FORMAT_BINARY) {
    const char magic[8] = {'S', 'K', 'F', 'A', 'C', 'T', '0', '1'};
    ok = f.write(magic, 8) && f.write(&rows, 8) && f.write(&cols, 8);
  } else {
    ok = f.write("%%MatrixMarket matrix array real general\n" + std::to_string(rows) + " " +
                 std::to_string(cols) + "\n");
  }
  // ~256 MB of values per chunk
  const int64_t per = std::max<int64_t>(1, (int64_t)(32 << 20) / std::max<int64_t>(1, rows));
  std::vector<double> buf((size_t)(rows * std::min(per, std::max<int64_t>(cols, 1))));
  for (int64_t c0 = 0; ok && c0 < cols; c0 += per) {
    const int64_t nc = std::min(per, cols - c0);
    const sk_status rc = copy(sol, c0, nc, buf.data());
    if (rc != SK_OK) return rc;
    ok = format == SK_FORMAT_BINARY ? f.write(buf.data(), sizeof(double) * (size_t)(rows * nc))
                                    : write_values_parallel(f, buf.data(), rows * nc);
  }
  if (!ok || !f.close()) return io_error("write failed: " + path);
  return SK_OK;
}

sk_status copy_core_cols(const sk_solution* sol, int64_t col0, int64_t ncols, double* out) {
  int64_t n, rv, m, rw;
  sk_solution_dims(sol, &n, &rv, &m, &rw);
  std::vector<double> all((size_t)(rv * rw));
  const sk_status rc = sk_solution_copy_core(sol, all.data());
  if (rc != SK_OK) return rc;
  std::memcpy(out, all.data() + col0 * rv, sizeof(double) * (size_t)(rv * ncols));
  return SK_OK;
}

}  // namespace

extern "C" {

sk_status sk_write_history_csv(const sk_solution* sol, const char* path) {
  const int64_t nrec = sk_solution_num_records(sol);
  std::vector<sk_iteration_record> rec((size_t)std::max<int64_t>(nrec, 0));
  if (nrec > 0) {
    const sk_status rc = sk_solution_history(sol, rec.data(), nrec);
    if (rc != SK_OK) return rc;
  }
  File f(path);
  if (!f.f) return io_error(std::string("cannot write ") + path);
  std::string out = "iteration,rel_residual,cumulative_time_s,basic_s,krylov_s,trunc_s\n";
  char buf[160];
  double cumulative = 0.0;
  for (const sk_iteration_record& r : rec) {
    cumulative += r.t_basic_s + r.t_krylov_s + r.t_trunc_s;
    const int len = std::snprintf(buf, sizeof buf, "%lld,%.17g,%.17g,%.17g,%.17g,%.17g\n", (long long)r.iteration,
                                  r.rel_residual, cumulative, r.t_basic_s, r.t_krylov_s, r.t_trunc_s);
    out.append(buf, (size_t)len);
  }
  if (!f.write(out) || !f.close()) return io_error(std::string("write failed: ") + path);
  return SK_OK;
}

sk_status sk_write_matrix_market_csr(const sk_csr* a, const char* path) {
  File f(path);
  if (!f.f) return io_error(std::string("cannot write ") + path);
  std::string out = "%%MatrixMarket matrix coordinate real general\n" + std::to_string(a->n_rows) + " " +
                    std::to_string(a->n_cols) + " " + std::to_string(a->nnz) + "\n";
  bool ok = f.write(out);
  // rows formatted in parallel chunks, written in row order
  const int64_t n = a->n_rows;
  const int64_t chunk = 1 << 18;
  for (int64_t r0 = 0; ok && r0 < n; r0 += chunk * host_threads()) {
    const int T = host_threads();
    std::vector<std::string> parts((size_t)T);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        const int64_t i0 = std::min(n, r0 + chunk * t), i1 = std::min(n, r0 + chunk * (t + 1));
        char buf[80];
        std::string& s = parts[(size_t)t];
        for (int64_t i = i0; i < i1; ++i)
          for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
            const int len = std::snprintf(buf, sizeof buf, "%lld %lld %.17g\n", (long long)(i + 1),
                                          (long long)(a->col_idx[k] + 1), a->values[k]);
            s.append(buf, (size_t)len);
          }
      });
    for (auto& x : th) x.join();
    for (auto& p : parts)
      if (ok) ok = f.write(p);
  }
  if (!ok || !f.close()) return io_error(std::string("write failed: ") + path);
  return SK_OK;
}

sk_status sk_write_matrix_market_dense(const double* a, int64_t rows, int64_t cols, const char* path) {
  File f(path);
  if (!f.f) return io_error(std::string("cannot write ") + path);
  bool ok = f.write("%%MatrixMarket matrix array real general\n" + std::to_string(rows) + " " +
                    std::to_string(cols) + "\n");
  if (ok) ok = write_values_parallel(f, a, rows * cols);
  if (!ok || !f.close()) return io_error(std::string("write failed: ") + path);
  return SK_OK;
}

sk_status sk_solution_write_factors(const sk_solution* sol, const char* dir, int32_t format) {
  if (format != SK_FORMAT_MATRIX_MARKET && format != SK_FORMAT_BINARY) {
    sk_internal_set_error("write_factors: unknown format");
    return SK_ERR_UNSUPPORTED;
  }
  int64_t n, rv, m, rw;
  sk_solution_dims(sol, &n, &rv, &m, &rw);
  const std::string d(dir), ext = format == SK_FORMAT_BINARY ? ".skb" : ".mtx";
  sk_status rc = write_streamed(d + "/V" + ext, n, rv, format, sol, sk_solution_copy_V_cols);
  if (rc == SK_OK) rc = write_streamed(d + "/core" + ext, rv, rw, format, sol, copy_core_cols);
  if (rc == SK_OK) rc = write_streamed(d + "/W" + ext, m, rw, format, sol, sk_solution_copy_W_cols);
  return rc;
}

}  // extern "C"
