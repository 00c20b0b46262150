// sk_launch.h -- host-side launchers of the sm_100a kernels (sk_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sk {
struct SolveConst;
int launch_count();
void launch_count_reset();
void launch_init(const SolveConst& c, const double* dc1, const double* dc2, cudaStream_t st);
void launch_spmm(const SolveConst& c, cudaStream_t st);
void launch_lanczos_gram(const SolveConst& c, cudaStream_t st);
bool lanczos_fused_ok(const SolveConst& c);
void launch_lanczos_p1(const SolveConst& c, cudaStream_t st);
void launch_lanczos_p2(const SolveConst& c, cudaStream_t st);
bool lanczos_sweep_ok(const SolveConst& c);
void launch_lanczos_sweep(const SolveConst& c, cudaStream_t st);
void launch_lanczos_update(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st);
void launch_rare(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st);
void launch_arnoldi_ext(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st);
void launch_export_block(int s, const double* blk, const double* nfac, int64_t b, double* out,
                         int64_t n, cudaStream_t st);
void launch_bicgstab_half(const SolveConst& c, int which, int64_t rmax, cudaStream_t st);
void launch_cg_a(const SolveConst& c, int64_t rmax, cudaStream_t st);
void launch_cg_b(const SolveConst& c, int64_t rmax, cudaStream_t st);
void launch_spmm_plain(int s, const int32_t* rp, const int32_t* ci, const double* val,
                       const double* x, double* y, int64_t n, cudaStream_t st);
// row partition (world > 1)
enum { DIST_FIN_P1 = 0, DIST_FIN_P2 = 1, DIST_FIN_CGRAM = 2, DIST_FIN_CSELF = 3 };
void launch_dist_fin(const SolveConst& c, int mode, int64_t msg, cudaStream_t st);
void launch_dist_pause(const SolveConst& c, cudaStream_t st);
void launch_dist_resume(const SolveConst& c, cudaStream_t st);
void launch_halo(const SolveConst& c, int unpack, int64_t H, cudaStream_t st);
void launch_householder(const SolveConst& c, int which, cudaStream_t st);
void launch_gram_loop(const SolveConst& c, cudaStream_t st);
void launch_update_clean(const SolveConst& c, cudaStream_t st);
void launch_block_to_colmajor(const double* blk, double* out, int64_t n, int s, cudaStream_t st);
void launch_colmajor_to_block(const double* in, double* blk, int64_t n, int s, cudaStream_t st);
// device true residual (sk_residual.cu)
struct TrOp;
void launch_tr_gather_blocks(const double* const* blocks, const double* nfac, int s, int nblk, int64_t n, int64_t r0,
                             int64_t rows, double* G, cudaStream_t st);
void launch_tr_gather_dense(const double* X, int64_t n, int cols, int64_t r0, int64_t rows, double* G,
                            cudaStream_t st);
void launch_tr_apply(const TrOp& op, const double* X, int64_t h, int64_t r0, int64_t rows, int r, double* Y,
                     cudaStream_t st);
void launch_tr_fill(double* M, int64_t ldm, int64_t off, int64_t rows, const double* C, int64_t n, int s, int64_t r0,
                    const double* P1, int64_t h1, const double* P2, int64_t h2, int r, double sgn, cudaStream_t st);
void launch_tr_keep_r(double* M, int64_t ldm, int wdt, cudaStream_t st);
void launch_tr_fill_rows(double* M, int64_t ldm, int64_t off, int64_t rows, const double* G, int cols,
                         cudaStream_t st);
}  // namespace sk
