// sk_residual.cu -- kernels of the device true residual:
//   ||A X + X B - C1 C2^T||_F / ||C1 C2^T||_F,  X = V core W^T,
// restating true_residual_factors (factorized_solvers.cpp:391-439): the
// residual is [C1, A V core, V core] diag(I, -I, -I) [C2, W, B^T W]^T, whose
// Frobenius norm is ||R_U D R_V^T|| for the R factors of the two stacked
// factor matrices. The stacked matrices (n x (s + 2r), 107 GB at config 5) are
// never formed: rows are produced chunk by chunk (with an operator halo) and
// folded into a running R by a streaming TSQR (geqrf of [R; chunk], driver side).
// Floating point, not the bitwise contract: parity is a tolerance (tests).
#include "sk_device.cuh"
#include "sk_launch.h"

#include <cuda_runtime.h>
#include <stdint.h>

namespace sk {

// G (row-major rows x nblk*s) <- normalised basis rows [r0, r0 + rows) of the
// raw blocks (V_b = U_b N_b^{-1}, oracle apply_norm); rows outside [0, n) -> 0
__global__ void k_tr_gather_blocks(const double* const* __restrict__ blocks, const double* __restrict__ nfac,
                                   int s, int nblk, int64_t n, int64_t r0, int64_t rows, double* __restrict__ G) {
  const int64_t total = rows * nblk;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(idx % nblk);
    const int64_t ii = idx / nblk, i = r0 + ii;
    double* out = G + ii * (int64_t)nblk * s + (int64_t)b * s;
    if (i < 0 || i >= n) {
      for (int u = 0; u < s; ++u) out[u] = 0.0;
      continue;
    }
    const double* u = blocks[b] + i * s;
    const double* N = nfac + (int64_t)b * (s * s + s);
    const double* dinv = N + s * s;
    double q[kMaxS];
    for (int c = 0; c < s; ++c) {
      double acc = u[c];
      for (int t = 0; t < c; ++t) acc = __dsub_rn(acc, __dmul_rn(q[t], N[c * s + t]));
      q[c] = __dmul_rn(acc, dinv[c]);
      out[c] = q[c];
    }
  }
}

// G (row-major rows x cols) <- rows [r0, r0 + rows) of a column-major n x cols matrix
__global__ void k_tr_gather_dense(const double* __restrict__ X, int64_t n, int cols, int64_t r0, int64_t rows,
                                  double* __restrict__ G) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % cols);
    const int64_t ii = idx / cols, i = r0 + ii;
    G[idx] = (i >= 0 && i < n) ? X[(int64_t)j * n + i] : 0.0;
  }
}

// Y (row-major rows x r) <- op applied to rows [r0, r0 + rows) of X, where X is
// row-major (rows + 2h) x r holding global rows [r0 - h, r0 + rows + h).
// Row sums in ascending column order (sparse_matrix.cpp:151-155).
__global__ void k_tr_apply(TrOp op, const double* __restrict__ X, int64_t h, int64_t r0, int64_t rows, int r,
                           double* __restrict__ Y) {
  const int64_t total = rows * r;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % r);
    const int64_t ii = idx / r, i = r0 + ii;
    const double* xc = X + (ii + h) * r + j;  // row i of X, column j
    double acc = 0.0;
    if (op.sdim == 0) {
      for (int32_t k = op.rp[i]; k < op.rp[i + 1]; ++k)
        acc = __dadd_rn(acc, __dmul_rn(op.val[k], xc[((int64_t)op.ci[k] - i) * r]));
    } else {
      const int64_t g = op.g, g2 = g * g;
      const int64_t ix = i % g, iy = (i / g) % g, iz = i / g2;
      if (op.sdim == 2) {
        if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(op.c[0], xc[-g * r]));
        if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(op.c[1], xc[-r]));
        acc = __dadd_rn(acc, __dmul_rn(op.c[2], xc[0]));
        if (ix < g - 1) acc = __dadd_rn(acc, __dmul_rn(op.c[3], xc[r]));
        if (iy < g - 1) acc = __dadd_rn(acc, __dmul_rn(op.c[4], xc[g * r]));
      } else {
        if (iz > 0) acc = __dadd_rn(acc, __dmul_rn(op.c[0], xc[-g2 * r]));
        if (iy > 0) acc = __dadd_rn(acc, __dmul_rn(op.c[1], xc[-g * r]));
        if (ix > 0) acc = __dadd_rn(acc, __dmul_rn(op.c[2], xc[-r]));
        acc = __dadd_rn(acc, __dmul_rn(op.c[3], xc[0]));
        if (ix < g - 1) acc = __dadd_rn(acc, __dmul_rn(op.c[4], xc[r]));
        if (iy < g - 1) acc = __dadd_rn(acc, __dmul_rn(op.c[5], xc[g * r]));
        if (iz < g - 1) acc = __dadd_rn(acc, __dmul_rn(op.c[6], xc[g2 * r]));
      }
    }
    Y[idx] = acc;
  }
}

// M (column-major, leading dimension ldm) rows [off, off + rows) <- chunk of the
// stacked factor [C, sgn * P1, sgn * P2]: C column-major n x s (global rows
// r0..), P1 / P2 row-major with r columns, chunk row ii at row ii + h1 / ii + h2
__global__ void k_tr_fill(double* __restrict__ M, int64_t ldm, int64_t off, int64_t rows, const double* __restrict__ C,
                          int64_t n, int s, int64_t r0, const double* __restrict__ P1, int64_t h1,
                          const double* __restrict__ P2, int64_t h2, int r, double sgn) {
  const int wdt = s + 2 * r;
  const int64_t total = rows * wdt;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ii = idx % rows;
    const int c = (int)(idx / rows);
    double v;
    if (c < s)
      v = C[(int64_t)c * n + r0 + ii];
    else if (c < s + r)
      v = sgn * P1[(ii + h1) * r + (c - s)];
    else
      v = sgn * P2[(ii + h2) * r + (c - s - r)];
    M[(int64_t)c * ldm + off + ii] = v;
  }
}

// keep R (upper triangle of the leading wdt x wdt block of M) as the next
// chunk's top rows: zero the Householder vectors below its diagonal
__global__ void k_tr_keep_r(double* __restrict__ M, int64_t ldm, int wdt) {
  const int64_t total = (int64_t)wdt * wdt;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % wdt), c = (int)(idx / wdt);
    if (i > c) M[(int64_t)c * ldm + i] = 0.0;
  }
}

// M (column-major, ldm) rows [off, off + rows), columns [0, cols) <- G (row-major rows x cols)
__global__ void k_tr_fill_rows(double* __restrict__ M, int64_t ldm, int64_t off, int64_t rows,
                               const double* __restrict__ G, int cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ii = idx % rows;
    const int c = (int)(idx / rows);
    M[(int64_t)c * ldm + off + ii] = G[ii * cols + c];
  }
}

static unsigned tr_grid(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (unsigned)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}
void launch_tr_gather_blocks(const double* const* blocks, const double* nfac, int s, int nblk, int64_t n, int64_t r0,
                             int64_t rows, double* G, cudaStream_t st) {
  k_tr_gather_blocks<<<tr_grid(rows * nblk), 256, 0, st>>>(blocks, nfac, s, nblk, n, r0, rows, G);
}
void launch_tr_gather_dense(const double* X, int64_t n, int cols, int64_t r0, int64_t rows, double* G,
                            cudaStream_t st) {
  k_tr_gather_dense<<<tr_grid(rows * cols), 256, 0, st>>>(X, n, cols, r0, rows, G);
}
void launch_tr_apply(const TrOp& op, const double* X, int64_t h, int64_t r0, int64_t rows, int r, double* Y,
                     cudaStream_t st) {
  k_tr_apply<<<tr_grid(rows * r), 256, 0, st>>>(op, X, h, r0, rows, r, Y);
}
void launch_tr_fill(double* M, int64_t ldm, int64_t off, int64_t rows, const double* C, int64_t n, int s, int64_t r0,
                    const double* P1, int64_t h1, const double* P2, int64_t h2, int r, double sgn, cudaStream_t st) {
  k_tr_fill<<<tr_grid(rows * (s + 2 * r)), 256, 0, st>>>(M, ldm, off, rows, C, n, s, r0, P1, h1, P2, h2, r, sgn);
}
void launch_tr_fill_rows(double* M, int64_t ldm, int64_t off, int64_t rows, const double* G, int cols,
                         cudaStream_t st) {
  k_tr_fill_rows<<<tr_grid(rows * cols), 256, 0, st>>>(M, ldm, off, rows, G, cols);
}
void launch_tr_keep_r(double* M, int64_t ldm, int wdt, cudaStream_t st) {
  k_tr_keep_r<<<tr_grid((int64_t)wdt * wdt), 256, 0, st>>>(M, ldm, wdt);
}

}  // namespace sk
