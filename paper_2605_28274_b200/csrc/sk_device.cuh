// sk_device.cuh -- shared device-side definitions of the B200 factorized-Krylov
// path: the arithmetic contract (reduction trees), solver state layout and the
// single-thread small-matrix routines (Cholesky, one-sided Jacobi).
//
// Everything here must be compiled with --fmad=false: the written operation
// order is the contract that oracle/sk_oracle.c (SKO_REPRODUCIBLE) restates on
// the CPU, so GPU results are bitwise identical to the oracle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sk {

// ---- arithmetic contract ----
constexpr int kLanes = 32;
constexpr int kLRows = 16;                 // rows per lane per segment
constexpr int kSeg = kLanes * kLRows;      // R1 segment: 512 rows
constexpr int kSegsPerWarp = 4;            // aligned level-2 subtree per warp
constexpr int kWarpsPerCta = 8;            // aligned level-5 subtree per CTA
constexpr int kSegsPerCta = kSegsPerWarp * kWarpsPerCta;  // 32
constexpr int kRowsPerCta = kSeg * kSegsPerCta;           // 16384
// fused Lanczos / self-Gram kernels: one warp per segment, kFusedSegsPerCta
// warps per CTA (an aligned subtree of the canonical tree)
#ifndef SK_FUSED_SEGS
#define SK_FUSED_SEGS 8
#endif
constexpr int kFusedSegsPerCta = SK_FUSED_SEGS;
constexpr int kFusedThreads = 32 * kFusedSegsPerCta;
#ifndef SK_P1_WARPS
#define SK_P1_WARPS 32  // resident warps / SM for pass 1 (register budget 64)
#endif
#ifndef SK_P2_WARPS
#define SK_P2_WARPS 48  // resident warps / SM for pass 2 (register budget 40)
#endif
constexpr int kP1Blocks = SK_P1_WARPS / kFusedSegsPerCta;
constexpr int kP2Blocks = SK_P2_WARPS / kFusedSegsPerCta;
constexpr int kTile = 32;                  // R2 core tile
constexpr int kMaxS = 8;                   // device block-size limit
constexpr double kPythGuard = 0x1p-10;
constexpr double kHHRatio = 1e-6;

enum Status : int { RUNNING = 0, CONVERGED = 1, MAXITER = 2, BREAKDOWN = 3, RANKDEF = 4, FAILED = 5,
                    PAUSED = 6 /* row partition: a rare path waits for the host-driven sequence */ };

// per-extension stage machine of one basis side
enum Stage : int {
  ST_NONE = 0,
  ST_GROW_DIRECT,   // accepted: U_k holds the candidate, N_k = R (CholQR of the direct Gram)
  ST_GROW_HH,       // accepted: U_k holds the Householder Q, N_k = I
  ST_NEED_HH,       // direct Gram ambiguous: Householder on the candidate (first pass)
  ST_NEED_CLEANUP,  // Lanczos clean-up: Gram vs all blocks, update, direct Gram
  ST_NEED_HH2,      // Householder after the clean-up
  ST_DONE_NOGROW,   // exhausted or broken this step (no new block)
  ST_INIT_DIRECT,   // init: U_0 = C, N_0 = R
  ST_INIT_HH        // init: U_0 = Householder Q of C, N_0 = I
};

struct SideState {
  int64_t blocks;      // orthonormal blocks in V
  int64_t steps;       // completed extensions (H block columns)
  int32_t exhausted, broken, stage, pad;
  double hfro2;        // running ||H||_F^2
  double coeff2, r2, scale;
  double smax, smin;
  double R[kMaxS * kMaxS];      // triangular factor of the current candidate
  double gbase[kMaxS * kMaxS];  // R1 Gram of the candidate
  int64_t paths[4];             // direct / householder / clean-up / unused
};

struct DevState {
  int32_t status;
  int32_t phase_err;
  int64_t k;            // iterations completed
  int64_t nrec;         // history records written
  int64_t rows_p, cols_p;  // shape of the current residual / direction core
  int64_t rows_x, cols_x;  // shape of the iterate core
  int64_t rows_q, cols_q;  // shape of the image window of this iteration
  double rho, alpha, beta, omega, norm_r0, norm_shadow, denom;
  int64_t rows_s, cols_s;  // BiCGSTAB: shape of S (= Q's shape)
  int64_t rows_t, cols_t;  // BiCGSTAB: shape of T (= the next residual's shape)
  double tt, ss, st;       // BiCGSTAB reductions
  int64_t rows_po, cols_po;  // BiCGSTAB: shape of the previous direction core
  SideState side[2];
};

// Constant description of one basis side (operator, storage, scratch).
struct SideConst {
  int64_t n;                 // rows
  const int32_t* rp;         // CSR of the operator this side applies (A, or B^T)
  const int32_t* ci;
  const double* val;
  double* const* blocks;     // device table of block pointers (row-interleaved n x s)
  double* w;                 // scratch n x s: op * V_last
  double* wx;                // scratch n x s: CGS2 intermediate / transposed start block
  double* qh;                // scratch n x s: Householder Q
  double* hw;                // scratch n x s: Householder work copy
  double* hband;             // Lanczos H bands [cap_steps][3][s*s] | Arnoldi packed H:
                             // column block e has (e+2)s rows at offset s^2 e(e+3)/2
  int64_t hld;               // unused
  double* nfac;              // [cap_blocks][s*s + s] normalisation factor N_b and 1/diag
  double* coef;              // [cap_blocks][s*s] CGS coefficients (pass 1)
  double* coef2;             // [cap_blocks][s*s] second-pass coefficients
  double* mcoef;             // [cap_blocks][s*s] M_b = N_b^{-1} c_b (pass 1)
  double* mcoef2;            // [cap_blocks][s*s] second-pass M_b
  double* hsq;               // [cap_blocks] Arnoldi: per-block sum of squared H coefficients
  double* part;              // R1 CTA partials
  unsigned int* counter;     // last-CTA counters (several slots)
  int64_t ncta;              // CTAs covering n rows (kRowsPerCta each)
  int64_t nseg;              // R1 segments
  // matrix-free stencil form of the operator (0: use the CSR). Detected on the
  // host from the CSR itself: rows are exactly the Dirichlet-truncated grid
  // stencil with one constant value per offset, in CSR (ascending) order.
  int32_t sdim;              // 2 or 3
  int32_t sg_pow2;           // log2(g) if g is a power of two, else -1
  int64_t sg;                // grid edge g
  double scoef[7];           // values by ascending offset
  // row partition (SolveConst::world > 1): local rows are global rows
  // [row0, row0 + n); block storage carries `halo` ghost rows on each side.
  int64_t row0;
  int32_t dist;              // 1: last CTAs emit chunk nodes instead of finalising
  int32_t pad_;
  int64_t chunk_f;           // fused-kernel CTAs (8 segments) per reduction chunk
  int64_t chunk_g;           // general-kernel CTAs (32 segments) per reduction chunk
  int64_t nch;               // local reduction chunks
  int64_t halo;              // ghost rows per side of a block (0: none)
  double* spart;             // wavefront pass: tile partials (self, raw Grams), final scratch
  unsigned int* sctr;        // wavefront pass: [0] ticket, [1] launch done, [2] side done, [4..] tile flags
  int64_t bw;                // operator bandwidth max |col - row| (wavefront lag)
  double* hsend;             // [2][halo][s] first / last local rows of the newest block
  double* hrecv;             // [2][halo][s] rows received from the previous / next rank
};

struct SolveConst {
  SideConst side[2];
  int32_t nsides;       // 1 (Lyapunov) or 2
  int32_t lyap, arnoldi, full_reorth;
  int32_t s;
  double tol, eps;
  int64_t max_iter;
  // cores (column-major, leading dimension ld)
  double* X;
  double* R;
  double* P[2];
  double* Q;      // BiCGSTAB image of P
  double* S;      // BiCGSTAB S
  double* T;      // BiCGSTAB image of S
  double* Rs;     // BiCGSTAB shadow residual (s x s)
  int64_t ld;
  // row partition: reduction-chunk nodes (outbound, this rank) and the
  // all-gathered messages of every rank (inbound), see sk_kernels.cu "partition"
  int32_t world, rank;
  int64_t nch_max;         // chunk slots per (slot, side) in a message
  int64_t nex;             // doubles per node (2 s^2)
  const int32_t* rank_nch; // [world] chunks owned by each rank
  double* nodes;
  double* gnodes;
  double* cpart;  // R2 tile partials
  unsigned int* ccounter;
  double* hist_rel;   // [max_iter+1]
  double* hist_tk;    // device timestamps (ns) per iteration: extension done
  double* hist_tb;    // device timestamps (ns) per iteration: core done
  DevState* st;
};

// operator description for the true-residual kernels (sk_residual.cu)
struct TrOp {
  int32_t sdim;  // 0: CSR, 2 / 3: matrix-free grid stencil
  int64_t g;
  double c[7];
  const int32_t* rp;
  const int32_t* ci;
  const double* val;
};

__host__ __device__ __forceinline__ int64_t mn64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t mx64(int64_t a, int64_t b) { return a > b ? a : b; }

// ---- reduction building blocks ----
__device__ __forceinline__ double shfl_xor_d(double v, int d) {
  return __shfl_xor_sync(0xffffffffu, v, d);
}
// xor butterfly: t_l <- t_l + t_{l^d}, d = 16..1 (all lanes end identical)
__device__ __forceinline__ double butterfly(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = __dadd_rn(v, shfl_xor_d(v, d));
  return v;
}
// canonical pairwise tree over a[0..count) (in place), aligned-group composable
__device__ inline double tree_reduce_local(double* a, int count) {
  if (count <= 0) return 0.0;
  while (count > 1) {
    const int half = (count + 1) / 2;
    for (int i = 0; i < half; ++i)
      a[i] = (2 * i + 1 < count) ? __dadd_rn(a[2 * i], a[2 * i + 1]) : a[2 * i];
    count = half;
  }
  return a[0];
}
// Streaming evaluation of the canonical pairwise tree (binary-counter stack):
// identical to tree_reduce_local over the same sequence.
struct TreeStream {
  double v[40];
  int lvl[40];
  int top;
  int64_t idx;
  __device__ void init() { top = 0; idx = 0; }
  __device__ void push(double x) {
    // merge while the number of leaves pushed so far has trailing ones
    double cur = x;
    int l = 0;
    int64_t n = idx;
    while (n & 1) {
      cur = __dadd_rn(v[--top], cur);
      ++l;
      n >>= 1;
    }
    v[top] = cur;
    lvl[top] = l;
    ++top;
    ++idx;
  }
  __device__ double finish() {
    if (top == 0) return 0.0;
    double cur = v[--top];
    while (top > 0) cur = __dadd_rn(v[--top], cur);
    return cur;
  }
};
__device__ inline double tree_stream(const double* a, int64_t count, int64_t stride) {
  TreeStream ts;
  ts.init();
  for (int64_t i = 0; i < count; ++i) ts.push(__ldcg(a + i * stride));
  return ts.finish();
}

// ---- small matrices (single thread; identical to oracle/sk_oracle.c) ----
// Cholesky G = R^T R (column-major s x s), R upper. Returns false on failure.
__device__ inline bool cholesky_upper(const double* G, int s, double* R) {
  for (int e = 0; e < s * s; ++e) R[e] = 0.0;
  for (int j = 0; j < s; ++j) {
    for (int i = 0; i < j; ++i) {
      double acc = G[j * s + i];
      for (int t = 0; t < i; ++t) acc = __dsub_rn(acc, __dmul_rn(R[i * s + t], R[j * s + t]));
      R[j * s + i] = __ddiv_rn(acc, R[i * s + i]);
    }
    double acc = G[j * s + j];
    for (int t = 0; t < j; ++t) acc = __dsub_rn(acc, __dmul_rn(R[j * s + t], R[j * s + t]));
    if (!(acc > 0.0) || !isfinite(acc)) return false;
    R[j * s + j] = __dsqrt_rn(acc);
  }
  return true;
}
// One-sided Jacobi singular-value extremes (oracle: jacobi_extremes). Called by
// one thread of a CTA; the work arrays live in shared memory (a runtime-indexed
// local array would go to local memory, i.e. an L2 round trip per access while
// the rest of the GPU waits on this serial finalisation).
__device__ inline void jacobi_extremes(const double* m, int rows, int cols, double* smax,
                                       double* smin) {
  __shared__ double A[kMaxS * kMaxS];
  __shared__ double nv[kMaxS];
  for (int e = 0; e < rows * cols; ++e) A[e] = m[e];
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < cols; ++p)
      for (int q = p + 1; q < cols; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = 0; i < rows; ++i) {
          const double ap = A[p * rows + i], aq = A[q * rows + i];
          al = __dadd_rn(al, __dmul_rn(ap, ap));
          be = __dadd_rn(be, __dmul_rn(aq, aq));
          ga = __dadd_rn(ga, __dmul_rn(ap, aq));
        }
        if (ga == 0.0) continue;
        if (fabs(ga) <= __dmul_rn(__dmul_rn(1e-15, __dsqrt_rn(al)), __dsqrt_rn(be))) continue;
        const double zeta = __ddiv_rn(__dsub_rn(be, al), __dmul_rn(2.0, ga));
        double t;
        if (fabs(zeta) > 1e150)
          t = __ddiv_rn(1.0, __dmul_rn(2.0, zeta));
        else
          t = __ddiv_rn(zeta >= 0.0 ? 1.0 : -1.0,
                        __dadd_rn(fabs(zeta), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(zeta, zeta)))));
        const double c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t))));
        const double sn = __dmul_rn(c, t);
        for (int i = 0; i < rows; ++i) {
          const double ap = A[p * rows + i], aq = A[q * rows + i];
          A[p * rows + i] = __dsub_rn(__dmul_rn(c, ap), __dmul_rn(sn, aq));
          A[q * rows + i] = __dadd_rn(__dmul_rn(sn, ap), __dmul_rn(c, aq));
        }
        rotated = true;
      }
    if (!rotated) break;
  }
  const int k = rows < cols ? rows : cols;
  for (int j = 0; j < cols; ++j) {
    double acc = 0.0;
    for (int i = 0; i < rows; ++i) acc = __dadd_rn(acc, __dmul_rn(A[j * rows + i], A[j * rows + i]));
    nv[j] = __dsqrt_rn(acc);
  }
  for (int x = 0; x < k; ++x) {
    int best = x;
    for (int y = x + 1; y < cols; ++y)
      if (nv[y] > nv[best]) best = y;
    const double t = nv[x];
    nv[x] = nv[best];
    nv[best] = t;
  }
  *smax = k > 0 ? nv[0] : 0.0;
  *smin = k > 0 ? nv[k - 1] : 0.0;
}

// last-CTA-done: returns true in exactly one CTA (the last to arrive).
__device__ inline bool last_cta_arrive(unsigned int* counter, unsigned int total) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == total - 1);
    if (am_last) *counter = 0u;  // reset for the next launch (stream-ordered)
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

__device__ __forceinline__ double ld_nc(const double* p) { return __ldg(p); }

}  // namespace sk
