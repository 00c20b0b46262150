// sk_kernels.cu -- sm_100a kernels of the factorized-Krylov hot path.
//
//  K1  k_spmm<S>          w = op * V_last (CSR gather, stored order, mul+add)
//  K2  k_gram<S>          R1 Gram coefficients V_b^T x (+ x^T x) with last-CTA trees
//      k_update<S>        x -= sum_b V_b c_b (+ R1 self Gram)
//  K3  k_pass2<S>         V_k = (base - V cc) R^-1 (forward substitution per row)
//      k_householder      rare-path single-CTA Householder QR (exact classification)
//  K4  k_cg_a<S>/k_cg_b<S> fused CG core updates: P = R + beta P, Q = H P + P G^T on
//                         the fly from the Lanczos bands, <R,Q>, X += alpha P,
//                         R -= alpha Q, ||R||^2 (R2 tile trees)
//
// Reference ops restated (proj/src): sparse_matrix.cpp:142-200 (SpMM),
// block_krylov.cpp:63-145 (extension), :173-213 (banded products),
// factorized_solvers.cpp:134-192 (CG loop), decompositions.cpp:16-78 (QR).
#include "sk_device.cuh"
#include "sk_launch.h"

#include <cstdio>

namespace sk {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// =====================================================================
// Side finalisation logic (single thread). Mirrors oracle norm_repro +
// classification (block_krylov.cpp:102-144).
// =====================================================================
struct FinalCtx {
  const SolveConst* c;
  int side;
};

__device__ inline double* hb_ptr(const SideConst& sc, int64_t e, int d, int s) {
  return sc.hband + (e * 3 + d) * (int64_t)(s * s);
}

// first block of the orthogonalisation window J
__device__ inline int64_t first_block(const SolveConst& c, int64_t k) {
  return c.arnoldi ? 0 : (k - 2 > 0 ? k - 2 : 0);
}

// coeff2 in the reference loop order (block_krylov.cpp:105-108) over J blocks
__device__ inline double coeff2_of(const SolveConst& c, const SideConst& sc, int64_t k) {
  const int s = c.s, ss = s * s;
  double acc = 0.0;
  for (int64_t jb = first_block(c, k); jb < k; ++jb) {
    const double* h = sc.coef + jb * ss;
    for (int cc = 0; cc < s; ++cc)
      for (int r = 0; r < s; ++r) acc = __dadd_rn(acc, __dmul_rn(h[cc * s + r], h[cc * s + r]));
  }
  return acc;
}

// Commit the outcome of an extension step into H / counters.
__device__ inline void commit_grow(const SolveConst& c, int side) {
  const SideConst& sc = c.side[side];
  SideState& st = c.st->side[side];
  const int s = c.s, ss = s * s;
  const int64_t k = st.blocks, e = st.steps;
  if (!c.arnoldi) {
    double* h0 = hb_ptr(sc, e, 0, s);
    double* h1 = hb_ptr(sc, e, 1, s);
    double* h2 = hb_ptr(sc, e, 2, s);
    for (int x = 0; x < ss; ++x) {
      h0[x] = (k >= 2) ? sc.coef[(k - 2) * ss + x] : 0.0;
      h1[x] = sc.coef[(k - 1) * ss + x];
      h2[x] = st.R[x];
    }
  } else {
    // dense upper block Hessenberg column e: rows [0, (k+1)s)
    for (int cc = 0; cc < s; ++cc) {
      double* col = sc.hband + (e * s + cc) * sc.hld;
      for (int64_t jb = 0; jb < k; ++jb)
        for (int r = 0; r < s; ++r) col[jb * s + r] = sc.coef[jb * ss + cc * s + r];
      for (int r = 0; r < s; ++r) col[k * s + r] = st.R[cc * s + r];
    }
  }
  st.hfro2 = __dadd_rn(__dadd_rn(st.hfro2, st.coeff2), st.r2);
  st.steps = e + 1;
  st.blocks = k + 1;
}
__device__ inline void commit_exhausted(const SolveConst& c, int side) {
  const SideConst& sc = c.side[side];
  SideState& st = c.st->side[side];
  const int s = c.s, ss = s * s;
  const int64_t k = st.blocks, e = st.steps;
  if (!c.arnoldi) {
    double* h0 = hb_ptr(sc, e, 0, s);
    double* h1 = hb_ptr(sc, e, 1, s);
    double* h2 = hb_ptr(sc, e, 2, s);
    for (int x = 0; x < ss; ++x) {
      h0[x] = (k >= 2) ? sc.coef[(k - 2) * ss + x] : 0.0;
      h1[x] = sc.coef[(k - 1) * ss + x];
      h2[x] = 0.0;
    }
  } else {
    for (int cc = 0; cc < s; ++cc) {
      double* col = sc.hband + (e * s + cc) * sc.hld;
      for (int64_t jb = 0; jb < k; ++jb)
        for (int r = 0; r < s; ++r) col[jb * s + r] = sc.coef[jb * ss + cc * s + r];
      for (int r = 0; r < s; ++r) col[k * s + r] = 0.0;
    }
  }
  st.hfro2 = __dadd_rn(st.hfro2, st.coeff2);
  st.steps = e + 1;
  st.exhausted = 1;
  st.stage = ST_DONE_NOGROW;
}

// Classification after sigma extremes are known. first_pass: compute scale.
// grow_stage: stage to use when the block is accepted.
__device__ inline void classify(const SolveConst& c, int side, bool first_pass, int grow_stage) {
  SideState& st = c.st->side[side];
  const int s = c.s, ss = s * s;
  if (first_pass) {
    st.coeff2 = coeff2_of(c, c.side[side], st.blocks);
    double r2 = 0.0;
    for (int x = 0; x < ss; ++x) r2 = __dadd_rn(r2, __dmul_rn(st.R[x], st.R[x]));
    st.r2 = r2;
    st.scale = __dsqrt_rn(__dadd_rn(__dadd_rn(st.hfro2, st.coeff2), st.r2));
    if (!c.arnoldi && st.smin < __dmul_rn(c.tol, st.scale)) {
      st.stage = (grow_stage == ST_GROW_PYTH) ? ST_NEED_MAT_CLEANUP : ST_NEED_CLEANUP;
      return;
    }
  }
  const double lim = __dmul_rn(c.tol, st.scale);
  if (st.smax <= lim || st.scale == 0.0) {
    commit_exhausted(c, side);
    return;
  }
  if (st.smin < lim) {
    st.broken = 1;
    st.stage = ST_DONE_NOGROW;
    return;
  }
  st.stage = grow_stage;
  commit_grow(c, side);
}

// After the Pythagorean Gram is known (gbase, coefficients cc over blocks [c0,k)).
__device__ inline void finalize_pyth(const SolveConst& c, int side, const double* cc, int64_t c0,
                                     int64_t c1) {
  SideState& st = c.st->side[side];
  const int s = c.s, ss = s * s;
  double G[kMaxS * kMaxS];
  for (int u = 0; u < s; ++u)
    for (int t = 0; t < s; ++t) {
      double acc = st.gbase[u * s + t];
      for (int64_t b = c0; b < c1; ++b) {
        const double* cb = cc + b * ss;
        for (int v = 0; v < s; ++v) acc = __dsub_rn(acc, __dmul_rn(cb[t * s + v], cb[u * s + v]));
      }
      G[u * s + t] = acc;
    }
  bool ok = true;
  for (int u = 0; u < s; ++u)
    if (!(G[u * s + u] > __dmul_rn(st.gbase[u * s + u], kPythGuard))) ok = false;
  if (ok) ok = cholesky_upper(G, s, st.R);
  if (ok) {
    jacobi_extremes(st.R, s, s, &st.smax, &st.smin);
    if (st.smin < __dmul_rn(kHHRatio, st.smax)) {
      st.stage = ST_NEED_MAT;  // materialise, then Householder (no direct Gram)
      st.cleanup_done = 2;     // marker: skip direct Gram
      return;
    }
    st.paths[0]++;
    classify(c, side, true, ST_GROW_PYTH);
    return;
  }
  st.stage = ST_NEED_MAT;
  st.cleanup_done = 0;
}

// After a direct Gram of the materialised wx (gbase holds it).
__device__ inline void finalize_direct(const SolveConst& c, int side, bool first_pass) {
  SideState& st = c.st->side[side];
  const int s = c.s;
  bool ok = cholesky_upper(st.gbase, s, st.R);
  if (ok) {
    jacobi_extremes(st.R, s, s, &st.smax, &st.smin);
    if (st.smin < __dmul_rn(kHHRatio, st.smax)) ok = false;
  }
  if (!ok) {
    st.stage = first_pass ? ST_NEED_HH : ST_NEED_HH2;
    return;
  }
  if (first_pass) st.paths[1]++;
  classify(c, side, first_pass, ST_GROW_WX);
}

// =====================================================================
// R1 machinery: per-CTA aligned subtree over 32 segments
// =====================================================================
// Lane-owner storage of NE entries after butterflies: lane owns e = lane + 32*j.
template <int NE>
struct OwnerVals {
  static constexpr int J = (NE + 31) / 32;
  double v[J > 0 ? J : 1];
};

// Combine the per-lane accumulators of one segment into owner registers.
template <int NE>
__device__ __forceinline__ void seg_butterfly(const double* acc, OwnerVals<NE>& out, int lane) {
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double v = butterfly(acc[e]);
    if ((e & 31) == lane) out.v[e >> 5] = v;
  }
}

// After the warp's 4 segments produced owner values segv[q], build the warp node
// and then the CTA node; thread e < NE writes part_out[e].
template <int NE>
__device__ __forceinline__ void cta_combine(OwnerVals<NE> (&segv)[kSegsPerWarp], int nvalid_warp,
                                            int nvalid_cta_segs, double* part_out) {
  __shared__ double wnode[kWarpsPerCta][NE > 0 ? NE : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < OwnerVals<NE>::J; ++j) {
    const int e = lane + 32 * j;
    if (e < NE) {
      double a[kSegsPerWarp];
#pragma unroll
      for (int q = 0; q < kSegsPerWarp; ++q) a[q] = segv[q].v[j];
      wnode[warp][e] = tree_reduce_local(a, nvalid_warp);
    }
  }
  __syncthreads();
  const int nwarps = (nvalid_cta_segs + kSegsPerWarp - 1) / kSegsPerWarp;
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    double a[kWarpsPerCta];
    for (int w = 0; w < kWarpsPerCta; ++w) a[w] = (w < nwarps) ? wnode[w][e] : 0.0;
    part_out[e] = tree_reduce_local(a, nwarps);
  }
}

// =====================================================================
// K1: SpMM  w = op * V_last   (sparse_matrix.cpp:142-158, order preserved)
// =====================================================================
template <int S>
__global__ void __launch_bounds__(256) k_spmm(SolveConst c) {
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.exhausted || ss.broken) return;
  const SideConst& sc = c.side[side];
  const double* __restrict__ x = sc.blocks[ss.blocks - 1];
  double* __restrict__ w = sc.w;
  const int64_t n = sc.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc[S];
#pragma unroll
    for (int u = 0; u < S; ++u) acc[u] = 0.0;
    const int32_t k0 = __ldg(sc.rp + i), k1 = __ldg(sc.rp + i + 1);
    for (int32_t kk = k0; kk < k1; ++kk) {
      const int64_t col = __ldg(sc.ci + kk);
      const double v = __ldg(sc.val + kk);
#pragma unroll
      for (int u = 0; u < S; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(v, __ldg(x + col * S + u)));
    }
#pragma unroll
    for (int u = 0; u < S; ++u) w[i * S + u] = acc[u];
  }
}

// =====================================================================
// K2: R1 Gram of x against blocks [b0, b0+gridDim.y-1) and x^T x (last y).
// Each CTA handles one (row-group, block) pair. Two-level last-CTA:
// per-block trees, then a side-level finalisation in the very last CTA.
// =====================================================================
enum GramMode : int { GM_LANCZOS1 = 0, GM_MAT = 1, GM_CLEAN = 2, GM_ARN1 = 3, GM_ARN2 = 4 };

template <int S>
__device__ void gram_side_finalize(const SolveConst& c, int side, int mode);

// which x does this mode read, and which blocks
template <int S>
__device__ inline bool gram_setup(const SolveConst& c, int side, int mode, const double*& x,
                                  int64_t& b0, int64_t& b1) {
  const DevState* st = c.st;
  if (st->status != RUNNING) return false;
  const SideState& ss = st->side[side];
  const SideConst& sc = c.side[side];
  const int64_t k = ss.blocks;
  switch (mode) {
    case GM_LANCZOS1:  // pass 1 of a Lanczos step: x = w, blocks J
      if (ss.exhausted || ss.broken) return false;
      x = sc.w;
      b0 = first_block(c, k);
      b1 = k;
      return true;
    case GM_MAT:  // direct Gram of materialised wx (self only)
      if (ss.stage != ST_NEED_MAT || ss.cleanup_done == 2) return false;
      x = sc.wx;
      b0 = b1 = 0;
      return true;
    case GM_CLEAN:  // clean-up Gram of wx vs all blocks (no self)
      if (ss.stage != ST_NEED_CLEANUP) return false;
      x = sc.wx;
      b0 = 0;
      b1 = k;
      return true;
    case GM_ARN1:  // Arnoldi pass 1: x = w vs all blocks (no self)
      if (ss.exhausted || ss.broken) return false;
      x = sc.w;
      b0 = 0;
      b1 = k;
      return true;
    case GM_ARN2:  // Arnoldi pass 2: x = wx (= w1) vs all blocks + self
      if (ss.exhausted || ss.broken) return false;
      x = sc.wx;
      b0 = 0;
      b1 = k;
      return true;
  }
  return false;
}
__device__ inline bool gram_has_self(int mode) {
  return mode == GM_LANCZOS1 || mode == GM_MAT || mode == GM_ARN2;
}
__device__ inline double* gram_coef_out(const SideConst& sc, int mode) {
  return (mode == GM_CLEAN || mode == GM_ARN2) ? sc.coef2 : sc.coef;
}

template <int S>
__global__ void __launch_bounds__(256) k_gram(SolveConst c, int mode) {
  constexpr int NB = S * S;
  constexpr int NS = S * (S + 1) / 2;
  const int side = blockIdx.z;
  if (side >= c.nsides) return;
  const double* x;
  int64_t b0, b1;
  if (!gram_setup<S>(c, side, mode, x, b0, b1)) return;
  const bool self = gram_has_self(mode);
  const SideConst& sc = c.side[side];
  const int64_t nblk = (b1 - b0) + (self ? 1 : 0);
  const int64_t by = blockIdx.y;
  if (by >= nblk) return;
  const int64_t cta = blockIdx.x;
  if (cta >= sc.ncta) return;
  const bool is_self = self && by == nblk - 1;
  const double* __restrict__ vb = is_self ? x : sc.blocks[b0 + by];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = sc.n, nseg = sc.nseg;
  const int64_t seg_cta0 = cta * kSegsPerCta;
  const int nvalid_cta = (int)mn64(kSegsPerCta, nseg - seg_cta0);
  const int64_t seg_w0 = seg_cta0 + warp * kSegsPerWarp;
  const int nvalid_warp = (int)mx64(0, mn64(kSegsPerWarp, nseg - seg_w0));
  double* part = sc.part + ((by * sc.ncta + cta) * NB);

  if (!is_self) {
    OwnerVals<NB> segv[kSegsPerWarp];
#pragma unroll
    for (int q = 0; q < kSegsPerWarp; ++q) {
      double acc[NB];
#pragma unroll
      for (int e = 0; e < NB; ++e) acc[e] = 0.0;
      if (q < nvalid_warp) {
        const int64_t base = (seg_w0 + q) * kSeg;
#pragma unroll 4
        for (int m = 0; m < kLRows; ++m) {
          const int64_t i = base + lane + 32 * m;
          if (i < n) {
            double a[S], y[S];
#pragma unroll
            for (int t = 0; t < S; ++t) {
              a[t] = __ldg(vb + i * S + t);
              y[t] = __ldg(x + i * S + t);
            }
#pragma unroll
            for (int u = 0; u < S; ++u)
#pragma unroll
              for (int t = 0; t < S; ++t) acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(a[t], y[u]));
          }
        }
      }
      seg_butterfly<NB>(acc, segv[q], lane);
    }
    cta_combine<NB>(segv, nvalid_warp, nvalid_cta, part);
  } else {
    OwnerVals<NS> segv[kSegsPerWarp];
#pragma unroll
    for (int q = 0; q < kSegsPerWarp; ++q) {
      double acc[NS];
#pragma unroll
      for (int e = 0; e < NS; ++e) acc[e] = 0.0;
      if (q < nvalid_warp) {
        const int64_t base = (seg_w0 + q) * kSeg;
#pragma unroll 4
        for (int m = 0; m < kLRows; ++m) {
          const int64_t i = base + lane + 32 * m;
          if (i < n) {
            double y[S];
#pragma unroll
            for (int t = 0; t < S; ++t) y[t] = __ldg(x + i * S + t);
            int e = 0;
#pragma unroll
            for (int u = 0; u < S; ++u)
#pragma unroll
              for (int t = 0; t <= u; ++t) {
                acc[e] = __dadd_rn(acc[e], __dmul_rn(y[t], y[u]));
                ++e;
              }
          }
        }
      }
      seg_butterfly<NS>(acc, segv[q], lane);
    }
    cta_combine<NS>(segv, nvalid_warp, nvalid_cta, part);
  }

  // level 1: the last CTA of this (side, block) reduces over row groups
  unsigned int* ctr = sc.counter;  // slot 2+by: per-block, slot 0: side
  if (!last_cta_arrive(ctr + 2 + by, (unsigned)sc.ncta)) return;
  {
    const int ne = is_self ? NS : NB;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
      const double v = tree_stream(sc.part + by * sc.ncta * NB + e, sc.ncta, NB);
      if (is_self) {
        // unpack upper triangle into the full symmetric gbase
        int u = 0, t = e;
        while (t > u) {
          t -= u + 1;
          ++u;
        }
        c.st->side[side].gbase[u * S + t] = v;
        c.st->side[side].gbase[t * S + u] = v;
      } else {
        gram_coef_out(sc, mode)[(b0 + by) * NB + e] = v;
      }
    }
  }
  // level 2: the last block-level reducer finalises the side
  if (!last_cta_arrive(ctr + 0, (unsigned)nblk)) return;
  if (threadIdx.x == 0) gram_side_finalize<S>(c, side, mode);
}

template <int S>
__device__ void gram_side_finalize(const SolveConst& c, int side, int mode) {
  SideState& st = c.st->side[side];
  const SideConst& sc = c.side[side];
  const int64_t k = st.blocks;
  switch (mode) {
    case GM_LANCZOS1:
      st.cleanup_done = 0;
      finalize_pyth(c, side, sc.coef, first_block(c, k), k);
      break;
    case GM_MAT:
      finalize_direct(c, side, true);
      break;
    case GM_CLEAN:
      break;  // coefficients stored; update kernel follows
    case GM_ARN1:
      break;  // update kernel follows
    case GM_ARN2: {
      // H column = c1 + c2 (block_krylov.cpp:87-93 folds both passes)
      // keep c2 for the Pythagorean Gram; coef becomes the H coefficients after.
      double cc2[kMaxS * kMaxS];
      (void)cc2;
      st.cleanup_done = 0;
      finalize_pyth(c, side, sc.coef2, 0, k);
      break;
    }
  }
}

// =====================================================================
// x_out = x_in - sum_{b in [b0,b1)} V_b c_b  (+ R1 self Gram of x_out)
// modes: UM_MAT (wx = base - V cc, then direct Gram),
//        UM_CLEAN (wx -= V d over all blocks, then direct Gram),
//        UM_ARN (wx = w - V c1 over all blocks; Gram vs blocks follows)
// =====================================================================
enum UpdMode : int { UM_MAT = 0, UM_CLEAN = 1, UM_ARN = 2 };

template <int S>
__global__ void __launch_bounds__(256) k_update(SolveConst c, int mode) {
  constexpr int NS = S * (S + 1) / 2;
  const int side = blockIdx.z;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  const SideConst& sc = c.side[side];
  const int64_t k = ss.blocks;
  const double* xin;
  const double* coef;
  int64_t b0, b1;
  bool gram = true;
  if (mode == UM_MAT) {
    if (!(ss.stage == ST_NEED_MAT || ss.stage == ST_NEED_MAT_CLEANUP)) return;
    // base = w (Lanczos) or w1 (Arnoldi / full reorth, already in wx)
    xin = c.arnoldi ? sc.wx : sc.w;
    coef = c.arnoldi ? sc.coef2 : sc.coef;
    b0 = c.arnoldi ? 0 : first_block(c, k);
    b1 = k;
    gram = (ss.stage == ST_NEED_MAT && ss.cleanup_done != 2);
  } else if (mode == UM_CLEAN) {
    if (ss.stage != ST_NEED_CLEANUP) return;
    xin = sc.wx;
    coef = sc.coef2;
    b0 = 0;
    b1 = k;
  } else {
    if (ss.exhausted || ss.broken) return;
    xin = sc.w;
    coef = sc.coef;
    b0 = 0;
    b1 = k;
    gram = false;
  }
  const int64_t cta = blockIdx.x;
  if (cta >= sc.ncta) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = sc.n, nseg = sc.nseg;
  const int64_t seg_cta0 = cta * kSegsPerCta;
  const int nvalid_cta = (int)mn64(kSegsPerCta, nseg - seg_cta0);
  const int64_t seg_w0 = seg_cta0 + warp * kSegsPerWarp;
  const int nvalid_warp = (int)mx64(0, mn64(kSegsPerWarp, nseg - seg_w0));
  double* __restrict__ xout = sc.wx;
  __shared__ double cs[kMaxS * kMaxS * 16];

  OwnerVals<NS> segv[kSegsPerWarp];
#pragma unroll 1
  for (int q = 0; q < kSegsPerWarp; ++q) {
    double acc[NS];
#pragma unroll
    for (int e = 0; e < NS; ++e) acc[e] = 0.0;
    if (q < nvalid_warp) {
      const int64_t base = (seg_w0 + q) * kSeg;
#pragma unroll 1
      for (int m = 0; m < kLRows; ++m) {
        const int64_t i = base + lane + 32 * m;
        if (i < n) {
          double y[S];
#pragma unroll
          for (int u = 0; u < S; ++u) y[u] = __ldcg(xin + i * S + u);
          for (int64_t b = b0; b < b1; ++b) {
            const double* vb = sc.blocks[b];
            const double* cb = coef + b * (S * S);
            double a[S];
#pragma unroll
            for (int t = 0; t < S; ++t) a[t] = __ldg(vb + i * S + t);
#pragma unroll
            for (int u = 0; u < S; ++u) {
              double tmp = 0.0;
#pragma unroll
              for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(a[t], __ldg(cb + u * S + t)));
              y[u] = __dsub_rn(y[u], tmp);
            }
          }
#pragma unroll
          for (int u = 0; u < S; ++u) xout[i * S + u] = y[u];
          int e = 0;
#pragma unroll
          for (int u = 0; u < S; ++u)
#pragma unroll
            for (int t = 0; t <= u; ++t) {
              acc[e] = __dadd_rn(acc[e], __dmul_rn(y[t], y[u]));
              ++e;
            }
        }
      }
    }
    if (gram) seg_butterfly<NS>(acc, segv[q], lane);
  }
  (void)cs;
  if (!gram) return;
  double* part = sc.part + cta * NS;
  cta_combine<NS>(segv, nvalid_warp, nvalid_cta, part);
  if (!last_cta_arrive(sc.counter + 1, (unsigned)sc.ncta)) return;
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    const double v = tree_stream(sc.part + e, sc.ncta, NS);
    int u = 0, t = e;
    while (t > u) {
      t -= u + 1;
      ++u;
    }
    c.st->side[side].gbase[u * S + t] = v;
    c.st->side[side].gbase[t * S + u] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    SideState& sst = c.st->side[side];
    if (mode == UM_MAT) {
      finalize_direct(c, side, true);
    } else if (mode == UM_CLEAN) {
      sst.paths[3]++;
      sst.cleanup_done = 1;
      finalize_direct(c, side, false);
    }
  }
}

// Materialise only (no Gram): NEED_MAT with Householder marker, or clean-up prep.
// Implemented by k_update(UM_MAT) with gram=false; stage transition here:
static __global__ void k_mat_transition(SolveConst c) {
  const int side = threadIdx.x;
  if (side >= c.nsides || c.st->status != RUNNING) return;
  SideState& st = c.st->side[side];
  if (st.stage == ST_NEED_MAT && st.cleanup_done == 2) st.stage = ST_NEED_HH;
  else if (st.stage == ST_NEED_MAT_CLEANUP) st.stage = ST_NEED_CLEANUP;
}

// =====================================================================
// Rare path: single-CTA Householder QR of wx (decompositions.cpp:16-78 with
// R1 reductions). Writes Q to qh (row-interleaved) and R to the side state.
// =====================================================================
static __device__ double cta_r1_dot(const double* x, int sx, int cx, const double* y, int sy, int cy,
                             int64_t n, int64_t row0, double* segbuf) {
  // R1 over rows [row0, n) of x(i,cx)*y(i,cy); segment partials by warps, then stream tree.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t nseg = (n + kSeg - 1) / kSeg;
  for (int64_t g = warp; g < nseg; g += nw) {
    double acc = 0.0;
    for (int m = 0; m < kLRows; ++m) {
      const int64_t i = g * kSeg + lane + 32 * m;
      if (i < n && i >= row0) acc = __dadd_rn(acc, __dmul_rn(x[i * sx + cx], y[i * sy + cy]));
    }
    acc = butterfly(acc);
    if (lane == 0) segbuf[g] = acc;
  }
  __threadfence_block();
  __syncthreads();
  __shared__ double res;
  if (threadIdx.x == 0) res = tree_stream(segbuf, nseg, 1);
  __syncthreads();
  const double r = res;
  __syncthreads();
  return r;
}

template <int S>
__device__ void householder_cta(double* W, double* Q, int64_t n, double* R, double* segbuf) {
  const int p = (int)(n < S ? n : S);
  __shared__ double tau[kMaxS], proj[kMaxS], sh[4];
  for (int j = 0; j < p; ++j) {
    const double nrm2 = cta_r1_dot(W, S, j, W, S, j, n, j, segbuf);
    const double norm = __dsqrt_rn(nrm2);
    if (threadIdx.x == 0) tau[j] = 0.0;
    __syncthreads();
    if (norm == 0.0) continue;
    if (threadIdx.x == 0) {
      const double wjj = W[j * S + j];
      const double alpha = wjj >= 0.0 ? -norm : norm;
      const double v0 = __dsub_rn(wjj, alpha);
      W[j * S + j] = alpha;
      tau[j] = __ddiv_rn(-v0, alpha);
      sh[0] = v0;
    }
    __syncthreads();
    const double v0 = sh[0], t = tau[j];
    for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x) W[i * S + j] = __ddiv_rn(W[i * S + j], v0);
    __threadfence_block();
    __syncthreads();
    const int64_t tail = n - j - 1;
    if (S - j - 1 > 0) {
      for (int cc = j + 1; cc < S; ++cc) {
        double d = 0.0;
        if (tail > 0) d = cta_r1_dot(W, S, j, W, S, cc, n, j + 1, segbuf);
        if (threadIdx.x == 0) {
          double pr = W[j * S + cc];
          if (tail > 0) pr = __dadd_rn(pr, d);
          proj[cc] = __dmul_rn(pr, t);
        }
        __syncthreads();
      }
      if (threadIdx.x == 0)
        for (int cc = j + 1; cc < S; ++cc) W[j * S + cc] = __dsub_rn(W[j * S + cc], proj[cc]);
      for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
        for (int cc = j + 1; cc < S; ++cc)
          W[i * S + cc] = __dsub_rn(W[i * S + cc], __dmul_rn(W[i * S + j], proj[cc]));
      __threadfence_block();
      __syncthreads();
    }
  }
  // Q accumulation
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    for (int cc = 0; cc < S; ++cc) Q[i * S + cc] = (i == cc && cc < p) ? 1.0 : 0.0;
  __threadfence_block();
  __syncthreads();
  for (int j = p - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    const int64_t tail = n - j - 1;
    for (int cc = j; cc < p; ++cc) {
      double d = 0.0;
      if (tail > 0) d = cta_r1_dot(W, S, j, Q, S, cc, n, j + 1, segbuf);
      if (threadIdx.x == 0) {
        double pr = Q[j * S + cc];
        if (tail > 0) pr = __dadd_rn(pr, d);
        proj[cc] = __dmul_rn(pr, t);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0)
      for (int cc = j; cc < p; ++cc) Q[j * S + cc] = __dsub_rn(Q[j * S + cc], proj[cc]);
    for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
      for (int cc = j; cc < p; ++cc) Q[i * S + cc] = __dsub_rn(Q[i * S + cc], __dmul_rn(W[i * S + j], proj[cc]));
    __threadfence_block();
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int e = 0; e < S * S; ++e) R[e] = 0.0;
    for (int jj = 0; jj < S; ++jj)
      for (int i = 0; i <= (jj < p - 1 ? jj : p - 1); ++i) R[jj * S + i] = W[i * S + jj];
  }
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    const bool neg = R[j * S + j] < 0.0;
    __syncthreads();
    if (neg) {
      if (threadIdx.x == 0)
        for (int cc = j; cc < S; ++cc) R[cc * S + j] = -R[cc * S + j];
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) Q[i * S + j] = -Q[i * S + j];
    }
    __threadfence_block();
    __syncthreads();
  }
}

// Householder of wx (work, destroyed) for sides whose stage asks for it.
template <int S>
__global__ void __launch_bounds__(1024) k_householder(SolveConst c, int which /*0: HH, 1: HH2*/) {
  const int side = blockIdx.x;
  if (side >= c.nsides || c.st->status != RUNNING) return;
  SideState& st = c.st->side[side];
  const int want = which == 0 ? ST_NEED_HH : ST_NEED_HH2;
  if (st.stage != want) return;
  const SideConst& sc = c.side[side];
  __shared__ double R[kMaxS * kMaxS];
  for (int64_t i = threadIdx.x; i < sc.n * S; i += blockDim.x) sc.hw[i] = sc.wx[i];
  __syncthreads();
  householder_cta<S>(sc.hw, sc.qh, sc.n, R, sc.part);
  if (threadIdx.x == 0) {
    for (int e = 0; e < S * S; ++e) st.R[e] = R[e];
    jacobi_extremes(st.R, S, S, &st.smax, &st.smin);
    if (which == 0) st.paths[2]++;
    classify(c, side, which == 0, ST_GROW_HH);
  }
}

// =====================================================================
// K3: write the new block  (block_krylov.cpp:139-144 append_block)
// =====================================================================
template <int S>
__global__ void __launch_bounds__(256) k_pass2(SolveConst c) {
  const int side = blockIdx.y;
  if (side >= c.nsides || c.st->status != RUNNING) return;
  const SideState& st = c.st->side[side];
  const int stage = st.stage;
  if (stage != ST_GROW_PYTH && stage != ST_GROW_WX && stage != ST_GROW_HH) return;
  const SideConst& sc = c.side[side];
  const int64_t knew = st.blocks - 1;  // committed already
  double* __restrict__ out = sc.blocks[knew];
  const int64_t n = sc.n;
  __shared__ double Rs[S * S];
  __shared__ double cs[2 * S * S];
  if (threadIdx.x < S * S) Rs[threadIdx.x] = st.R[threadIdx.x];
  const int64_t kold = knew;  // blocks before this step
  const int64_t b0 = c.arnoldi ? 0 : first_block(c, kold);
  const double* coef = c.arnoldi ? sc.coef2 : sc.coef;
  const double* base = c.arnoldi ? sc.wx : sc.w;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double y[S];
    if (stage == ST_GROW_HH) {
#pragma unroll
      for (int u = 0; u < S; ++u) out[i * S + u] = sc.qh[i * S + u];
      continue;
    }
    if (stage == ST_GROW_WX) {
#pragma unroll
      for (int u = 0; u < S; ++u) y[u] = __ldcg(sc.wx + i * S + u);
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u) y[u] = __ldcg(base + i * S + u);
      for (int64_t b = b0; b < kold; ++b) {
        const double* vb = sc.blocks[b];
        const double* cb = coef + b * (S * S);
        double a[S];
#pragma unroll
        for (int t = 0; t < S; ++t) a[t] = __ldg(vb + i * S + t);
#pragma unroll
        for (int u = 0; u < S; ++u) {
          double tmp = 0.0;
#pragma unroll
          for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(a[t], __ldg(cb + u * S + t)));
          y[u] = __dsub_rn(y[u], tmp);
        }
      }
    }
    double q[S];
#pragma unroll
    for (int u = 0; u < S; ++u) {
      double acc = y[u];
#pragma unroll
      for (int t = 0; t < u; ++t) acc = __dsub_rn(acc, __dmul_rn(q[t], Rs[u * S + t]));
      q[u] = __ddiv_rn(acc, Rs[u * S + u]);
    }
#pragma unroll
    for (int u = 0; u < S; ++u) out[i * S + u] = q[u];
  }
  (void)cs;
}

// =====================================================================
// Basis initialisation (block_krylov.cpp:27-52): C (column-major, n x s) is
// transposed into wx, R1 Gram, CholQR with Householder fallback, rank check.
// =====================================================================
template <int S>
__global__ void k_init_transpose(SolveConst c, const double* c1, const double* c2) {
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const SideConst& sc = c.side[side];
  const double* src = side == 0 ? c1 : c2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < sc.n;
       i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int u = 0; u < S; ++u) sc.wx[i * S + u] = src[u * sc.n + i];
}

template <int S>
__global__ void __launch_bounds__(256) k_init_gram(SolveConst c) {
  constexpr int NS = S * (S + 1) / 2;
  const int side = blockIdx.z;
  if (side >= c.nsides) return;
  const SideConst& sc = c.side[side];
  const int64_t cta = blockIdx.x;
  if (cta >= sc.ncta) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = sc.n, nseg = sc.nseg;
  const int64_t seg_cta0 = cta * kSegsPerCta;
  const int nvalid_cta = (int)mn64(kSegsPerCta, nseg - seg_cta0);
  const int64_t seg_w0 = seg_cta0 + warp * kSegsPerWarp;
  const int nvalid_warp = (int)mx64(0, mn64(kSegsPerWarp, nseg - seg_w0));
  const double* x = sc.wx;
  OwnerVals<NS> segv[kSegsPerWarp];
  for (int q = 0; q < kSegsPerWarp; ++q) {
    double acc[NS];
#pragma unroll
    for (int e = 0; e < NS; ++e) acc[e] = 0.0;
    if (q < nvalid_warp) {
      const int64_t base = (seg_w0 + q) * kSeg;
      for (int m = 0; m < kLRows; ++m) {
        const int64_t i = base + lane + 32 * m;
        if (i < n) {
          double y[S];
#pragma unroll
          for (int t = 0; t < S; ++t) y[t] = x[i * S + t];
          int e = 0;
#pragma unroll
          for (int u = 0; u < S; ++u)
#pragma unroll
            for (int t = 0; t <= u; ++t) {
              acc[e] = __dadd_rn(acc[e], __dmul_rn(y[t], y[u]));
              ++e;
            }
        }
      }
    }
    seg_butterfly<NS>(acc, segv[q], lane);
  }
  cta_combine<NS>(segv, nvalid_warp, nvalid_cta, sc.part + cta * NS);
  if (!last_cta_arrive(sc.counter + 1, (unsigned)sc.ncta)) return;
  SideState& st = c.st->side[side];
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    const double v = tree_stream(sc.part + e, sc.ncta, NS);
    int u = 0, t = e;
    while (t > u) {
      t -= u + 1;
      ++u;
    }
    st.gbase[u * S + t] = v;
    st.gbase[t * S + u] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // Pythagorean step with no prior blocks: G' = G; guard G(u,u) > 2^-10 G(u,u)
    bool ok = true;
    for (int u = 0; u < S; ++u)
      if (!(st.gbase[u * S + u] > __dmul_rn(st.gbase[u * S + u], kPythGuard))) ok = false;
    if (ok) ok = cholesky_upper(st.gbase, S, st.R);
    if (ok) {
      jacobi_extremes(st.R, S, S, &st.smax, &st.smin);
      if (st.smin < __dmul_rn(kHHRatio, st.smax)) {
        st.stage = ST_NEED_HH;  // Householder directly on C
        st.paths[2]++;
      } else {
        st.stage = ST_GROW_WX;
        st.paths[0]++;
      }
    } else {
      // direct Gram of the same data == gbase: repeat the decision (explicit path)
      ok = cholesky_upper(st.gbase, S, st.R);
      if (ok) {
        jacobi_extremes(st.R, S, S, &st.smax, &st.smin);
        if (st.smin < __dmul_rn(kHHRatio, st.smax)) ok = false;
      }
      if (ok) {
        st.stage = ST_GROW_WX;
        st.paths[1]++;
      } else {
        st.stage = ST_NEED_HH;
        st.paths[2]++;
      }
    }
  }
}

template <int S>
__global__ void __launch_bounds__(1024) k_init_householder(SolveConst c) {
  const int side = blockIdx.x;
  if (side >= c.nsides) return;
  SideState& st = c.st->side[side];
  if (st.stage != ST_NEED_HH) return;
  const SideConst& sc = c.side[side];
  __shared__ double R[kMaxS * kMaxS];
  householder_cta<S>(sc.wx, sc.qh, sc.n, R, sc.part);
  if (threadIdx.x == 0) {
    for (int e = 0; e < S * S; ++e) st.R[e] = R[e];
    jacobi_extremes(st.R, S, S, &st.smax, &st.smin);
    st.stage = ST_GROW_HH;
  }
}

// V_0 = C R^-1 (or Q_h); rank check (block_krylov.cpp:38-40)
template <int S>
__global__ void k_init_write(SolveConst c) {
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const SideState& st = c.st->side[side];
  const SideConst& sc = c.side[side];
  if (st.smin < __dmul_rn(1e-12, st.smax) || st.smax == 0.0) return;  // rank deficient
  double* out = sc.blocks[0];
  __shared__ double Rs[S * S];
  if (threadIdx.x < S * S) Rs[threadIdx.x] = st.R[threadIdx.x];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < sc.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (st.stage == ST_GROW_HH) {
#pragma unroll
      for (int u = 0; u < S; ++u) out[i * S + u] = sc.qh[i * S + u];
      continue;
    }
    double q[S];
#pragma unroll
    for (int u = 0; u < S; ++u) {
      double acc = sc.wx[i * S + u];
#pragma unroll
      for (int t = 0; t < u; ++t) acc = __dsub_rn(acc, __dmul_rn(q[t], Rs[u * S + t]));
      q[u] = __ddiv_rn(acc, Rs[u * S + u]);
    }
#pragma unroll
    for (int u = 0; u < S; ++u) out[i * S + u] = q[u];
  }
}

// R_0 = R_L R_R^T, P_0 = R_0, rho_0 = <R_0,R_0> (factorized_solvers.cpp:121-131)
static __global__ void k_core_init(SolveConst c) {
  DevState* st = c.st;
  const int s = c.s;
  if (threadIdx.x != 0) return;
  const SideState& a = st->side[0];
  const SideState& b = st->side[c.nsides > 1 ? 1 : 0];
  bool rd = false;
  for (int sd = 0; sd < c.nsides; ++sd) {
    const SideState& x = st->side[sd];
    if (x.smin < __dmul_rn(1e-12, x.smax) || x.smax == 0.0) rd = true;
  }
  if (rd) {
    st->status = RANKDEF;
    return;
  }
  for (int sd = 0; sd < c.nsides; ++sd) {
    st->side[sd].blocks = 1;
    st->side[sd].steps = 0;
    st->side[sd].stage = ST_NONE;
  }
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < s; ++i) {
      double acc = 0.0;
      for (int t = 0; t < s; ++t) acc = __dadd_rn(acc, __dmul_rn(a.R[t * s + i], b.R[t * s + j]));
      c.R[j * c.ld + i] = acc;
      c.P[0][j * c.ld + i] = acc;
      if (c.Rs) c.Rs[j * s + i] = acc;
    }
  // R2 contract over the s x s window (single tile)
  double lane[32];
  for (int l = 0; l < 32; ++l) {
    double acc = 0.0;
    if (l < s)
      for (int j = 0; j < s && j < 32; ++j) acc = __dadd_rn(acc, __dmul_rn(c.R[j * c.ld + l], c.R[j * c.ld + l]));
    lane[l] = acc;
  }
  for (int d = 16; d >= 1; d >>= 1) {
    double tmp[32];
    for (int l = 0; l < 32; ++l) tmp[l] = __dadd_rn(lane[l], lane[l ^ d]);
    for (int l = 0; l < 32; ++l) lane[l] = tmp[l];
  }
  st->rho = lane[0];
  st->norm_r0 = __dsqrt_rn(lane[0]);
  st->norm_shadow = st->norm_r0;
  st->rows_p = st->cols_p = s;
  st->rows_x = st->cols_x = 0;
  st->k = 0;
  st->nrec = 1;
  c.hist_rel[0] = 1.0;
  c.hist_tb[0] = (double)globaltimer();
  c.hist_tk[0] = c.hist_tb[0];
  st->status = RUNNING;
}

// =====================================================================
// K4: CG core kernels (factorized_solvers.cpp:150-189 fused)
// =====================================================================
// Band coefficient H(i,l) for |b(i)-b(l)| <= 1 from the Lanczos band store.
__device__ __forceinline__ double band_at(const double* hband, int s, int64_t i, int64_t l) {
  const int64_t bi = i / s, bl = l / s;
  const int64_t d = bi - bl + 1;
  return hband[(bl * 3 + d) * (s * s) + (l % s) * s + (i % s)];
}

template <int S>
struct CgTile {
  static constexpr int H = 2 * S;           // halo
  static constexpr int D = kTile + 2 * H;   // staged edge
};

// Load the staged P region (rows [i0-H, i0+32+H) x cols [j0-H, j0+32+H)).
// mode 0: P = R (k==0) or R + beta*Pprev; mode 1: P read from Pcur.
template <int S>
__device__ void stage_p(double* sp, const SolveConst& c, int64_t i0, int64_t j0, int64_t rows_p,
                        int64_t cols_p, int mode, const double* Pprev, const double* Pcur, double beta,
                        bool first) {
  constexpr int H = CgTile<S>::H, D = CgTile<S>::D;
  for (int idx = threadIdx.x; idx < D * D; idx += blockDim.x) {
    const int li = idx % D, lj = idx / D;
    const int64_t i = i0 - H + li, j = j0 - H + lj;
    double v = 0.0;
    if (i >= 0 && j >= 0 && i < rows_p && j < cols_p) {
      const int64_t o = j * c.ld + i;
      if (mode == 1)
        v = Pcur[o];
      else if (first)
        v = c.R[o];
      else
        v = __dadd_rn(c.R[o], __dmul_rn(beta, Pprev[o]));
    }
    sp[lj * D + li] = v;
  }
}

// q(i,j) from the staged P (local coords), bands of V (hv) and W (hw)
template <int S>
__device__ __forceinline__ double image_at(const double* sp, const double* hv, const double* hw,
                                           int64_t i, int64_t j, int64_t i0, int64_t j0, int64_t pr,
                                           int64_t pc) {
  constexpr int H = CgTile<S>::H, D = CgTile<S>::D;
  const int64_t JBr = pr / S, JBc = pc / S;
  const bool hasH = j < pc, hasG = i < pr;
  double hpart = 0.0, gpart = 0.0;
  if (hasH) {
    const int64_t bi = i / S;
    const int64_t lo = bi - 1 > 0 ? bi - 1 : 0, hi = bi + 1 < JBr - 1 ? bi + 1 : JBr - 1;
    for (int64_t jb = lo; jb <= hi; ++jb) {
      double d = 0.0;
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const int64_t l = jb * S + t;
        d = __dadd_rn(d, __dmul_rn(band_at(hv, S, i, l), sp[(j - j0 + H) * D + (l - i0 + H)]));
      }
      hpart = __dadd_rn(hpart, d);
    }
  }
  if (hasG) {
    const int64_t bj = j / S;
    const int64_t lo = bj - 1 > 0 ? bj - 1 : 0, hi = bj + 1 < JBc - 1 ? bj + 1 : JBc - 1;
    for (int64_t jb = lo; jb <= hi; ++jb) {
      double d = 0.0;
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const int64_t l = jb * S + t;
        d = __dadd_rn(d, __dmul_rn(sp[(l - j0 + H) * D + (i - i0 + H)], band_at(hw, S, j, l)));
      }
      gpart = __dadd_rn(gpart, d);
    }
  }
  if (hasH && hasG) return __dadd_rn(hpart, gpart);
  return hasH ? hpart : (hasG ? gpart : 0.0);
}

// tile partial: f values in smem f[c][row]; warp 0 sums sequentially, butterflies.
__device__ __forceinline__ double tile_reduce(const double* f, int nrows, int ncols) {
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  if (lane < nrows)
    for (int cc = 0; cc < ncols; ++cc) acc = __dadd_rn(acc, f[cc * kTile + lane]);
  return butterfly(acc);
}

// R2 final: per tile column tree over ti, then over tj (streamed).
static __device__ double r2_final(const double* part, int64_t nti, int64_t ntj, double* scratch) {
  for (int64_t tj = threadIdx.x; tj < ntj; tj += blockDim.x)
    scratch[tj] = tree_stream(part + tj * nti, nti, 1);
  __threadfence_block();
  __syncthreads();
  __shared__ double res;
  if (threadIdx.x == 0) {
    TreeStream ts;
    ts.init();
    for (int64_t tj = 0; tj < ntj; ++tj) ts.push(scratch[tj]);
    res = ts.finish();
  }
  __syncthreads();
  return res;
}

__device__ inline bool any_side_broken(const SolveConst& c) {
  for (int s = 0; s < c.nsides; ++s)
    if (c.st->side[s].broken) return true;
  return false;
}

template <int S>
__global__ void __launch_bounds__(256) k_cg_a(SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  if (any_side_broken(c)) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      st->status = BREAKDOWN;
      c.hist_rel[st->k + 1] = c.hist_rel[st->k];
      c.hist_tk[st->k + 1] = (double)globaltimer();
      c.hist_tb[st->k + 1] = c.hist_tk[st->k + 1];
      st->nrec = st->k + 2;
    }
    return;
  }
  const int64_t k = st->k;
  const int64_t rows_p = st->rows_p, cols_p = st->cols_p;
  const int64_t nti = (rows_p + kTile - 1) / kTile, ntj = (cols_p + kTile - 1) / kTile;
  const int64_t ti = blockIdx.x, tj = blockIdx.y;
  if (ti >= nti || tj >= ntj) return;
  if (ti == 0 && tj == 0 && threadIdx.x == 0) c.hist_tk[k + 1] = (double)globaltimer();
  constexpr int D = CgTile<S>::D;
  __shared__ double sp[D * D];
  __shared__ double f[kTile * kTile];
  const int64_t i0 = ti * kTile, j0 = tj * kTile;
  const double* Pprev = c.P[(k + 1) & 1];
  double* Pnew = c.P[k & 1];
  stage_p<S>(sp, c, i0, j0, rows_p, cols_p, 0, Pprev, nullptr, st->beta, k == 0);
  __syncthreads();
  const SideConst& sv = c.side[0];
  const SideConst& sw = c.side[c.nsides > 1 ? 1 : 0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = i0 + lane;
  for (int q = 0; q < 4; ++q) {
    const int lc = warp * 4 + q;
    const int64_t j = j0 + lc;
    double fv = 0.0;
    if (i < rows_p && j < cols_p) {
      constexpr int H = CgTile<S>::H;
      const double pv = sp[(lc + H) * D + (lane + H)];
      Pnew[j * c.ld + i] = pv;
      const double qv = image_at<S>(sp, sv.hband, sw.hband, i, j, i0, j0, rows_p, cols_p);
      fv = __dmul_rn(c.R[j * c.ld + i], qv);
    }
    f[lc * kTile + lane] = fv;
  }
  __syncthreads();
  if (warp == 0) {
    const int nr = (int)mn64(kTile, rows_p - i0), nc = (int)mn64(kTile, cols_p - j0);
    const double v = tile_reduce(f, nr, nc);
    if (lane == 0) c.cpart[tj * nti + ti] = v;
  }
  if (!last_cta_arrive(c.ccounter, (unsigned)(nti * ntj))) return;
  __shared__ double scratch[256];
  double* scr = ntj <= 256 ? scratch : c.cpart + nti * ntj;
  const double denom = r2_final(c.cpart, nti, ntj, scr);
  if (threadIdx.x == 0) {
    st->denom = denom;
    // breakdown guard (factorized_solvers.cpp:155-160)
    if (fabs(denom) < __dmul_rn(c.tol, st->rho)) {
      st->status = BREAKDOWN;
      c.hist_rel[k + 1] = c.hist_rel[k];
      c.hist_tb[k + 1] = (double)globaltimer();
      st->nrec = k + 2;
      return;
    }
    st->alpha = __ddiv_rn(st->rho, denom);
    const int64_t vc = st->side[0].blocks * S;
    const int64_t wc = st->side[c.nsides > 1 ? 1 : 0].blocks * S;
    const int64_t sched = (k + 2) * S;
    st->rows_q = sched < vc ? sched : vc;
    st->cols_q = sched < wc ? sched : wc;
  }
}

template <int S>
__global__ void __launch_bounds__(256) k_cg_b(SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int64_t k = st->k;
  const int64_t rows_p = st->rows_p, cols_p = st->cols_p;
  const int64_t rows_q = st->rows_q, cols_q = st->cols_q;
  const int64_t nti = (rows_q + kTile - 1) / kTile, ntj = (cols_q + kTile - 1) / kTile;
  const int64_t ti = blockIdx.x, tj = blockIdx.y;
  if (ti >= nti || tj >= ntj) return;
  constexpr int D = CgTile<S>::D, H = CgTile<S>::H;
  __shared__ double sp[D * D];
  __shared__ double f[kTile * kTile];
  const int64_t i0 = ti * kTile, j0 = tj * kTile;
  const double* Pcur = c.P[k & 1];
  stage_p<S>(sp, c, i0, j0, rows_p, cols_p, 1, nullptr, Pcur, 0.0, false);
  __syncthreads();
  const SideConst& sv = c.side[0];
  const SideConst& sw = c.side[c.nsides > 1 ? 1 : 0];
  const double alpha = st->alpha, nalpha = -alpha;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = i0 + lane;
  for (int q = 0; q < 4; ++q) {
    const int lc = warp * 4 + q;
    const int64_t j = j0 + lc;
    double fv = 0.0;
    if (i < rows_q && j < cols_q) {
      const double qv = image_at<S>(sp, sv.hband, sw.hband, i, j, i0, j0, rows_p, cols_p);
      const int64_t o = j * c.ld + i;
      const bool inp = i < rows_p && j < cols_p;
      const double remb = inp ? c.R[o] : 0.0;
      const double rn = __dadd_rn(remb, __dmul_rn(nalpha, qv));
      c.R[o] = rn;
      fv = __dmul_rn(rn, rn);
      if (inp) {
        const double pv = sp[(lc + H) * D + (lane + H)];
        c.X[o] = __dadd_rn(c.X[o], __dmul_rn(alpha, pv));
      }
    }
    f[lc * kTile + lane] = fv;
  }
  __syncthreads();
  if (warp == 0) {
    const int nr = (int)mn64(kTile, rows_q - i0), nc = (int)mn64(kTile, cols_q - j0);
    const double v = tile_reduce(f, nr, nc);
    if (lane == 0) c.cpart[tj * nti + ti] = v;
  }
  if (!last_cta_arrive(c.ccounter, (unsigned)(nti * ntj))) return;
  __shared__ double scratch[256];
  double* scr = ntj <= 256 ? scratch : c.cpart + nti * ntj;
  const double rho_next = r2_final(c.cpart, nti, ntj, scr);
  if (threadIdx.x == 0) {
    const double norm_r = __dsqrt_rn(rho_next);
    const double rel = __ddiv_rn(norm_r, st->norm_r0);
    c.hist_rel[k + 1] = rel;
    c.hist_tb[k + 1] = (double)globaltimer();
    st->nrec = k + 2;
    st->rows_x = rows_p;
    st->cols_x = cols_p;
    st->rows_p = rows_q;
    st->cols_p = cols_q;
    st->k = k + 1;
    if (norm_r <= __dmul_rn(st->norm_r0, c.eps)) {
      st->status = CONVERGED;
      return;
    }
    st->beta = __ddiv_rn(rho_next, st->rho);
    st->rho = rho_next;
    if (st->k >= c.max_iter) st->status = MAXITER;
  }
}

// =====================================================================
// launchers
// =====================================================================
// standalone SpMM for parity tests (row-interleaved x, y)
template <int S>
__global__ void k_spmm_plain(const int32_t* rp, const int32_t* ci, const double* val,
                             const double* x, double* y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc[S];
#pragma unroll
    for (int u = 0; u < S; ++u) acc[u] = 0.0;
    for (int32_t kk = rp[i]; kk < rp[i + 1]; ++kk) {
      const int64_t col = ci[kk];
      const double v = val[kk];
#pragma unroll
      for (int u = 0; u < S; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(v, x[col * S + u]));
    }
#pragma unroll
    for (int u = 0; u < S; ++u) y[i * S + u] = acc[u];
  }
}

static int rows_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}
static void dims(const SolveConst& c, int64_t& nmax, int64_t& cmax) {
  nmax = 0;
  cmax = 0;
  for (int s = 0; s < c.nsides; ++s) {
    nmax = c.side[s].n > nmax ? c.side[s].n : nmax;
    cmax = c.side[s].ncta > cmax ? c.side[s].ncta : cmax;
  }
}

// Per-S launchers (explicitly instantiated, one translation unit per S).
#ifdef SK_INST_COMMON
template <int S>
struct Launch {
  static void init(const SolveConst& c, const double* dc1, const double* dc2, cudaStream_t st);
  static void spmm(const SolveConst& c, cudaStream_t st);
  static void gram_lanczos(const SolveConst& c, cudaStream_t st);
  static void rare(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st);
  static void pass2(const SolveConst& c, cudaStream_t st);
  static void cg_a(const SolveConst& c, int64_t rmax, cudaStream_t st);
  static void cg_b(const SolveConst& c, int64_t rmax, cudaStream_t st);
  static void spmm_plain(const int32_t* rp, const int32_t* ci, const double* val, const double* x,
                         double* y, int64_t n, cudaStream_t st);
};
#else
template <int S>
struct Launch {
  static void init(const SolveConst& c, const double* dc1, const double* dc2, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    dim3 g1(rows_grid(nmax), c.nsides);
    k_init_transpose<S><<<g1, 256, 0, st>>>(c, dc1, dc2);
    dim3 g2((unsigned)cmax, 1, c.nsides);
    k_init_gram<S><<<g2, 256, 0, st>>>(c);
    k_init_householder<S><<<c.nsides, 1024, 0, st>>>(c);
    k_init_write<S><<<g1, 256, 0, st>>>(c);
  }
  static void spmm(const SolveConst& c, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    dim3 g1(rows_grid(nmax), c.nsides);
    k_spmm<S><<<g1, 256, 0, st>>>(c);
  }
  static void gram_lanczos(const SolveConst& c, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    dim3 gg((unsigned)cmax, 3, c.nsides);
    k_gram<S><<<gg, 256, 0, st>>>(c, (int)GM_LANCZOS1);
  }
  static void rare(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    dim3 gu((unsigned)cmax, 1, c.nsides);
    k_update<S><<<gu, 256, 0, st>>>(c, (int)UM_MAT);
    k_mat_transition<<<1, 32, 0, st>>>(c);
    k_householder<S><<<c.nsides, 1024, 0, st>>>(c, 0);
    dim3 gc((unsigned)cmax, (unsigned)(kmax_blocks > 0 ? kmax_blocks : 1), c.nsides);
    k_gram<S><<<gc, 256, 0, st>>>(c, (int)GM_CLEAN);
    k_update<S><<<gu, 256, 0, st>>>(c, (int)UM_CLEAN);
    k_householder<S><<<c.nsides, 1024, 0, st>>>(c, 1);
  }
  static void pass2(const SolveConst& c, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    dim3 g1(rows_grid(nmax), c.nsides);
    k_pass2<S><<<g1, 256, 0, st>>>(c);
  }
  static void cg_a(const SolveConst& c, int64_t rmax, cudaStream_t st) {
    const unsigned nt = (unsigned)((rmax + kTile - 1) / kTile);
    k_cg_a<S><<<dim3(nt, nt), 256, 0, st>>>(c);
  }
  static void cg_b(const SolveConst& c, int64_t rmax, cudaStream_t st) {
    const unsigned nt = (unsigned)((rmax + kTile - 1) / kTile);
    k_cg_b<S><<<dim3(nt, nt), 256, 0, st>>>(c);
  }
  static void spmm_plain(const int32_t* rp, const int32_t* ci, const double* val, const double* x,
                         double* y, int64_t n, cudaStream_t st) {
    k_spmm_plain<S><<<rows_grid(n), 256, 0, st>>>(rp, ci, val, x, y, n);
  }
};

#endif  // SK_INST_COMMON

#ifdef SK_INST_S
template struct Launch<SK_INST_S>;
#endif

#ifdef SK_INST_COMMON
static int g_launches = 0;
int launch_count() { return g_launches; }
void launch_count_reset() { g_launches = 0; }

#define SK_DISPATCH_S(s, CALL)                  \
  switch (s) {                                  \
    case 1: Launch<1>::CALL; break;             \
    case 2: Launch<2>::CALL; break;             \
    case 3: Launch<3>::CALL; break;             \
    case 4: Launch<4>::CALL; break;             \
    case 5: Launch<5>::CALL; break;             \
    case 6: Launch<6>::CALL; break;             \
    case 7: Launch<7>::CALL; break;             \
    case 8: Launch<8>::CALL; break;             \
    default: break;                             \
  }

void launch_init(const SolveConst& c, const double* dc1, const double* dc2, cudaStream_t st) {
  SK_DISPATCH_S(c.s, init(c, dc1, dc2, st));
  k_core_init<<<1, 32, 0, st>>>(c);
  g_launches += 5;
}
void launch_spmm(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, spmm(c, st));
  g_launches += 1;
}
void launch_gram_lanczos(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, gram_lanczos(c, st));
  g_launches += 1;
}
void launch_rare(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st) {
  SK_DISPATCH_S(c.s, rare(c, kmax_blocks, st));
  g_launches += 6;
}
void launch_pass2(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, pass2(c, st));
  g_launches += 1;
}
void launch_cg_a(const SolveConst& c, int64_t rmax, cudaStream_t st) {
  SK_DISPATCH_S(c.s, cg_a(c, rmax, st));
  g_launches += 1;
}
void launch_cg_b(const SolveConst& c, int64_t rmax, cudaStream_t st) {
  SK_DISPATCH_S(c.s, cg_b(c, rmax, st));
  g_launches += 1;
}
void launch_spmm_plain(int s, const int32_t* rp, const int32_t* ci, const double* val,
                       const double* x, double* y, int64_t n, cudaStream_t st) {
  SK_DISPATCH_S(s, spmm_plain(rp, ci, val, x, y, n, st));
  g_launches += 1;
}

__global__ void k_block_to_colmajor(const double* blk, double* out, int64_t n, int s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int u = 0; u < s; ++u) out[u * n + i] = blk[i * s + u];
}
void launch_block_to_colmajor(const double* blk, double* out, int64_t n, int s, cudaStream_t st) {
  k_block_to_colmajor<<<rows_grid(n), 256, 0, st>>>(blk, out, n, s);
}
__global__ void k_colmajor_to_block(const double* in, double* blk, int64_t n, int s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int u = 0; u < s; ++u) blk[i * s + u] = in[u * n + i];
}
void launch_colmajor_to_block(const double* in, double* blk, int64_t n, int s, cudaStream_t st) {
  k_colmajor_to_block<<<rows_grid(n), 256, 0, st>>>(in, blk, n, s);
}
#endif

}  // namespace sk
