// sk_kernels.cu -- sm_100a kernels of the factorized-Krylov hot path.
//
// Basis blocks are stored UNNORMALISED (U_b, row-interleaved n x s) together
// with their triangular factor N_b and 1/diag(N_b); every reader forms the
// orthonormal row v_b(i,:) = U_b(i,:) N_b^{-1} on the fly (forward substitution
// with the reciprocal diagonal). The candidate of each extension is written
// straight into the next block's storage, so an extension needs no separate
// normalisation pass:
//
//  K1  k_spmm<S>       w = op * V_last (CSR gather in stored order, mul+add)
//  K2  k_gram<S>       R1 Gram coefficients V_b^T x, last-CTA trees (fixed order)
//      k_update<S>     x_out = x_in - sum_b V_b c_b, + R1 Gram of x_out, finalise
//                      (Cholesky, sigma extremes, classification, H column)
//      k_householder   rare path: single-CTA Householder QR (exact classification)
//  K4  k_cg_a/k_cg_b   fused CG core updates (P = R + beta P; Q = H P + P G^T on the
//                      fly from the Lanczos bands; <R,Q>; X += alpha P; R -= alpha Q;
//                      ||R||^2) with R2 tile trees
//
// Reference ops restated (proj/src): sparse_matrix.cpp:142-200 (SpMM),
// block_krylov.cpp:27-145 (init / extension), :173-213 (banded products),
// factorized_solvers.cpp:121-192 (CG loop), decompositions.cpp:16-78 (QR).
#include "sk_device.cuh"
#include "sk_launch.h"

#include <cstdlib>
#include <cstdio>

namespace sk {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// =====================================================================
// On-the-fly normalisation of basis rows
// =====================================================================
template <int S>
struct NF {
  double N[S * S];
  double d[S];
};
template <int S>
__device__ __forceinline__ void load_nf(const double* nfac, int64_t b, NF<S>& f) {
  const double* p = nfac + b * (S * S + S);
#pragma unroll
  for (int e = 0; e < S * S; ++e) f.N[e] = __ldg(p + e);
#pragma unroll
  for (int u = 0; u < S; ++u) f.d[u] = __ldg(p + S * S + u);
}
template <int S>
__device__ __forceinline__ void norm_row(const double* u, const NF<S>& f, double* q) {
#pragma unroll
  for (int c = 0; c < S; ++c) {
    double acc = u[c];
#pragma unroll
    for (int t = 0; t < c; ++t) acc = __dsub_rn(acc, __dmul_rn(q[t], f.N[c * S + t]));
    q[c] = __dmul_rn(acc, f.d[c]);
  }
}
template <int S>
__device__ __forceinline__ void load_vrow(const double* blk, const NF<S>& f, int64_t i, double* q) {
  double u[S];
#pragma unroll
  for (int t = 0; t < S; ++t) u[t] = __ldg(blk + i * S + t);
  norm_row<S>(u, f, q);
}

// =====================================================================
// Single-thread finalisation logic (mirrors oracle sk_basis_try_extend)
// =====================================================================
__device__ inline int64_t first_block(const SolveConst& c, int64_t k) {
  return c.arnoldi ? 0 : (k - 2 > 0 ? k - 2 : 0);
}
__device__ inline double* hb_ptr(const SideConst& sc, int64_t e, int d, int s) {
  return sc.hband + (e * 3 + d) * (int64_t)(s * s);
}
// Arnoldi H: dense column-major with leading dimension hld (zero-initialised,
// so the structural zeros below the block Hessenberg band read as 0.0)
__device__ inline double* hcol_ptr(const SideConst& sc, int64_t e, int cc, int s) {
  return sc.hband + (e * s + cc) * sc.hld;
}

// coeff2 (block_krylov.cpp:105-108): Lanczos in the reference loop order; Arnoldi
// as the canonical tree over per-block sums hsq[b] (written by the Gram pass).
// cc (optional): shared-memory copy of the coefficient blocks k-2, k-1 (s*s each)
__device__ inline double coeff2_of(const SolveConst& c, int side, int64_t k, int64_t e, const double* cc) {
  const SideConst& sc = c.side[side];
  const int s = c.s, ss = s * s;
  if (c.arnoldi) {
    TreeStream ts;
    ts.init();
    for (int64_t jb = 0; jb < k; ++jb) ts.push(__ldcg(sc.hsq + jb));
    return ts.finish();
  }
  double acc = 0.0;
  for (int64_t jb = first_block(c, k); jb < k; ++jb)
    for (int col = 0; col < s; ++col)
      for (int r = 0; r < s; ++r) {
        const double h = cc ? cc[(jb - (k - 2)) * ss + col * s + r] : __ldcg(sc.coef + jb * ss + col * s + r);
        acc = __dadd_rn(acc, __dmul_rn(h, h));
      }
  (void)e;
  return acc;
}
// block-parallel canonical tree over a[0..count) (all threads; result to all)
static __device__ double block_tree(const double* a, int64_t count, double* sbuf /* >= 1024 */) {
  // level 1: aligned groups of 8 per thread, then a stream over the group nodes
  __shared__ double res;
  const int64_t ng = (count + 7) / 8;
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
    double v[8];
    const int cnt = (int)mn64(8, count - 8 * g);
    for (int j = 0; j < cnt; ++j) v[j] = __ldcg(a + 8 * g + j);
    double node = tree_reduce_local(v, cnt);
    if (ng <= 1024) sbuf[g] = node;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ng <= 1024) {
      TreeStream ts;
      ts.init();
      for (int64_t g = 0; g < ng; ++g) ts.push(sbuf[g]);
      res = ts.finish();
    } else {
      TreeStream ts;
      ts.init();
      for (int64_t j = 0; j < count; ++j) ts.push(__ldcg(a + j));
      res = ts.finish();
    }
  }
  __syncthreads();
  return res;
}
__device__ inline void set_nfac(const SideConst& sc, int64_t b, int s, const double* N, bool identity) {
  double* p = sc.nfac + b * (s * s + s);
  for (int e = 0; e < s * s; ++e) p[e] = identity ? ((e % (s + 1)) == 0 ? 1.0 : 0.0) : N[e];
  for (int u = 0; u < s; ++u) p[s * s + u] = __ddiv_rn(1.0, identity ? 1.0 : N[u * s + u]);
}

// c = N^{-T} G and M = N^{-1} c (oracle tri_ntinv / tri_ninv), N with 1/diag in nfac
__device__ inline void block_coefs(const double* nf, const double* G, int s, double* c, double* M) {
  const double* N = nf;
  const double* dinv = nf + s * s;
  for (int u = 0; u < s; ++u)
    for (int t = 0; t < s; ++t) {
      double acc = G[u * s + t];
      for (int r = 0; r < t; ++r) acc = __dsub_rn(acc, __dmul_rn(N[t * s + r], c[u * s + r]));
      c[u * s + t] = __dmul_rn(acc, dinv[t]);
    }
  for (int u = 0; u < s; ++u)
    for (int t = s - 1; t >= 0; --t) {
      double acc = c[u * s + t];
      for (int r = t + 1; r < s; ++r) acc = __dsub_rn(acc, __dmul_rn(N[r * s + t], M[u * s + r]));
      M[u * s + t] = __dmul_rn(acc, dinv[t]);
    }
}

__device__ inline void commit_grow(const SolveConst& c, int side, int grow_stage, SideState& st, const double* cc) {
  const SideConst& sc = c.side[side];
  const int s = c.s, ss = s * s;
  const int64_t k = st.blocks, e = st.steps;
  if (!c.arnoldi) {
    double* h0 = hb_ptr(sc, e, 0, s);
    double* h1 = hb_ptr(sc, e, 1, s);
    double* h2 = hb_ptr(sc, e, 2, s);
    for (int x = 0; x < ss; ++x) {
      h0[x] = (k >= 2) ? (cc ? cc[x] : __ldcg(sc.coef + (k - 2) * ss + x)) : 0.0;
      h1[x] = cc ? cc[ss + x] : __ldcg(sc.coef + (k - 1) * ss + x);
      h2[x] = st.R[x];
    }
  } else {
    for (int cc = 0; cc < s; ++cc)
      for (int r = 0; r < s; ++r) hcol_ptr(sc, e, cc, s)[k * s + r] = st.R[cc * s + r];
  }
  set_nfac(sc, k, s, st.R, grow_stage == ST_GROW_HH);
  st.hfro2 = __dadd_rn(__dadd_rn(st.hfro2, st.coeff2), st.r2);
  st.steps = e + 1;
  st.blocks = k + 1;
  st.stage = grow_stage;
}
__device__ inline void commit_exhausted(const SolveConst& c, int side, SideState& st, const double* cc) {
  const SideConst& sc = c.side[side];
  const int s = c.s, ss = s * s;
  const int64_t k = st.blocks, e = st.steps;
  if (!c.arnoldi) {
    double* h0 = hb_ptr(sc, e, 0, s);
    double* h1 = hb_ptr(sc, e, 1, s);
    double* h2 = hb_ptr(sc, e, 2, s);
    for (int x = 0; x < ss; ++x) {
      h0[x] = (k >= 2) ? (cc ? cc[x] : __ldcg(sc.coef + (k - 2) * ss + x)) : 0.0;
      h1[x] = cc ? cc[ss + x] : __ldcg(sc.coef + (k - 1) * ss + x);
      h2[x] = 0.0;
    }
  } else {
    for (int cc = 0; cc < s; ++cc)
      for (int r = 0; r < s; ++r) hcol_ptr(sc, e, cc, s)[k * s + r] = 0.0;
  }
  st.hfro2 = __dadd_rn(st.hfro2, st.coeff2);
  st.steps = e + 1;
  st.exhausted = 1;
  st.stage = ST_DONE_NOGROW;
}

// classification (block_krylov.cpp:105-137)
__device__ inline void classify(const SolveConst& c, int side, bool first_pass, int grow_stage, SideState& st,
                                const double* cc = nullptr) {
  const int s = c.s, ss = s * s;
  if (first_pass) {
    if (!(c.arnoldi && st.pad == 1)) st.coeff2 = coeff2_of(c, side, st.blocks, st.steps, cc);
    st.pad = 0;
    double r2 = 0.0;
    for (int x = 0; x < ss; ++x) r2 = __dadd_rn(r2, __dmul_rn(st.R[x], st.R[x]));
    st.r2 = r2;
    st.scale = __dsqrt_rn(__dadd_rn(__dadd_rn(st.hfro2, st.coeff2), st.r2));
    if (!c.arnoldi && st.smin < __dmul_rn(c.tol, st.scale)) {
      st.stage = ST_NEED_CLEANUP;
      return;
    }
  }
  const double lim = __dmul_rn(c.tol, st.scale);
  if (st.smax <= lim || st.scale == 0.0) {
    commit_exhausted(c, side, st, cc);
    return;
  }
  if (st.smin < lim) {
    st.broken = 1;
    st.stage = ST_DONE_NOGROW;
    return;
  }
  commit_grow(c, side, grow_stage, st, cc);
}

// after the direct Gram (gbase) of the candidate in U_k
#ifdef SK_CS_PROF
__device__ long long g_fdprof[4];
#endif
__device__ inline void finalize_direct(const SolveConst& c, int side, bool first_pass, SideState& st,
                                       const double* cc = nullptr) {
  const int s = c.s;
#ifdef SK_CS_PROF
  const long long f0 = clock64();
#endif
  bool ok = cholesky_upper(st.gbase, s, st.R);
#ifdef SK_CS_PROF
  const long long f1 = clock64();
#endif
  if (ok) {
    jacobi_extremes(st.R, s, s, &st.smax, &st.smin);
    if (st.smin < __dmul_rn(kHHRatio, st.smax)) ok = false;
  }
#ifdef SK_CS_PROF
  g_fdprof[0] = f1 - f0;
  g_fdprof[1] = clock64() - f1;
#endif
  if (!ok) {
    st.stage = first_pass ? ST_NEED_HH : ST_NEED_HH2;
    return;
  }
  if (first_pass) st.paths[0]++;
  classify(c, side, first_pass, ST_GROW_DIRECT, st, cc);
}
__device__ inline void finalize_init(const SolveConst& c, int side, SideState& st) {
  const int s = c.s;
  bool ok = cholesky_upper(st.gbase, s, st.R);
  if (ok) {
    jacobi_extremes(st.R, s, s, &st.smax, &st.smin);
    if (st.smin < __dmul_rn(kHHRatio, st.smax)) ok = false;
  }
  if (ok) {
    set_nfac(c.side[side], 0, s, st.R, false);
    st.stage = ST_INIT_DIRECT;
    st.paths[0]++;
  } else {
    st.stage = ST_INIT_HH;
    st.paths[1]++;
  }
}

// =====================================================================
// R1 machinery: per-CTA aligned subtree over 32 segments
// =====================================================================
template <int NE>
struct OwnerVals {
  static constexpr int J = (NE + 31) / 32;
  double v[J > 0 ? J : 1];
};
template <int NE>
__device__ __forceinline__ void seg_butterfly(const double* acc, OwnerVals<NE>& out, int lane) {
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double v = butterfly(acc[e]);
    if ((e & 31) == lane) out.v[e >> 5] = v;
  }
}
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
struct SegGeom {
  int64_t seg_w0;
  int nvalid_cta, nvalid_warp;
};
__device__ __forceinline__ SegGeom seg_geom(int64_t cta, int64_t nseg) {
  SegGeom g;
  const int warp = threadIdx.x >> 5;
  const int64_t seg_cta0 = cta * kSegsPerCta;
  g.nvalid_cta = (int)mn64(kSegsPerCta, nseg - seg_cta0);
  g.seg_w0 = seg_cta0 + warp * kSegsPerWarp;
  g.nvalid_warp = (int)mx64(0, mn64(kSegsPerWarp, nseg - g.seg_w0));
  return g;
}
__device__ __forceinline__ void unpack_tri(int e, int& t, int& u) {
  u = 0;
  t = e;
  while (t > u) {
    t -= u + 1;
    ++u;
  }
}

// =====================================================================
// One row of w = op * V (normalised on the fly): CSR gather or matrix-free
// stencil. Both accumulate the row's terms in ascending column order with
// mul+add (sparse_matrix.cpp:151-155), so the stencil form is bitwise the CSR.
// =====================================================================
template <int S>
__device__ __forceinline__ void grid_coords(const SideConst& sc, int64_t i, int64_t& a, int64_t& b,
                                            int64_t& cz) {
  // 2D: a = ix, b = iy; 3D: a = ix, b = iy, cz = iz
  const int64_t g = sc.sg;
  if (sc.sg_pow2 >= 0) {
    const int sh = sc.sg_pow2;
    a = i & (g - 1);
    const int64_t r = i >> sh;
    if (sc.sdim == 2) {
      b = r;
      cz = 0;
    } else {
      b = r & (g - 1);
      cz = r >> sh;
    }
  } else {
    a = i % g;
    const int64_t r = i / g;
    if (sc.sdim == 2) {
      b = r;
      cz = 0;
    } else {
      b = r % g;
      cz = r / g;
    }
  }
}
// raw row of op * U (no normalisation): CSR gather or stencil, ascending columns
template <int S>
__device__ __forceinline__ void raw_row_csr(const SideConst& sc, const double* __restrict__ x, int64_t i,
                                            double* acc, double* own) {
#pragma unroll
  for (int u = 0; u < S; ++u) acc[u] = 0.0;
  const int32_t k0 = __ldg(sc.rp + i), k1 = __ldg(sc.rp + i + 1);
  for (int32_t kk = k0; kk < k1; ++kk) {
    const double v = __ldg(sc.val + kk);
    const int64_t col = __ldg(sc.ci + kk);
#pragma unroll
    for (int u = 0; u < S; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(v, __ldg(x + col * S + u)));
  }
#pragma unroll
  for (int u = 0; u < S; ++u) own[u] = __ldg(x + i * S + u);
}

// =====================================================================
// Raw-block arithmetic contract: the basis is stored as raw
// blocks U_b with triangular factors N_b (V_b = U_b N_b^{-1}). Per row, only the
// operator output is normalised: w = (op U_{k-1}) N_{k-1}^{-1}. Gram sums run on
// raw blocks, G_b = U_b^T x (R1), then c_b = N_b^{-T} G_b and M_b = N_b^{-1} c_b
// are formed once per block; updates are x - sum_b U_b M_b.
// =====================================================================
enum UpdMode : int { UM_LANCZOS = 0, UM_FIRST = 1, UM_SECOND = 2, UM_CLEAN = 3, UM_INIT = 4 };

template <int S>
__device__ __forceinline__ void ld_raw(const double* __restrict__ x, int64_t i, double* u) {
  if constexpr (S % 2 == 0) {
    const double2* p = reinterpret_cast<const double2*>(x + i * S);
#pragma unroll
    for (int h = 0; h < S / 2; ++h) {
      const double2 v = __ldg(p + h);
      u[2 * h] = v.x;
      u[2 * h + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) u[t] = __ldg(x + i * S + t);
  }
}
template <int S>
__device__ __forceinline__ void ld_raw_cg(const double* __restrict__ x, int64_t i, double* u) {
  if constexpr (S % 2 == 0) {
    const double2* p = reinterpret_cast<const double2*>(x + i * S);
#pragma unroll
    for (int h = 0; h < S / 2; ++h) {
      const double2 v = __ldcg(p + h);
      u[2 * h] = v.x;
      u[2 * h + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) u[t] = __ldcg(x + i * S + t);
  }
}
template <int S>
__device__ __forceinline__ void st_row(double* __restrict__ x, int64_t i, const double* y) {
  if constexpr (S % 2 == 0) {
    double2* p = reinterpret_cast<double2*>(x + i * S);
#pragma unroll
    for (int h = 0; h < S / 2; ++h) p[h] = make_double2(y[2 * h], y[2 * h + 1]);
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) x[i * S + t] = y[t];
  }
}

// Matrix-free stencil row of op * U (raw), 32-bit index arithmetic (device
// n < 2^31). An absent neighbour is not loaded: its operand is +0.0, so its
// term v*0 = +-0 leaves the running sum unchanged (the sum starts at +0.0 and
// never becomes -0.0) -- bitwise the CSR gather that skips it, given finite
// coefficients (enforced by the host-side detection).
template <int S, int DIM, bool POW2 = false, bool CGL = false>
__device__ __forceinline__ void stencil_row(const SideConst& sc, const double* __restrict__ x, int64_t i64,
                                            double* acc, double* own) {
  constexpr int K = DIM == 2 ? 5 : 7;
  constexpr int C = DIM == 2 ? 2 : 3;
  const int i = (int)i64;              // local row (addressing; halo rows at i < 0, i >= n)
  const int gi = i + (int)sc.row0;     // global row (grid coordinates)
  const int g = (int)sc.sg;
  int ix, iy, iz = 0;
  if (POW2) {
    const int sh = sc.sg_pow2;
    ix = gi & (g - 1);
    if (DIM == 2) {
      iy = gi >> sh;
    } else {
      iy = (gi >> sh) & (g - 1);
      iz = gi >> (2 * sh);
    }
  } else {
    const int r = gi / g;
    ix = gi - r * g;
    if (DIM == 2) {
      iy = r;
    } else {
      iz = r / g;
      iy = r - iz * g;
    }
  }
  bool pr[K];
  int col[K];
  if (DIM == 2) {
    pr[0] = iy > 0; col[0] = i - g;
    pr[1] = ix > 0; col[1] = i - 1;
    pr[2] = true;   col[2] = i;
    pr[3] = ix < g - 1; col[3] = i + 1;
    pr[4] = iy < g - 1; col[4] = i + g;
  } else {
    const int g2 = g * g;
    pr[0] = iz > 0; col[0] = i - g2;
    pr[1] = iy > 0; col[1] = i - g;
    pr[2] = ix > 0; col[2] = i - 1;
    pr[3] = true;   col[3] = i;
    pr[4] = ix < g - 1; col[4] = i + 1;
    pr[5] = iy < g - 1; col[5] = i + g;
    pr[6] = iz < g - 1; col[6] = i + g2;
  }
  double u[K][S];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (pr[k]) {
      if (CGL)
        ld_raw_cg<S>(x, col[k], u[k]);  // written earlier in the same launch (wavefront pass)
      else
        ld_raw<S>(x, col[k], u[k]);
    } else {
#pragma unroll
      for (int t = 0; t < S; ++t) u[k][t] = 0.0;
    }
  }
#pragma unroll
  for (int t = 0; t < S; ++t) {
    own[t] = u[C][t];
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) a = __dadd_rn(a, __dmul_rn(sc.scoef[k], u[k][t]));
    acc[t] = a;
  }
}

// w row (normalised) and the raw own row of U_{k-1}. MODE: 0 CSR, 2/3 stencil
// (general grid edge), 12/13 stencil with a power-of-two grid edge.
template <int S, int MODE, bool CGL = false>
__device__ __forceinline__ void z_row(const SideConst& sc, const double* __restrict__ x, int64_t i, double* z,
                                      double* own) {
  if constexpr (MODE == 2 || MODE == 3)
    stencil_row<S, MODE, false, CGL>(sc, x, i, z, own);
  else if constexpr (MODE == 12 || MODE == 13)
    stencil_row<S, MODE - 10, true, CGL>(sc, x, i, z, own);
  else
    raw_row_csr<S>(sc, x, i, z, own);
}
template <int S, int MODE>
__device__ __forceinline__ void w_row(const SideConst& sc, const double* __restrict__ x, const NF<S>& f,
                                      int64_t i, double* w, double* own) {
  double acc[S];
  z_row<S, MODE>(sc, x, i, acc, own);
  norm_row<S>(acc, f, w);
}
__device__ __forceinline__ int row_mode(const SideConst& sc) {
  if (sc.sdim == 0) return 0;
  return sc.sdim + (sc.sg_pow2 >= 0 ? 10 : 0);
}

// =====================================================================
// K1: SpMM  w = (op U_{k-1}) N^{-1}   (sparse_matrix.cpp:142-158, order kept)
// =====================================================================
template <int S>
__global__ void __launch_bounds__(256) k_spmm(const __grid_constant__ SolveConst c) {
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.exhausted || ss.broken) return;
  const SideConst& sc = c.side[side];
  const int64_t kl = ss.blocks - 1;
  const double* __restrict__ x = sc.blocks[kl];
  NF<S> f;
  load_nf<S>(sc.nfac, kl, f);
  const int64_t n = sc.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double z[S], y[S], own[S];
    switch (row_mode(sc)) {
      case 2: z_row<S, 2>(sc, x, i, z, own); break;
      case 3: z_row<S, 3>(sc, x, i, z, own); break;
      case 12: z_row<S, 12>(sc, x, i, z, own); break;
      case 13: z_row<S, 13>(sc, x, i, z, own); break;
      default: z_row<S, 0>(sc, x, i, z, own); break;
    }
    norm_row<S>(z, f, y);
    st_row<S>(sc.w, i, y);
    if (!c.arnoldi) st_row<S>(sc.wx, i, z);  // Lanczos Grams are raw
  }
}

// =====================================================================
// Canonical-tree helpers for one-warp-per-segment kernels
// =====================================================================
__device__ __forceinline__ double tree32(double* a) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) a[i] = __dadd_rn(a[2 * i], a[2 * i + 1]);
  return a[0];
}
// Canonical tree over P CTA partials part[p*NE + e] for every e (last CTA):
// levels of aligned groups of 32 (a tree over 32 = four aligned trees of 8),
// intermediate nodes in global scratch (>= 2 * ceil(P/32) * NE doubles), the
// last <= 32 nodes reduced per e. Aligned power-of-two groups compose, so this
// is the canonical tree for any P.
template <int NE>
__device__ __noinline__ void final_tree(const double* part, int64_t P, double* out, double* scratch) {
  const double* src = part;
  int64_t cnt = P;
  double* dst = scratch;
  double* other = scratch + ((P + 31) / 32) * NE;
  while (cnt > 32) {
    const int64_t ngroups = (cnt + 31) / 32;
    for (int64_t idx = threadIdx.x; idx < NE * ngroups; idx += blockDim.x) {
      const int e = (int)(idx % NE);
      const int64_t grp = idx / NE;
      const int64_t p0 = grp * 32;
      const int n32 = (int)mn64(32, cnt - p0);
      double node;
      if (n32 == 32) {
        double q4[4];
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          double a[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) a[j] = __ldcg(src + (p0 + 8 * q + j) * NE + e);
#pragma unroll
          for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
            for (int j = 0; j < w; ++j) a[j] = __dadd_rn(a[2 * j], a[2 * j + 1]);
          q4[q] = a[0];
        }
        node = __dadd_rn(__dadd_rn(q4[0], q4[1]), __dadd_rn(q4[2], q4[3]));
      } else {
        node = tree_stream(src + p0 * NE + e, n32, NE);
      }
      dst[grp * NE + e] = node;
    }
    __threadfence_block();
    __syncthreads();
    src = dst;
    cnt = ngroups;
    double* t = dst;
    dst = other;
    other = t;
  }
  for (int e = threadIdx.x; e < NE; e += blockDim.x) out[e] = tree_stream(src + e, cnt, NE);
  __syncthreads();
}
template <int NE>
__device__ __forceinline__ void warp_seg_to_cta(const double* acc, int nvalid_cta, double* part_out) {
  __shared__ double snode[kFusedSegsPerCta][NE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double v = butterfly(acc[e]);
    if (lane == (e & 31)) snode[warp][e] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    double a[kFusedSegsPerCta];
#pragma unroll
    for (int w = 0; w < kFusedSegsPerCta; ++w) a[w] = snode[w][e];
    part_out[e] = tree_reduce_local(a, nvalid_cta);
  }
}

// =====================================================================
// Row partition. Rank boundaries sit on reduction chunks: aligned
// power-of-two groups of R1 segments (>= 32), so a chunk node is a node of the
// canonical tree and the canonical tree over all ranks' chunk nodes, in global
// order, is bitwise the single-GPU root. The last CTA of a partitioned pass
// writes its chunk nodes; after the all-gather, k_dist_fin forms the root and
// runs the same finalisation as the single-GPU last CTA.
// Node (slot, side, chunk j) lives at ((slot * nsides + side) * nch_max + j) * nex.
// =====================================================================
__device__ __forceinline__ int64_t node_off(const SolveConst& c, int64_t slot, int side, int64_t j) {
  return ((slot * c.nsides + side) * c.nch_max + j) * c.nex;
}
template <int NE>
__device__ __noinline__ void dist_emit(const SolveConst& c, int side, int64_t slot, const double* part, int64_t ncta,
                          int64_t chunk, double* scratch) {
  const SideConst& sc = c.side[side];
  for (int64_t j = 0; j < sc.nch; ++j) {
    const int64_t p0 = j * chunk;
    final_tree<NE>(part + p0 * NE, mn64(chunk, ncta - p0), c.nodes + node_off(c, slot, side, j), scratch);
  }
}
// canonical tree over every rank's chunk nodes (all threads call; result in out)
template <int NE>
__device__ void dist_root(const SolveConst& c, int side, int64_t slot, int64_t msg, double* out) {
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    TreeStream ts;
    ts.init();
    for (int r = 0; r < c.world; ++r) {
      const double* base = c.gnodes + r * msg + node_off(c, slot, side, 0) + e;
      const int nr = c.rank_nch[side * c.world + r];
      for (int j = 0; j < nr; ++j) ts.push(__ldcg(base + (int64_t)j * c.nex));
    }
    out[e] = ts.finish();
  }
  __syncthreads();
}

// =====================================================================
// K2: R1 Gram G_b = U_b^T x against blocks [b0, b1); one CTA per (row group,
// block); the last CTA of each block forms c_b = N_b^{-T} G_b and M_b.
// =====================================================================
enum GramMode : int { GM_J = 0, GM_ALL_W = 1, GM_ALL_X = 2, GM_CLEAN = 3 };

template <int S>
__device__ inline bool gram_setup(const SolveConst& c, int side, int mode, const double*& x,
                                  double*& out, double*& mout, int64_t& b0, int64_t& b1) {
  const DevState* st = c.st;
  if (st->status != RUNNING) return false;
  const SideState& ss = st->side[side];
  const SideConst& sc = c.side[side];
  const int64_t k = ss.blocks;
  if (mode == GM_CLEAN) {
    if (ss.stage != ST_NEED_CLEANUP) return false;
    x = sc.blocks[k];
    out = sc.coef2;
    mout = sc.mcoef2;
    b0 = 0;
    b1 = k;
    return true;
  }
  if (ss.exhausted || ss.broken) return false;
  switch (mode) {
    case GM_J:
      x = c.arnoldi ? sc.w : sc.wx;  // Lanczos: raw z = op U_{k-1} (k_spmm)
      out = sc.coef;
      mout = sc.mcoef;
      b0 = first_block(c, k);
      b1 = k;
      return true;
    case GM_ALL_W:
      x = sc.w;
      out = sc.coef;
      mout = sc.mcoef;
      b0 = 0;
      b1 = k;
      return true;
    case GM_ALL_X:
      x = sc.wx;
      out = sc.coef2;
      mout = sc.mcoef2;
      b0 = 0;
      b1 = k;
      return true;
  }
  return false;
}

// Output halves per block: for S = 8 the 64 accumulators plus four rows of
// operands in flight took 254 registers (8 warps per SM, 2.3 TB/s at config 4);
// two CTAs per (block, row range), each owning half of the u index (32
// accumulators, two rows in flight, 2 CTAs per SM), adjacent in launch order so
// the second read of U_b's rows hits L2. Every entry keeps its R1 order.
template <int S>
struct GramSplit {
  static constexpr int H = S >= 8 ? 2 : 1;
  static constexpr int UNR = H == 2 ? 2 : 4;
  static constexpr int MINB = H == 2 ? 2 : (S <= 4 ? 3 : 1);  // CTAs per SM (register budget)
};
#ifndef SK_GRAM_RING
#define SK_GRAM_RING 0  // cp.async row rings, per-lane rows (20.2 s at config 4) and coalesced pieces (17.4 s), against 17.0 s: LDGSTS costs the L1TEX pipe on both sides
#endif
#ifndef SK_GRAM_STAGES
#define SK_GRAM_STAGES 3
#endif
constexpr int kGramStages = SK_GRAM_STAGES;
// Shared-memory row ring of k_gram (even S: rows are whole 16-byte units). ncu (profiles/r2):
// k_gram<8> ran with the L1TEX pipe 92% busy and DRAM 30%, L2 31%, FP64 29% -- a lane reading
// its own 64-byte row makes every LDG.128 of the warp touch 16 cache lines for 512 useful bytes.
// Here the warp copies the 32 consecutive rows of a step as CONTIGUOUS 16-byte pieces (cp.async,
// lane l takes pieces l, l + 32, ...: four fully used lines per instruction) into a per-warp
// ring whose rows are padded to an odd number of 16-byte units, so the lane's own row then
// comes out of shared memory conflict-free.
template <int S>
struct GramRing {
  static constexpr bool ON = (S % 2 == 0);
  static constexpr int SU = S / GramSplit<S>::H;
  static constexpr int UA = S / 2, UY = SU / 2;      // 16-byte units per row of U_b / of x's half
  static constexpr int PA = UA | 1, PY = UY | 1;     // padded row strides (units)
  static constexpr int STAGE = 32 * (PA + PY) * 2;   // doubles per warp and stage
  static constexpr size_t BYTES = ON ? sizeof(double) * (size_t)8 * kGramStages * STAGE : 0;
};
#ifndef SK_GRAM_NOINLINE
#define SK_GRAM_NOINLINE 1
#endif
#ifndef SK_GRAM_XPOSE
#define SK_GRAM_XPOSE 1  // s = 4, 8: coalesced loads with transposed accumulator ownership
#endif
// One R1 segment of the Arnoldi Gram (rows base + lane + 32 m, m = 0 .. 15, of U_b against x,
// output half h) as a separately compiled function: inside k_gram ptxas sank the loads of every
// row to their first use (one row in flight per warp, long-scoreboard bound at 0.38 of HBM);
// here rows are register double-buffered explicitly, two ahead of the accumulation. Returns the
// lane's owner values of the xor butterflies (entry e lives in lane e & 31).
template <int S>
__device__ __noinline__ OwnerVals<(S / GramSplit<S>::H) * S> gram_segment(const double* __restrict__ ub,
                                                                        const double* __restrict__ x, int64_t base,
                                                                        int64_t n, int h, int lane) {
  constexpr int H = GramSplit<S>::H, SU = S / H, NH = SU * S;
  double acc[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) acc[e] = 0.0;
  auto load = [&](int m, double* a, double* y) {
    const int64_t i = base + lane + 32 * m;
    if (i < n) {
      ld_raw<S>(ub, i, a);
      if constexpr (H == 1) {
        ld_raw<S>(x, i, y);
      } else {
        const double2* py = reinterpret_cast<const double2*>(x + i * S + h * SU);
#pragma unroll
        for (int u = 0; u < SU / 2; ++u) {
          const double2 v = __ldg(py + u);
          y[2 * u] = v.x;
          y[2 * u + 1] = v.y;
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < S; ++t) a[t] = 0.0;
#pragma unroll
      for (int u = 0; u < SU; ++u) y[u] = 0.0;
    }
  };
  // rows past n contribute acc + 0 * 0 = acc + (+0): the sums are unchanged bit for bit
  // (acc starts at +0 and a + (+0) = a for every a, including -0 + (+0) = +0 = the skipped form
  // only if acc were -0, which a sum starting at +0 with round-to-nearest never is)
  double a0[S], y0[SU], a1[S], y1[SU];
  load(0, a0, y0);
  load(1, a1, y1);
#pragma unroll
  for (int m = 0; m < kLRows; m += 2) {
    double a2[S], y2[SU], a3[S], y3[SU];
    if (m + 2 < kLRows) {
      load(m + 2, a2, y2);
      load(m + 3, a3, y3);
    }
#pragma unroll
    for (int u = 0; u < SU; ++u)
#pragma unroll
      for (int t = 0; t < S; ++t) acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(a0[t], y0[u]));
#pragma unroll
    for (int u = 0; u < SU; ++u)
#pragma unroll
      for (int t = 0; t < S; ++t) acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(a1[t], y1[u]));
    if (m + 2 < kLRows) {
#pragma unroll
      for (int t = 0; t < S; ++t) {
        a0[t] = a2[t];
        a1[t] = a3[t];
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        y0[u] = y2[u];
        y1[u] = y3[u];
      }
    }
  }
  OwnerVals<NH> out;
  seg_butterfly<NH>(acc, out, lane);
  return out;
}
template <int S>
__global__ void __launch_bounds__(256, GramSplit<S>::MINB) k_gram(const __grid_constant__ SolveConst c, int mode) {
  constexpr int NB = S * S;
  constexpr int H = GramSplit<S>::H, SU = S / H, NH = SU * S, UNR = GramSplit<S>::UNR;
  const int side = blockIdx.z;
  if (side >= c.nsides) return;
  const double* x;
  double *out, *mout;
  int64_t b0, b1;
  if (!gram_setup<S>(c, side, mode, x, out, mout, b0, b1)) return;
  const SideConst& sc = c.side[side];
  const int64_t nblk = b1 - b0;
  // grid x runs over the blocks, y over row ranges: the CTAs that are resident
  // together share a row range, so x's rows stay in L2 across all blocks (one
  // HBM read of x per pass instead of one per block)
  const int64_t by = blockIdx.x / H;
  const int h = (int)(blockIdx.x % H);
  if (by >= nblk) return;
  const int64_t cta = blockIdx.y;
  if (cta >= sc.ncta) return;
  const int64_t b = b0 + by;
  const double* __restrict__ ub = sc.blocks[b];
  const int lane = threadIdx.x & 31;
  const int64_t n = sc.n;
  const SegGeom g = seg_geom(cta, sc.nseg);
  double* part = sc.part + ((by * sc.ncta + cta) * NB) + h * NH;  // entries u*S+t, u in this half
  OwnerVals<NH> segv[kSegsPerWarp];
#if SK_GRAM_RING
  if constexpr (GramRing<S>::ON) {
    using GR = GramRing<S>;
    constexpr int D = kGramStages, UA = GR::UA, UY = GR::UY, PA = GR::PA, PY = GR::PY;
    extern __shared__ __align__(16) double gram_ring[];
    double* wring = gram_ring + (size_t)(threadIdx.x >> 5) * D * GR::STAGE;
    const int nsteps = g.nvalid_warp * kLRows;
    auto issue = [&](int step) {
      if (step < nsteps) {
        const int64_t row0 = (g.seg_w0 + step / kLRows) * kSeg + 32 * (step % kLRows);
        double* sa = wring + (size_t)(step % D) * GR::STAGE;
        double* sy = sa + 32 * PA * 2;
#pragma unroll
        for (int j = 0; j < UA; ++j) {
          const int p_ = lane + 32 * j, rr = p_ / UA, cc = p_ % UA;
          if (row0 + rr < n)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(sa + (rr * PA + cc) * 2)),
                         "l"(ub + (row0 + rr) * S + cc * 2)
                         : "memory");
        }
#pragma unroll
        for (int j = 0; j < UY; ++j) {
          const int p_ = lane + 32 * j, rr = p_ / UY, cc = p_ % UY;
          if (row0 + rr < n)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(sy + (rr * PY + cc) * 2)),
                         "l"(x + (row0 + rr) * S + h * SU + cc * 2)
                         : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int p_ = 0; p_ < D - 1; ++p_) issue(p_);
#pragma unroll
    for (int q = 0; q < kSegsPerWarp; ++q) {
      double acc[NH];
#pragma unroll
      for (int e = 0; e < NH; ++e) acc[e] = 0.0;
      if (q < g.nvalid_warp) {
        const int64_t base = (g.seg_w0 + q) * kSeg;
#pragma unroll 2
        for (int m = 0; m < kLRows; ++m) {
          const int step = q * kLRows + m;
          // this step's pieces (copied by all lanes) have landed, and every lane is done
          // reading the stage the next issue overwrites
          asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");
          __syncwarp();
          issue(step + D - 1);
          const int64_t i = base + lane + 32 * m;
          if (i < n) {
            const double* sa = wring + (size_t)(step % D) * GR::STAGE + lane * PA * 2;
            const double* sy = wring + (size_t)(step % D) * GR::STAGE + 32 * PA * 2 + lane * PY * 2;
            double a[S], y[SU];
#pragma unroll
            for (int t = 0; t < UA; ++t) {
              const double2 v = reinterpret_cast<const double2*>(sa)[t];
              a[2 * t] = v.x;
              a[2 * t + 1] = v.y;
            }
#pragma unroll
            for (int u = 0; u < UY; ++u) {
              const double2 v = reinterpret_cast<const double2*>(sy)[u];
              y[2 * u] = v.x;
              y[2 * u + 1] = v.y;
            }
#pragma unroll
            for (int u = 0; u < SU; ++u)
#pragma unroll
              for (int t = 0; t < S; ++t)
                acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(a[t], y[u]));
          }
        }
      }
      seg_butterfly<NH>(acc, segv[q], lane);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else
#endif
  {
#pragma unroll
  for (int q = 0; q < kSegsPerWarp; ++q) {
    double acc[NH];
#pragma unroll
    for (int e = 0; e < NH; ++e) acc[e] = 0.0;
#if SK_GRAM_XPOSE
    if constexpr (S == 8 || S == 4) {
      // Transposed ownership (ncu, profiles/r2: the L1TEX pipe was 92% busy because a lane
      // reading its own row makes every LDG.128 touch 16 lines): the warp loads the step's 32
      // consecutive rows as contiguous 16-byte pieces, so lane p holds column pair c = p % UA of
      // the rows rho = p / UA + RP j (j < UA) and accumulates, for those UA logical lanes, the
      // entries (u, 2c), (u, 2c + 1). Every logical lane's sum still runs over the steps
      // m = 0 .. 15 in order; the xor butterfly over logical lanes (d = 16 .. 1) has its high
      // rounds inside the thread (IEEE addition is commutative: both partners hold the same
      // bits) and its low rounds as shuffles by d UA. Bitwise the row-per-lane form.
      constexpr int UA = S / 2, RP = 32 / UA;
      const int cpair = lane % UA, rho0 = lane / UA;
      double acc2[UA][SU][2];
#pragma unroll
      for (int j = 0; j < UA; ++j)
#pragma unroll
        for (int u = 0; u < SU; ++u) acc2[j][u][0] = acc2[j][u][1] = 0.0;
      if (q < g.nvalid_warp) {
        const int64_t base = (g.seg_w0 + q) * kSeg;
#pragma unroll 2
        for (int m = 0; m < kLRows; ++m) {
          const int64_t r0 = base + 32 * m;
          double2 av[UA];
          double yv[UA][SU];
#pragma unroll
          for (int j = 0; j < UA; ++j) {
            const int64_t i = r0 + rho0 + RP * j;
            if (i < n) {
              av[j] = __ldg(reinterpret_cast<const double2*>(ub + i * S) + cpair);
              const double2* py = reinterpret_cast<const double2*>(x + i * S + h * SU);
#pragma unroll
              for (int u = 0; u < SU / 2; ++u) {
                const double2 v = __ldg(py + u);
                yv[j][2 * u] = v.x;
                yv[j][2 * u + 1] = v.y;
              }
            } else {
              av[j] = make_double2(0.0, 0.0);
#pragma unroll
              for (int u = 0; u < SU; ++u) yv[j][u] = 0.0;
            }
          }
#pragma unroll
          for (int j = 0; j < UA; ++j)
#pragma unroll
            for (int u = 0; u < SU; ++u) {
              acc2[j][u][0] = __dadd_rn(acc2[j][u][0], __dmul_rn(av[j].x, yv[j][u]));
              acc2[j][u][1] = __dadd_rn(acc2[j][u][1], __dmul_rn(av[j].y, yv[j][u]));
            }
        }
      }
      // butterfly over the logical lanes: in-thread rounds (lane bits held by j), then shuffles
      double ent[SU][2];
#pragma unroll
      for (int u = 0; u < SU; ++u)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
          double w_[UA];
#pragma unroll
          for (int j = 0; j < UA; ++j) w_[j] = acc2[j][u][b2];
#pragma unroll
          for (int dj = UA / 2; dj >= 1; dj >>= 1)
#pragma unroll
            for (int j = 0; j < dj; ++j) w_[j] = __dadd_rn(w_[j], w_[j + dj]);
          double v = w_[0];
#pragma unroll
          for (int d = RP / 2; d >= 1; d >>= 1) v = __dadd_rn(v, shfl_xor_d(v, d * UA));
          ent[u][b2] = v;
        }
      // entry e = u S + t of this half lives in the lanes with p % UA == t / 2: hand it to lane e
      double mine = 0.0;
#pragma unroll
      for (int u = 0; u < SU; ++u)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
          const double got = __shfl_sync(0xffffffffu, ent[u][b2], (lane % S) >> 1);
          if (lane / S == u && (lane & 1) == b2) mine = got;
        }
      segv[q].v[0] = mine;
      continue;
    }
#endif
#if SK_GRAM_NOINLINE
    if (q < g.nvalid_warp) {
      segv[q] = gram_segment<S>(ub, x, (g.seg_w0 + q) * kSeg, n, h, lane);
      continue;
    }
#endif
    if (q < g.nvalid_warp) {
      const int64_t base = (g.seg_w0 + q) * kSeg;
#pragma unroll UNR
      for (int m = 0; m < kLRows; ++m) {
        const int64_t i = base + lane + 32 * m;
        if (i < n) {
          double a[S], y[SU];
          ld_raw<S>(ub, i, a);
          if constexpr (H == 1) {
            ld_raw<S>(x, i, y);
          } else {
            const double2* py = reinterpret_cast<const double2*>(x + i * S + h * SU);
#pragma unroll
            for (int u = 0; u < SU / 2; ++u) {
              const double2 v = __ldg(py + u);
              y[2 * u] = v.x;
              y[2 * u + 1] = v.y;
            }
          }
#pragma unroll
          for (int u = 0; u < SU; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t)
              acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(a[t], y[u]));
        }
      }
    }
    seg_butterfly<NH>(acc, segv[q], lane);
  }
  }
  cta_combine<NH>(segv, g.nvalid_warp, g.nvalid_cta, part);

  unsigned int* ctr = sc.counter;  // slots: 0 pass 1, 1 update, 2 clean-up, 4.. per block
  if (!last_cta_arrive(ctr + 4 + by, (unsigned)(sc.ncta * H))) return;
  __shared__ double G[NB];
  for (int e = threadIdx.x; e < NB; e += blockDim.x)
    G[e] = tree_stream(sc.part + by * sc.ncta * NB + e, sc.ncta, NB);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == GM_J && !c.arnoldi) {
      // raw Gram Gamma_b -> Gamma_b N_{k-1}^{-1}, row by row (as p1_finish)
      NF<S> fk;
      load_nf<S>(sc.nfac, c.st->side[side].blocks - 1, fk);
      for (int t = 0; t < S; ++t) {
        double row[S], q[S];
        for (int u = 0; u < S; ++u) row[u] = G[u * S + t];
        norm_row<S>(row, fk, q);
        for (int u = 0; u < S; ++u) G[u * S + t] = q[u];
      }
    }
    double cb[NB], mb[NB];
    block_coefs(sc.nfac + b * (NB + S), G, S, cb, mb);
    for (int e = 0; e < NB; ++e) {
      out[b * NB + e] = cb[e];
      mout[b * NB + e] = mb[e];
    }
    if (mode == GM_ALL_X && c.arnoldi) {
      // H column = first + second CGS pass (block_krylov.cpp:87-93); hsq[b] =
      // its sum of squares in the reference's (column, row) order
      double hsq = 0.0;
      for (int e = 0; e < NB; ++e) {
        const int t = e % S, u = e / S;
        const double h = __dadd_rn(__ldcg(sc.coef + b * NB + e), cb[e]);
        hcol_ptr(sc, c.st->side[side].steps, u, S)[b * S + t] = h;
        hsq = __dadd_rn(hsq, __dmul_rn(h, h));
      }
      sc.hsq[b] = hsq;
    }
  }
}

#ifndef SK_WAVE_WARPS
#define SK_WAVE_WARPS 32  // resident warps / SM for the wavefront pass
#endif
constexpr int kWaveBlocks = SK_WAVE_WARPS / kFusedSegsPerCta;

// =====================================================================
// Fused Lanczos passes (S <= 4). One warp per R1 segment, 8 warps per CTA
// (the CTA node is the canonical tree's level-3 node).
// =====================================================================
template <int S, int MODE, bool TWO, bool CHECK, bool CGL = false>
__device__ __forceinline__ void p1_body(const SideConst& sc, const double* __restrict__ u1, const NF<S>& f1,
                                        const double* __restrict__ u0, int64_t base, int64_t n, double* acc) {
  constexpr int NB = S * S;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int m = 0; m < kLRows; ++m) {
    const int64_t i = base + lane + 32 * m;
    if (!CHECK || i < n) {
      double y[S], a1[S], a0[S];
      z_row<S, MODE, CGL>(sc, u1, i, y, a1);  // raw z = op U_{k-1}: the Grams are raw
      if (MODE == 0) {
        double w[S];
        norm_row<S>(y, f1, w);
        st_row<S>(sc.w, i, w);
      }
      if (TWO) ld_raw<S>(u0, i, a0);
#pragma unroll
      for (int u = 0; u < S; ++u)
#pragma unroll
        for (int t = 0; t < S; ++t) {
          if (TWO) acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(a0[t], y[u]));
          acc[NB + u * S + t] = __dadd_rn(acc[NB + u * S + t], __dmul_rn(a1[t], y[u]));
        }
    }
  }
}
template <int S, int MODE>
__device__ __forceinline__ void p1_dispatch(const SideConst& sc, const double* __restrict__ u1, const NF<S>& f1,
                                            const double* __restrict__ u0, bool two, int64_t base, int64_t n,
                                            double* acc) {
  const bool full = base + kSeg <= n;
  if (two) {
    if (full) p1_body<S, MODE, true, false>(sc, u1, f1, u0, base, n, acc);
    else p1_body<S, MODE, true, true>(sc, u1, f1, u0, base, n, acc);
  } else {
    if (full) p1_body<S, MODE, false, false>(sc, u1, f1, u0, base, n, acc);
    else p1_body<S, MODE, false, true>(sc, u1, f1, u0, base, n, acc);
  }
}

// pass-1 root (raw Grams Gamma_b = U_b^T z) -> G_b = Gamma_b N_{k-1}^{-1} (each row
// of Gamma normalised like a basis row) -> c_b, M_b for blocks k-2 (if any), k-1
template <int S>
__device__ __noinline__ void p1_finish(const SideConst& sc, int64_t k, const double* res) {
  constexpr int NB = S * S, NF1 = S * S + S;
  // factors of blocks k-2, k-1 staged by all threads (block k-1's was just
  // committed by this CTA's finalisation), then two threads finish the slots
  __shared__ double nfs[2 * NF1];
#ifdef SK_CS_PROF
  const long long pp0 = clock64();
#endif
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * NF1; i += blockDim.x) {
    const int64_t b = k - 2 + i / NF1;
    nfs[i] = b >= 0 ? sc.nfac[b * NF1 + i % NF1] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    const int slot = threadIdx.x;  // 0: block k-2, 1: block k-1
    if (slot == 1 || k >= 2) {
      const int64_t b = slot == 0 ? k - 2 : k - 1;
      NF<S> fk;
      for (int e = 0; e < NB; ++e) fk.N[e] = nfs[NF1 + e];
      for (int u = 0; u < S; ++u) fk.d[u] = nfs[NF1 + NB + u];
      double G[NB];
      for (int t = 0; t < S; ++t) {
        double row[S], q[S];
        for (int u = 0; u < S; ++u) row[u] = res[slot * NB + u * S + t];
        norm_row<S>(row, fk, q);
        for (int u = 0; u < S; ++u) G[u * S + t] = q[u];
      }
      double cb[NB], mb[NB];
      block_coefs(nfs + slot * NF1, G, S, cb, mb);
      for (int e = 0; e < NB; ++e) {
        sc.coef[b * NB + e] = cb[e];
        sc.mcoef[b * NB + e] = mb[e];
      }
    }
  }
#ifdef SK_CS_PROF
  __syncthreads();
  if (threadIdx.x == 0 && (k == 101 || k == 151)) printf("P1FIN %lld cyc\n", clock64() - pp0);
#endif
}
// self-Gram root -> gbase (symmetric), then finalisation. The finalisation is a
// single-thread chain of small dependent steps (Cholesky, Jacobi, classification,
// commit); it runs on a shared-memory copy of the side state, so the chain sees
// shared-memory latency instead of a global round trip per access.
template <int S>
__device__ __noinline__ void gram_finish(const SolveConst& c, int side, const double* res, int how) {
  constexpr int NS = S * (S + 1) / 2;
  constexpr int NW = (int)(sizeof(SideState) / sizeof(unsigned long long));
  static_assert(sizeof(SideState) % sizeof(unsigned long long) == 0, "SideState is word-sized");
  __shared__ SideState sst;
  unsigned long long* gw = reinterpret_cast<unsigned long long*>(&c.st->side[side]);
  unsigned long long* sw = reinterpret_cast<unsigned long long*>(&sst);
  __shared__ double ccache[2 * S * S];  // coefficient blocks k-2, k-1 (Lanczos)
  for (int i = threadIdx.x; i < NW; i += blockDim.x) sw[i] = __ldcg(gw + i);
  {
    const int64_t k = c.st->side[side].blocks;
    const SideConst& sc = c.side[side];
    for (int i = threadIdx.x; i < 2 * S * S; i += blockDim.x) {
      const int64_t b = k - 2 + i / (S * S);
      ccache[i] = (b >= 0 && !c.arnoldi) ? __ldcg(sc.coef + b * S * S + i % (S * S)) : 0.0;
    }
  }
  __syncthreads();
  const double* cc = c.arnoldi ? nullptr : ccache;
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    int t, u;
    unpack_tri(e, t, u);
    sst.gbase[u * S + t] = res[e];
    sst.gbase[t * S + u] = res[e];
  }
  __syncthreads();
#ifdef SK_CS_PROF
  long long pq0 = clock64();
#endif
  if (threadIdx.x == 0) {
    if (how == 2) {
      finalize_init(c, side, sst);
    } else if (how == 1) {
      sst.paths[2]++;
      finalize_direct(c, side, false, sst, cc);
    } else {
      finalize_direct(c, side, true, sst, cc);
    }
  }
  __syncthreads();
#ifdef SK_CS_PROF
  long long pq1 = clock64();
#endif
  for (int i = threadIdx.x; i < NW; i += blockDim.x) gw[i] = sw[i];
  __threadfence_block();
  __syncthreads();
#ifdef SK_CS_PROF
  if (threadIdx.x == 0 && (sst.blocks == 101 || sst.blocks == 151))
    printf("GFIN side %d chain %lld cyc, copyout %lld cyc (chol %lld jacobi %lld)\n", side, pq1 - pq0, clock64() - pq1,
           g_fdprof[0], g_fdprof[1]);
#endif
}

// Lanczos pass 1: w = (op U_{k-1}) N_{k-1}^{-1}; G = U_{k-2}^T w, U_{k-1}^T w
// (block_krylov.cpp:71-84, CGS form). w is stored only for CSR operators.
template <int S, int MODE>
__global__ void __launch_bounds__(kFusedThreads, kP1Blocks) k_lanczos_p1(const __grid_constant__ SolveConst c, int side0) {
  constexpr int NB = S * S;
  constexpr int NE = 2 * NB;
  const int side = blockIdx.z + side0;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.exhausted || ss.broken) return;
  const SideConst& sc = c.side[side];
  const int64_t nseg = sc.nseg;
  const int64_t ncta = (nseg + kFusedSegsPerCta - 1) / kFusedSegsPerCta;
  const int64_t cta = blockIdx.x;
  if (cta >= ncta) return;
  const int64_t k = ss.blocks;
  const bool two = k >= 2;
  const double* __restrict__ u1 = sc.blocks[k - 1];
  const double* __restrict__ u0 = two ? sc.blocks[k - 2] : u1;
  __shared__ NF<S> f1s;
  if (threadIdx.x == 0) load_nf<S>(sc.nfac, k - 1, f1s);
  __syncthreads();
  const NF<S>& f1 = f1s;
  const int warp = threadIdx.x >> 5;
  const int64_t seg = cta * kFusedSegsPerCta + warp;
  const int nvalid_cta = (int)mn64(kFusedSegsPerCta, nseg - cta * kFusedSegsPerCta);
  double acc[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) acc[e] = 0.0;
  if (seg < nseg) p1_dispatch<S, MODE>(sc, u1, f1, u0, two, seg * kSeg, sc.n, acc);
  warp_seg_to_cta<NE>(acc, nvalid_cta, sc.part + cta * NE);
  if (!last_cta_arrive(sc.counter + 0, (unsigned)ncta)) return;
  if (sc.dist) {
    dist_emit<NE>(c, side, 0, sc.part, ncta, sc.chunk_f, sc.part + ncta * NE);
    return;
  }
  __shared__ double res[NE];
  final_tree<NE>(sc.part, ncta, res, sc.part + ncta * NE);
  p1_finish<S>(sc, k, res);
}

template <int S, int MODE, bool TWO, bool CHECK>
__device__ __forceinline__ void p2_body(const SideConst& sc, const double* __restrict__ u1, const NF<S>& f1,
                                        const double* __restrict__ u0, const double* m1, const double* m0,
                                        double* __restrict__ out, int64_t base, int64_t n, double* acc) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int m = 0; m < kLRows; ++m) {
    const int64_t i = base + lane + 32 * m;
    if (!CHECK || i < n) {
      double y[S], a1[S], a0[S];
      if (MODE == 0) {
        ld_raw_cg<S>(sc.w, i, y);
        ld_raw<S>(u1, i, a1);
      } else {
        w_row<S, MODE>(sc, u1, f1, i, y, a1);
      }
      if (TWO) {
        ld_raw<S>(u0, i, a0);
#pragma unroll
        for (int u = 0; u < S; ++u) {
          double tmp = 0.0;
#pragma unroll
          for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(a0[t], m0[u * S + t]));
          y[u] = __dsub_rn(y[u], tmp);
        }
      }
#pragma unroll
      for (int u = 0; u < S; ++u) {
        double tmp = 0.0;
#pragma unroll
        for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(a1[t], m1[u * S + t]));
        y[u] = __dsub_rn(y[u], tmp);
      }
      st_row<S>(out, i, y);
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
template <int S, int MODE>
__device__ __forceinline__ void p2_dispatch(const SideConst& sc, const double* __restrict__ u1, const NF<S>& f1,
                                            const double* __restrict__ u0, bool two, const double* m1,
                                            const double* m0, double* __restrict__ out, int64_t base, int64_t n,
                                            double* acc) {
  const bool full = base + kSeg <= n;
  if (two) {
    if (full) p2_body<S, MODE, true, false>(sc, u1, f1, u0, m1, m0, out, base, n, acc);
    else p2_body<S, MODE, true, true>(sc, u1, f1, u0, m1, m0, out, base, n, acc);
  } else {
    if (full) p2_body<S, MODE, false, false>(sc, u1, f1, u0, m1, m0, out, base, n, acc);
    else p2_body<S, MODE, false, true>(sc, u1, f1, u0, m1, m0, out, base, n, acc);
  }
}

// Lanczos pass 2: U_k = w - U_{k-2} M_{k-2} - U_{k-1} M_{k-1} (+ R1 self Gram,
// finalise). Matrix-free operators recompute w from U_{k-1} instead of reading it.
template <int S, int MODE>
__global__ void __launch_bounds__(kFusedThreads, kP2Blocks) k_lanczos_p2(const __grid_constant__ SolveConst c, int side0) {
  constexpr int NS = S * (S + 1) / 2;
  const int side = blockIdx.z + side0;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.exhausted || ss.broken) return;
  const SideConst& sc = c.side[side];
  const int64_t nseg = sc.nseg;
  const int64_t ncta = (nseg + kFusedSegsPerCta - 1) / kFusedSegsPerCta;
  const int64_t cta = blockIdx.x;
  if (cta >= ncta) return;
  const int64_t k = ss.blocks;
  const bool two = k >= 2;
  const double* __restrict__ u1 = sc.blocks[k - 1];
  const double* __restrict__ u0 = two ? sc.blocks[k - 2] : u1;
  __shared__ NF<S> f1s;
  __shared__ double m1[S * S], m0[S * S];
  if (threadIdx.x == 0) load_nf<S>(sc.nfac, k - 1, f1s);
  if (threadIdx.x < S * S) {
    m1[threadIdx.x] = __ldcg(sc.mcoef + (k - 1) * S * S + threadIdx.x);
    m0[threadIdx.x] = two ? __ldcg(sc.mcoef + (k - 2) * S * S + threadIdx.x) : 0.0;
  }
  __syncthreads();
  const NF<S>& f1 = f1s;
  double* __restrict__ out = sc.blocks[k];
  const int warp = threadIdx.x >> 5;
  const int64_t seg = cta * kFusedSegsPerCta + warp;
  const int nvalid_cta = (int)mn64(kFusedSegsPerCta, nseg - cta * kFusedSegsPerCta);
  double acc[NS];
#pragma unroll
  for (int e = 0; e < NS; ++e) acc[e] = 0.0;
  if (seg < nseg) p2_dispatch<S, MODE>(sc, u1, f1, u0, two, m1, m0, out, seg * kSeg, sc.n, acc);
  warp_seg_to_cta<NS>(acc, nvalid_cta, sc.part + cta * NS);
  if (!last_cta_arrive(sc.counter + 1, (unsigned)ncta)) return;
  if (sc.dist) {
    dist_emit<NS>(c, side, 0, sc.part, ncta, sc.chunk_f, sc.part + ncta * NS);
    return;
  }
  __shared__ double res[NS];
  final_tree<NS>(sc.part, ncta, res, sc.part + ncta * NS);
  gram_finish<S>(c, side, res, 0);
}

template <int S>
__device__ __forceinline__ void sw_put(double* p, const double* v) {
  if constexpr (S % 2 == 0) {
#pragma unroll
    for (int h = 0; h < S / 2; ++h) reinterpret_cast<double2*>(p)[h] = make_double2(v[2 * h], v[2 * h + 1]);
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) p[t] = v[t];
  }
}
template <int S>
__device__ __forceinline__ void sw_get(const double* p, double* v) {
  if constexpr (S % 2 == 0) {
#pragma unroll
    for (int h = 0; h < S / 2; ++h) {
      const double2 q = reinterpret_cast<const double2*>(p)[h];
      v[2 * h] = q.x;
      v[2 * h + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) v[t] = p[t];
  }
}

// =====================================================================
// Wavefront Lanczos pass (matrix-free stencil operators, one GPU). One launch
// does pass 2 of extension k AND pass 1 of extension k+1:
//   phase 1, tile j:     U_k = w - U_{k-2} M_{k-2} - U_{k-1} M_{k-1} on the tile's
//                        rows (p2_body) + R1 self-Gram; then the tile's flag
//   phase 2, tile j - D: z' = op U_k on that tile's rows, raw Grams against
//                        U_{k-1} and U_k (p1_body of extension k+1)
// Raw Grams need no N_k, so pass 1 of the next extension runs in
// the same launch, D tiles behind pass 2: D - 1 tiles cover the operator's
// bandwidth, so every U_k row z' needs is final (flags of lower tiles only).
// Tiles are handed out in ticket order (atomic counter), so a CTA only ever
// waits for CTAs that already hold lower tickets: no deadlock. Per side and
// iteration HBM sees U_{k-1}, U_{k-2} read and U_k written once (3 blocks,
// against 5 for the two passes); phase 2 re-reads U_k and U_{k-1} from L2.
// Tile = 8 R1 segments = the CTA partial of the separate-pass kernels, so both
// reductions are bitwise those of k_lanczos_p2 / k_lanczos_p1.
// =====================================================================
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// wave geometry of one side: tiles of kFusedSegsPerCta segments, lag D
struct WaveGeom {
  int64_t ntile, lag;
};
__device__ __forceinline__ WaveGeom wave_geom(const SideConst& sc) {
  WaveGeom w;
  w.ntile = (sc.nseg + kFusedSegsPerCta - 1) / kFusedSegsPerCta;
  const int64_t trows = (int64_t)kSeg * kFusedSegsPerCta;
  w.lag = 1 + (sc.bw + trows - 1) / trows;
  return w;
}

template <int S, int MODE>
__global__ void __launch_bounds__(kFusedThreads, kWaveBlocks)
    k_lanczos_wave(const __grid_constant__ SolveConst c, int side0, int interleave) {
  constexpr int NS = S * (S + 1) / 2, NB = S * S;
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  unsigned* ctl = c.side[side0].sctr;  // [0] ticket, [1] CTAs done (launch-wide)
  __shared__ unsigned tk;
  if (threadIdx.x == 0) tk = atomicAdd(ctl, 1u);
  __syncthreads();
  const int side = interleave ? side0 + (int)(tk & 1u) : side0;
  const int64_t j = interleave ? (int64_t)(tk >> 1) : (int64_t)tk;
  const SideState& ss = st->side[side];
  const SideConst& sc = c.side[side];
  const WaveGeom wg = wave_geom(sc);
  const bool active = !(ss.exhausted || ss.broken) && j < wg.ntile + wg.lag;
  if (active) {
    const int64_t k = ss.blocks;
    const bool two = k >= 2;
    const unsigned stamp = (unsigned)k;
    unsigned* flag = sc.sctr + 4;  // per tile: extension whose U_k rows are final
    double* pself = sc.spart;                         // [ntile][NS]
    double* pgam = sc.spart + wg.ntile * NS;          // [ntile][2 NB]
    const double* __restrict__ u1 = sc.blocks[k - 1];
    const double* __restrict__ u0 = two ? sc.blocks[k - 2] : u1;
    double* __restrict__ out = sc.blocks[k];
    const int warp = threadIdx.x >> 5;
    __shared__ NF<S> f1s;
    if (j < wg.ntile) {
      // phase 1: U_k on tile j (pass 2 of extension k)
      __shared__ double m1[NB], m0[NB];
      if (threadIdx.x == 0) load_nf<S>(sc.nfac, k - 1, f1s);
      if (threadIdx.x < NB) {
        m1[threadIdx.x] = __ldcg(sc.mcoef + (k - 1) * NB + threadIdx.x);
        m0[threadIdx.x] = two ? __ldcg(sc.mcoef + (k - 2) * NB + threadIdx.x) : 0.0;
      }
      __syncthreads();
      const int64_t seg = j * kFusedSegsPerCta + warp;
      const int nvalid = (int)mn64(kFusedSegsPerCta, sc.nseg - j * kFusedSegsPerCta);
      double acc[NS];
#pragma unroll
      for (int e = 0; e < NS; ++e) acc[e] = 0.0;
      if (seg < sc.nseg) p2_dispatch<S, MODE>(sc, u1, f1s, u0, two, m1, m0, out, seg * kSeg, sc.n, acc);
      warp_seg_to_cta<NS>(acc, nvalid, pself + j * NS);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release_u32(flag + j, stamp);
    }
    const int64_t q = j - wg.lag;
    if (q >= 0) {
      // phase 2: z' = op U_k on tile q (pass 1 of extension k + 1); the rows of
      // U_k it reads lie in tiles [q - lag + 1, q + lag - 1], all below j
      if (threadIdx.x == 0) {
        const int64_t lo = mx64(0, q - wg.lag + 1), hi = mn64(wg.ntile - 1, q + wg.lag - 1);
        for (int64_t t = lo; t <= hi; ++t)
          while (ld_acquire_u32(flag + t) != stamp) __nanosleep(64);
      }
      __syncthreads();
      const int64_t seg = q * kFusedSegsPerCta + warp;
      const int nvalid = (int)mn64(kFusedSegsPerCta, sc.nseg - q * kFusedSegsPerCta);
      double acc[2 * NB];
#pragma unroll
      for (int e = 0; e < 2 * NB; ++e) acc[e] = 0.0;
      if (seg < sc.nseg) {
        const int64_t base = seg * kSeg;  // (f1s: unused by matrix-free rows, no w store)
        if (base + kSeg <= sc.n)
          p1_body<S, MODE, true, false, true>(sc, out, f1s, u1, base, sc.n, acc);
        else
          p1_body<S, MODE, true, true, true>(sc, out, f1s, u1, base, sc.n, acc);
      }
      warp_seg_to_cta<2 * NB>(acc, nvalid, pgam + q * 2 * NB);
    }
    // last CTA of this side: both roots, pass-2 finalisation, then pass-1 of k + 1
    if (last_cta_arrive(sc.sctr + 2, (unsigned)(wg.ntile + wg.lag))) {
      __shared__ double rself[NS], rgam[2 * NB];
      double* scratch = sc.spart + wg.ntile * (NS + 2 * NB);
      final_tree<NS>(pself, wg.ntile, rself, scratch);
      final_tree<2 * NB>(pgam, wg.ntile, rgam, scratch);
      gram_finish<S>(c, side, rself, 0);
      __syncthreads();
      if (st->side[side].stage == ST_GROW_DIRECT) p1_finish<S>(sc, k + 1, rgam);
    }
  }
  // launch-wide: the last CTA resets the ticket for the next launch
  if (last_cta_arrive(ctl + 1, gridDim.x)) {
    if (threadIdx.x == 0) *ctl = 0u;
  }
}

// =====================================================================
// Column sweep (2D grid stencil, g = 512 * 2^j <= 4096, s <= 2, one GPU): the
// same two passes as the wavefront kernel (pass 2 of extension k + pass 1 of
// k + 1), organised so that nothing is re-read: one thread per grid column of
// a 512-column strip walks down a range of grid lines. The two input streams
// (U_{k-1}, U_{k-2}) arrive in shared-memory line rings by cp.async, issued
// four lines ahead (so HBM latency never reaches the registers); the U_k lines
// the stencil needs stay in a three-line shared ring. Out-of-grid neighbours
// are stored as +0.0, so every row's stencil is the branch-free ascending-
// column sum of the CSR order.
// Step y (one __syncthreads): U_k(y) is formed and stored, then z' = op U_k on
// line y-1; meanwhile three reducer warps form R1 segment partials (lane l
// sums columns l, l+32, ... sequentially, then the xor butterfly) of the
// self-Gram of line y-1 and the raw Grams of line y-2 from the rings.
// A strip's piece of a line is one R1 segment; the last strip CTA of a line
// range forms the line nodes (aligned groups of nstrip segments) and the last
// range of a side reduces them and finalises both passes, bitwise as
// k_lanczos_p2 / k_lanczos_p1.
// =====================================================================
#ifndef SK_CS_NC
#define SK_CS_NC 2
#endif
#ifndef SK_CS_CARRY
#define SK_CS_CARRY 1
#endif
#ifndef SK_CS_TMA
#define SK_CS_TMA 1
#endif
#ifndef SK_CS_ROLEMAP
#define SK_CS_ROLEMAP 0  // reducer warps on one scheduler (needs SK_CS_NC == 2)
#endif
#ifndef SK_CS_NOINLINE_RED
#define SK_CS_NOINLINE_RED 1  // reducer warps call separately compiled (noinline) functions
#endif
#ifndef SK_CS_FAST
#define SK_CS_FAST 1  // V2: branch-free interior steps of the column warps, three per loop trip
#endif
#ifndef SK_CS_V2
#define SK_CS_V2 0  // EXPERIMENTAL, OFF: software-pipelined steps with a split-phase mbarrier step barrier.
                    // Faster (C5 1815 vs 1776 iter/s) but NOT reproducible: config 3 (2908 launches of
                    // 148 CTAs) shows rounding-level deviations at data-dependent iterations in every run
                    // (profiles/r2/README.md); the barrier-per-line schedule below is bit-stable.
#endif
constexpr int kCsNC = SK_CS_NC;            // grid columns per column thread
constexpr int kCsColWarps = 16 / kCsNC;    // 512 columns
#ifndef SK_CS_RED5
#define SK_CS_RED5 0  // (measured 1507 vs 1776 iter/s at C5: off) five reducer warps: self-Gram + (slot 0, slot 1) x (z' column u = 0, 1); needs SK_CS_V2 == 0
#endif
constexpr int kCsRedWarps = (SK_CS_RED5 && !SK_CS_V2) ? 5 : 3;  // self-Gram, raw Gram slots 0 / 1 (per z' column with RED5)
constexpr int kCsThreads = 32 * (kCsColWarps + 1 + kCsRedWarps);
constexpr int kCsA = kSeg + 4;             // U_{k-1} lines: columns x0-2 .. x0+513
constexpr int kCsK = kSeg + 2;             // U_k / U_{k-2} lines: columns x0-1 .. x0+512
constexpr int kCsAR = 8;                   // U_{k-1} ring: lines y-3 .. y+4 (prefetch 4)
#ifndef SK_CS_V3
#define SK_CS_V3 0  // (measured 1730 vs 1815 iter/s at C5: off) reducer warps decoupled from the step barrier (deeper K / Z rings); needs SK_CS_V2
#endif
constexpr int kCsBR = SK_CS_V3 ? 4 : 8;    // U_{k-2} ring (V3: lines y .. y+3; else y-3 .. y+4)
constexpr int kCsKR = SK_CS_V3 ? 8 : 4;    // U_k ring (V3: the reducers may lag two lines)
constexpr int kCsZR = SK_CS_V3 ? 4 : 2;    // z' ring
constexpr int kCsMaxLines = 1024;          // lines per range (the tail's line nodes fit in the rings)
constexpr int kCsBlk = 8;                  // lines per tail block node (range alignment)

template <int S>
__device__ __forceinline__ void cs_copy(double* dst, const double* src, bool ok) {
  if (ok) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if constexpr (S * 8 == 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) dst[t] = 0.0;
  }
}
__device__ __forceinline__ void cs_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// bulk (TMA) line copies completing on an mbarrier
__device__ __forceinline__ void mb_init(uint64_t* mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
__device__ __forceinline__ void mb_expect_arrive(uint64_t* mb, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(mb)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* mb, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(mb))
               : "memory");
}
__device__ __forceinline__ void cs_wait3() { asm volatile("cp.async.wait_group 3;" ::: "memory"); }
// 0 + c0 up + c1 left + c2 centre + c3 right + c4 down (CSR order, mul then add)
template <int S>
__device__ __forceinline__ void cs_stencil(const double* c5, const double* up, const double* le, const double* ce,
                                           const double* ri, const double* dn, double* z) {
#pragma unroll
  for (int t = 0; t < S; ++t) {
    double a = __dadd_rn(0.0, __dmul_rn(c5[0], up[t]));
    a = __dadd_rn(a, __dmul_rn(c5[1], le[t]));
    a = __dadd_rn(a, __dmul_rn(c5[2], ce[t]));
    a = __dadd_rn(a, __dmul_rn(c5[3], ri[t]));
    z[t] = __dadd_rn(a, __dmul_rn(c5[4], dn[t]));
  }
}

#ifdef SK_CS_PROF
__device__ unsigned long long g_csprof[2][1024][4];
#endif
// canonical tree over N values src[j * stride], j < N (N a power of two)
template <int N>
__device__ __forceinline__ double cs_group_tree(const double* __restrict__ src, int stride) {
  double a[N];
#pragma unroll
  for (int j = 0; j < N; ++j) a[j] = __ldcg(src + (int64_t)j * stride);
#pragma unroll
  for (int w = N / 2; w >= 1; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) a[j] = __dadd_rn(a[2 * j], a[2 * j + 1]);
  return a[0];
}
// line nodes of a range: ln[l*NE + e] = canonical tree over the NSTRIP segment
// partials gs[(l*NSTRIP + q)*NE + e]; four items per thread in flight
template <int NE, int NSTRIP>
__device__ __forceinline__ void cs_line_nodes(const double* __restrict__ gs, int nitem, double* ln) {
  constexpr int U = 4;
  for (int i0 = threadIdx.x; i0 < nitem; i0 += U * blockDim.x) {
    double vv[U][NSTRIP];
#pragma unroll
    for (int h = 0; h < U; ++h) {
      const int idx = i0 + h * blockDim.x;
      if (idx < nitem) {
        const int l = idx / NE, e = idx - l * NE;
#pragma unroll
        for (int q = 0; q < NSTRIP; ++q) vv[h][q] = __ldcg(gs + ((int64_t)l * NSTRIP + q) * NE + e);
      }
    }
#pragma unroll
    for (int h = 0; h < U; ++h) {
      const int idx = i0 + h * blockDim.x;
      if (idx < nitem) {
#pragma unroll
        for (int w = NSTRIP / 2; w >= 1; w >>= 1)
#pragma unroll
          for (int j = 0; j < w; ++j) vv[h][j] = __dadd_rn(vv[h][2 * j], vv[h][2 * j + 1]);
        ln[idx] = vv[h][0];
      }
    }
  }
}
// Reducer warps of the column sweep as separately compiled functions: inside the kernel
// (168 registers, three roles) ptxas sank every shared-memory load of these loops to its
// first use, so a line cost 16 dependent shared-memory round trips and the reducer warps
// were the critical path of every step (ncu, profiles/r2). Here the lane's 16 rows are
// loaded up front; the sums keep the R1 order (rows m = 0 .. 15 sequentially, then the xor
// butterfly), bitwise as before.
// Four xor butterflies at once (R1 lane combine, d = 16 .. 1) with halving exchanges: in
// round d = 16 the lanes with bit 4 clear keep entries 0, 1 and hand 2, 3 to their partner
// (and vice versa), in round d = 8 they split once more, rounds 4, 2, 1 run on the single
// entry a lane is left with. Every addition is "own + partner" exactly as in butterfly(), and
// IEEE addition is commutative, so every lane of the plain butterfly holds the same bits at
// every level: the entry e = lane >> 3 that a lane ends with is bitwise butterfly(v_e). 15
// shuffle/add pairs instead of 40 on the reducer warps' critical path.
__device__ __forceinline__ double butterfly4(double v0, double v1, double v2, double v3, int lane) {
  const bool h4 = (lane & 16) != 0, h3 = (lane & 8) != 0;
  double k0 = h4 ? v2 : v0, k1 = h4 ? v3 : v1;
  const double s0 = h4 ? v0 : v2, s1 = h4 ? v1 : v3;
  k0 = __dadd_rn(k0, shfl_xor_d(s0, 16));
  k1 = __dadd_rn(k1, shfl_xor_d(s1, 16));
  double kk = h3 ? k1 : k0;
  const double ss = h3 ? k0 : k1;
  kk = __dadd_rn(kk, shfl_xor_d(ss, 8));
#pragma unroll
  for (int d = 4; d >= 1; d >>= 1) kk = __dadd_rn(kk, shfl_xor_d(kk, d));
  return kk;
}
template <int S>
__device__ __noinline__ void cs_reduce_self(const double* __restrict__ K1, double* __restrict__ out, int lane) {
  constexpr int NS = S * (S + 1) / 2;
  double vv[kLRows][S];
#pragma unroll
  for (int m = 0; m < kLRows; ++m) sw_get<S>(K1 + (lane + 32 * m) * S, vv[m]);
  double acc[NS];
#pragma unroll
  for (int e = 0; e < NS; ++e) acc[e] = 0.0;
#pragma unroll
  for (int m = 0; m < kLRows; ++m) {
    int e = 0;
#pragma unroll
    for (int u = 0; u < S; ++u)
#pragma unroll
      for (int t = 0; t <= u; ++t) {
        acc[e] = __dadd_rn(acc[e], __dmul_rn(vv[m][t], vv[m][u]));
        ++e;
      }
  }
  if constexpr (NS == 3) {
    const double r = butterfly4(acc[0], acc[1], acc[2], 0.0, lane);
    if ((lane & 7) == 0 && (lane >> 3) < NS) out[lane >> 3] = r;
  } else {
#pragma unroll
    for (int e = 0; e < NS; ++e) {
      const double r = butterfly(acc[e]);
      if (lane == e) out[e] = r;
    }
  }
}
template <int S>
__device__ __noinline__ void cs_reduce_slot(const double* __restrict__ src, const double* __restrict__ Z,
                                            double* __restrict__ out, int lane) {
  constexpr int NB = S * S;
  double av[kLRows][S], z[kLRows][S];
#pragma unroll
  for (int m = 0; m < kLRows; ++m) {
    sw_get<S>(src + (lane + 32 * m) * S, av[m]);
    sw_get<S>(Z + (lane + 32 * m) * S, z[m]);
  }
  double acc[NB];
#pragma unroll
  for (int e = 0; e < NB; ++e) acc[e] = 0.0;
#pragma unroll
  for (int m = 0; m < kLRows; ++m)
#pragma unroll
    for (int u = 0; u < S; ++u)
#pragma unroll
      for (int t = 0; t < S; ++t) acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(av[m][t], z[m][u]));
  if constexpr (NB == 4) {
    const double r = butterfly4(acc[0], acc[1], acc[2], acc[3], lane);
    if ((lane & 7) == 0) out[lane >> 3] = r;
  } else {
#pragma unroll
    for (int e = 0; e < NB; ++e) {
      const double r = butterfly(acc[e]);
      if (lane == e) out[e] = r;
    }
  }
}

// One z' column of a raw-Gram slot: entries (u, t) = sum_rows src[row][t] * z'[row][u], t < S, for a
// fixed u (RED5: the four entries of a slot at s = 2 are split over two warps, so no reducer warp
// carries more than three entries per line). Same R1 order per entry as cs_reduce_slot.
template <int S>
__device__ __noinline__ void cs_reduce_slot_u(const double* __restrict__ src, const double* __restrict__ Z, int u,
                                              double* __restrict__ out, int lane) {
  double av[kLRows][S], zu[kLRows];
#pragma unroll
  for (int m = 0; m < kLRows; ++m) {
    sw_get<S>(src + (lane + 32 * m) * S, av[m]);
    zu[m] = Z[(lane + 32 * m) * S + u];
  }
  double acc[S];
#pragma unroll
  for (int t = 0; t < S; ++t) acc[t] = 0.0;
#pragma unroll
  for (int m = 0; m < kLRows; ++m)
#pragma unroll
    for (int t = 0; t < S; ++t) acc[t] = __dadd_rn(acc[t], __dmul_rn(av[m][t], zu[m]));
  if constexpr (S == 2) {
    // two butterflies with one halving exchange (see butterfly4): lanes with bit 4 clear end with
    // entry t = 0, the others with t = 1
    const bool h4 = (lane & 16) != 0;
    double kk = h4 ? acc[1] : acc[0];
    const double ss = h4 ? acc[0] : acc[1];
    kk = __dadd_rn(kk, shfl_xor_d(ss, 16));
#pragma unroll
    for (int d = 8; d >= 1; d >>= 1) kk = __dadd_rn(kk, shfl_xor_d(kk, d));
    if ((lane & 15) == 0) out[lane >> 4] = kk;
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) {
      const double r = butterfly(acc[t]);
      if (lane == t) out[t] = r;
    }
  }
}

template <int S>
__global__ void __launch_bounds__(kCsThreads, 1)
    k_lanczos_cols(const __grid_constant__ SolveConst c, int side0, int nranges) {
  constexpr int NS = S * (S + 1) / 2, NB = S * S, NE = NS + 2 * NB;
  constexpr int AL = kCsA * S, KL = kCsK * S, ZL = kSeg * S;  // ring line strides (doubles)
#if SK_CS_TMA
  constexpr int BL = AL, BO = 2;  // U_{k-2} lines span the same columns as U_{k-1} (16-byte aligned rows)
#else
  constexpr int BL = KL, BO = 1;
#endif
  const int side = side0 + blockIdx.y;
  if (side >= c.nsides) return;
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.exhausted || ss.broken) return;
  const SideConst& sc = c.side[side];
  const int g = (int)sc.sg;
  const int nstrip = g / kSeg;
  const int sx = blockIdx.x % nstrip, rg = blockIdx.x / nstrip;
  // line ranges are aligned to kCsBlk lines (the tail reduces whole line blocks)
  const int y0 = (int)((int64_t)rg * (g / kCsBlk) / nranges) * kCsBlk;
  const int y1 = (int)((int64_t)(rg + 1) * (g / kCsBlk) / nranges) * kCsBlk;
  const int x0 = sx * kSeg;
  const int64_t k = ss.blocks;
  const bool two = k >= 2;
#ifdef SK_CS_PROF
  if (threadIdx.x == 0) g_csprof[blockIdx.y][blockIdx.x][0] = globaltimer();
#endif
  extern __shared__ __align__(16) double cs_smem[];
  double* Ar = cs_smem;                    // [kCsAR][AL]
  double* Br = Ar + kCsAR * AL;            // [kCsBR][KL]
  double* Kb = Br + kCsBR * BL;            // [kCsKR][KL]
  double* Zs = Kb + kCsKR * KL;            // [kCsZR][ZL]
  __shared__ NF<S> f1s;
  __shared__ double m1[NB], m0[NB];
  if (threadIdx.x == 0) load_nf<S>(sc.nfac, k - 1, f1s);
  if (threadIdx.x < NB) {
    m1[threadIdx.x] = __ldcg(sc.mcoef + (k - 1) * NB + threadIdx.x);
    m0[threadIdx.x] = two ? __ldcg(sc.mcoef + (k - 2) * NB + threadIdx.x) : 0.0;
  }
  // Roles by hardware warp id: warp w issues on scheduler (SMSP) w % 4. The three reducer
  // warps sit together on SMSP 0 (hardware warps 0, 4, 8 -> roles 9, 10, 11) and the eight
  // column warps plus the halo warp share SMSPs 1 - 3, three each: the reducers' long
  // dependent FP64 chains then run beside each other instead of behind two column warps'
  // streams (ncu, profiles/r2: the reducers were the critical path of every step).
  const int lane = threadIdx.x & 31;
#if SK_CS_ROLEMAP
  const int hwarp = threadIdx.x >> 5;
  const int warp = (hwarp & 3) == 0 ? kCsColWarps + 1 + (hwarp >> 2) : (hwarp >> 2) * 3 + (hwarp & 3) - 1;
  static_assert(kCsColWarps == 8 && kCsThreads == 384, "role map assumes 8 column warps + halo + 3 reducers");
#else
  const int warp = threadIdx.x >> 5;
#endif
  const int64_t gS = (int64_t)g * S;
  // column roles: column warp w, lane l owns x0 + 32 w + l + 256 c (c < kCsNC);
  // the halo warp's lanes 0..3 own x0-1, x0+512 (computed), x0-2, x0+513 (loaded)
  int xs[kCsNC];
  bool cv[kCsNC];
  int nslot = 0;
  bool compute = false, inner = false;
  if (warp < kCsColWarps) {
#pragma unroll
    for (int q = 0; q < kCsNC; ++q) xs[q] = x0 + 32 * warp + lane + (kSeg / kCsNC) * q;
    nslot = kCsNC;
    compute = inner = true;
  } else if (warp == kCsColWarps && lane < 4) {
    xs[0] = lane == 0 ? x0 - 1 : lane == 1 ? x0 + kSeg : lane == 2 ? x0 - 2 : x0 + kSeg + 1;
#pragma unroll
    for (int q = 1; q < kCsNC; ++q) xs[q] = xs[0];
    nslot = 1;
    compute = lane < 2;
  }
#pragma unroll
  for (int q = 0; q < kCsNC; ++q) cv[q] = q < nslot && xs[q] >= 0 && xs[q] < g;
  const double* U1 = sc.blocks[k - 1];
  const double* U0 = two ? sc.blocks[k - 2] : U1;
  double* UK = sc.blocks[k];
  const int ys = y0 - 1;
#if !SK_CS_TMA
  // copies of line ya of U_{k-1} (and line yb of U_{k-2}) for this thread's columns
  auto copy_a = [&](int ya) {
    double* d = Ar + (ya & (kCsAR - 1)) * AL;
    const bool lok = ya >= 0 && ya < g;
#pragma unroll
    for (int q = 0; q < kCsNC; ++q)
      if (q < nslot) cs_copy<S>(d + (xs[q] - x0 + 2) * S, U1 + ((int64_t)ya * g + (cv[q] ? xs[q] : 0)) * S, lok && cv[q]);
  };
  auto copy_b = [&](int yb) {
    double* d = Br + (yb & (kCsBR - 1)) * BL;
    const bool lok = two && yb >= 0 && yb < g;
#pragma unroll
    for (int q = 0; q < kCsNC; ++q)
      if (q < nslot) cs_copy<S>(d + (xs[q] - x0 + BO) * S, U0 + ((int64_t)yb * g + (cv[q] ? xs[q] : 0)) * S, lok && cv[q]);
  };
#endif
#if SK_CS_TMA
  // line loads by one thread (reducer warp 0, lane 0) as bulk copies: group t
  // (issued at step ys + t - 4, consumed at step ys + t) completes on mbarrier
  // mbar[t & 7]. Columns outside the grid stay zero (written once here); lines
  // outside the grid are zero-filled by the issuing warp.
  __shared__ __align__(8) uint64_t mbar[8];
  const bool issuer = warp == (SK_CS_V3 ? kCsColWarps : kCsColWarps + 1);  // V3: the halo warp
  const int ca = x0 - 2 < 0 ? 0 : x0 - 2, cb = x0 + kSeg + 1 >= g ? g - 1 : x0 + kSeg + 1;
  const unsigned lbytes = (unsigned)((cb - ca + 1) * S * 8);
  if (threadIdx.x < 8) mb_init(&mbar[threadIdx.x]);
  for (int i = threadIdx.x; i < kCsAR + kCsBR; i += blockDim.x) {
    double* d = Ar + i * AL;  // Br follows Ar with the same stride
#pragma unroll
    for (int t = 0; t < 2 * S; ++t) {
      if (x0 == 0) d[t] = 0.0;
      if (x0 + kSeg >= g) d[(kCsA - 2) * S + t] = 0.0;
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // the issuing warp: one group = U_{k-1} lines [la0, la1] and U_{k-2} line lb (lb < 0: none)
  auto issue = [&](int t, int la0, int la1, int lb) {
    unsigned tx = 0;
    for (int ya = la0; ya <= la1; ++ya) tx += (ya >= 0 && ya < g) ? lbytes : 0u;
    const bool bok = two && lb >= 0 && lb < g;
    tx += bok ? lbytes : 0u;
    for (int ya = la0; ya <= la1; ++ya)
      if (ya < 0 || ya >= g) {
        double* d = Ar + (ya & (kCsAR - 1)) * AL;
        for (int i = lane; i < AL; i += 32) d[i] = 0.0;
      }
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint64_t* mb = &mbar[t & 7];
      mb_expect_arrive(mb, tx);
      for (int ya = la0; ya <= la1; ++ya)
        if (ya >= 0 && ya < g)
          bulk_g2s(Ar + (ya & (kCsAR - 1)) * AL + (ca - x0 + 2) * S, U1 + ((int64_t)ya * g + ca) * S, lbytes, mb);
      if (bok)
        bulk_g2s(Br + (lb & (kCsBR - 1)) * BL + (ca - x0 + 2) * S, U0 + ((int64_t)lb * g + ca) * S, lbytes, mb);
    }
  };
  // prologue: U_{k-1} lines ys-3 .. ys+4, U_{k-2} lines ys .. ys+3 (groups 0 .. 3)
  if (issuer) {
    issue(0, ys - 3, ys + 1, ys);
    for (int t = 1; t < (SK_CS_V3 ? 3 : 4); ++t) issue(t, ys + t + 1, ys + t + 1, ys + t);
  }
#else
  __syncthreads();
  // prologue: U_{k-1} lines ys-3 .. ys+4, U_{k-2} lines ys .. ys+3 (groups G(ys-4) .. G(ys-1))
  if (nslot) {
    for (int ya = ys - 3; ya <= ys; ++ya) copy_a(ya);
  }
  for (int v = ys - 4; v < ys; ++v) {
    if (nslot) copy_a(v + 5);
    if (compute) copy_b(v + 4);
    cs_commit();
  }
#endif
  double* gseg = sc.spart;                              // [g * nstrip][NE] segment partials
  double* lnode = sc.spart + (int64_t)g * nstrip * NE;  // [g][NE] line nodes

#if SK_CS_CARRY
  // a thread's own column is carried down the lines in registers: U_{k-1} lines
  // y-1, y (up, centre of the next stencil) and U_k lines y-2, y-1 (its own
  // earlier outputs); only the neighbours and the new lines come from shared memory
  double cup[kCsNC][S], cce[kCsNC][S], kup[kCsNC][S], kce[kCsNC][S];
#pragma unroll
  for (int q = 0; q < kCsNC; ++q)
#pragma unroll
    for (int t = 0; t < S; ++t) cup[q][t] = cce[q][t] = kup[q][t] = kce[q][t] = 0.0;
#endif
#if SK_CS_V2
  // ---- software-pipelined steps with a split-phase step barrier ----------------------
  // The step barrier is an mbarrier (one arrival per warp at the END of its step t,
  // waited for only where step t + 1 first touches another warp's data), and a column
  // warp's step is reordered so that nothing in its first half depends on other warps:
  //   A-part(y): U_k(y) from operands already in registers (the thread's own column of
  //              U_{k-1} is carried; its neighbours' and the U_{k-2} value were loaded
  //              from the TMA rings during the previous step), global store, K ring store
  //   wait(step t - 1 finished everywhere)
  //   loads: K(y-1) neighbours AND the A-part operands of line y + 1 (their latency
  //              overlaps the z-part)
  //   z-part(y-1): z' = op U_k on line y - 1, Z ring store; arrive.
  // Every point's arithmetic is unchanged (bitwise the barrier-per-line schedule).
#if SK_CS_V3
  // V3: two barrier rings. sbar[t & 3] completes when the nine producer warps (columns + halo)
  // have finished step t - 1; rbar[t & 3] when the three reducer warps have finished step t.
  // Producers wait for sbar of the previous step and for the reducers' step t - 2, so the
  // reducers may run up to two lines behind (K ring of 8, z' ring of 4 lines); their long
  // dependent sums no longer gate the producers' step. Reducers only wait for sbar.
  __shared__ __align__(8) uint64_t sbar[4], rbar[4];
  if (threadIdx.x < 8) {
    uint64_t* b = threadIdx.x < 4 ? &sbar[threadIdx.x] : &rbar[threadIdx.x - 4];
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
                 "r"(threadIdx.x < 4 ? (unsigned)(kCsColWarps + 1) : (unsigned)kCsRedWarps)
                 : "memory");
  }
  __syncthreads();
  const bool producer = warp <= kCsColWarps;
  auto step_arrive = [&](int t) {
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(producer ? &sbar[(t + 1) & 3] : &rbar[t & 3]))
                   : "memory");
  };
  auto step_wait = [&](int t) {  // t >= 1
    mb_wait(&sbar[t & 3], (unsigned)((t - 1) >> 2) & 1u);
    if (producer && t >= 2) mb_wait(&rbar[(t - 2) & 3], (unsigned)((t - 2) >> 2) & 1u);
  };
#else
#ifdef SK_CS_DBG_PADBAR
  __shared__ __align__(128) uint64_t sbar_pad[48];  // step barriers 128 bytes apart and away from mbar[]
  uint64_t* sbar = sbar_pad + 16;
  constexpr int kSbStride = 16;
#else
  __shared__ __align__(8) uint64_t sbar_arr[2];
  uint64_t* sbar = sbar_arr;
  constexpr int kSbStride = 1;
#endif
#ifdef SK_CS_DBG_ALLARRIVE
  constexpr unsigned kSbCount = kCsThreads;  // every thread arrives for itself
#else
  constexpr unsigned kSbCount = kCsThreads / 32;
#endif
  if (threadIdx.x < 2) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&sbar[threadIdx.x * kSbStride])),
                 "r"(kSbCount)
                 : "memory");
  }
  __syncthreads();
  auto step_arrive = [&](int t) {
#ifdef SK_CS_DBG_ALLARRIVE
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&sbar[((t + 1) & 1) * kSbStride]))
                 : "memory");
#else
#ifdef SK_CS_DBG_FENCE
    __threadfence_block();  // every lane's shared-memory stores performed before lane 0's arrive
#endif
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&sbar[((t + 1) & 1) * kSbStride]))
                   : "memory");
#endif
  };
  auto step_wait = [&](int t) {  // all warps finished step t - 1 (t >= 1)
#ifndef SK_CS_DBG_V1LIKE
    const unsigned par = (t & 1) ? (unsigned)(t >> 1) & 1u : (unsigned)((t >> 1) + 1) & 1u;
    mb_wait(&sbar[(t & 1) * kSbStride], par);
#endif
  };
#endif
  double ale[kCsNC][S], ari[kCsNC][S], adn[kCsNC][S], abb[kCsNC][S];  // A-part operands of line y
  auto load_a_ops = [&](int yy) {  // neighbours of U_{k-1}(yy), U_{k-1}(yy + 1) own, U_{k-2}(yy) own
    const double* A0 = Ar + (yy & (kCsAR - 1)) * AL;
    const double* Ap = Ar + ((yy + 1) & (kCsAR - 1)) * AL;
    const double* B0 = Br + (yy & (kCsBR - 1)) * BL;
#pragma unroll
    for (int q = 0; q < kCsNC; ++q)
      if (q < nslot) {
        const int ai = (xs[q] - x0 + 2) * S;
        sw_get<S>(A0 + ai - S, ale[q]);
        sw_get<S>(A0 + ai + S, ari[q]);
        sw_get<S>(Ap + ai, adn[q]);
        sw_get<S>(B0 + ai + (BO - 2) * S, abb[q]);
      }
  };
  if (warp <= kCsColWarps && compute) {
    mb_wait(&mbar[0], 0u);  // group 0: U_{k-1} lines ys-3 .. ys+1, U_{k-2} line ys
#pragma unroll
    for (int q = 0; q < kCsNC; ++q)
      if (q < nslot) {
        const int ai = (xs[q] - x0 + 2) * S;
        sw_get<S>(Ar + ((ys - 1) & (kCsAR - 1)) * AL + ai, cup[q]);
        sw_get<S>(Ar + (ys & (kCsAR - 1)) * AL + ai, cce[q]);
      }
    load_a_ops(ys);
  }
#if SK_CS_FAST
  // Interior steps of the column warps (lines y0+1 .. y1-1: every flag of the generic step
  // is true, every point is in the grid), three per loop trip so that the three-deep
  // register rotations (U_{k-1} own column: loaded -> centre -> up; U_k: new -> centre -> up)
  // come back to their registers without moves; coefficients live in registers.
  double rc5[5], rm0[NB], rm1[NB];
  NF<S> rf1;
#pragma unroll
  for (int e = 0; e < 5; ++e) rc5[e] = sc.scoef[e];
#pragma unroll
  for (int e = 0; e < NB; ++e) {
    rm0[e] = m0[e];
    rm1[e] = m1[e];
  }
  rf1 = f1s;
  const int ai0 = warp < kCsColWarps ? (xs[0] - x0 + 2) * S : 0, ki0 = ai0 - S, zi0 = ai0 - 2 * S;
  constexpr int QO = (kSeg / kCsNC) * S;  // doubles between a thread's columns
  double* pU = UK + ((int64_t)(y0 + 1) * g + (warp < kCsColWarps ? xs[0] : 0)) * S;
  auto main_step = [&](int y) {
    const int t = y - ys;
    double vq[kCsNC][S];
    {
      double* K0 = Kb + (y & (kCsKR - 1)) * KL + ki0;
#pragma unroll
      for (int q = 0; q < kCsNC; ++q) {
        double z[S], v[S], ce[S];
#pragma unroll
        for (int u = 0; u < S; ++u) ce[u] = cce[q][u];
        cs_stencil<S>(rc5, cup[q], ale[q], ce, ari[q], adn[q], z);
#pragma unroll
        for (int u = 0; u < S; ++u) {
          cup[q][u] = ce[u];
          cce[q][u] = adn[q][u];
        }
        norm_row<S>(z, rf1, v);
        if (two) {
#pragma unroll
          for (int u = 0; u < S; ++u) {
            double tmp = 0.0;
#pragma unroll
            for (int w_ = 0; w_ < S; ++w_) tmp = __dadd_rn(tmp, __dmul_rn(abb[q][w_], rm0[u * S + w_]));
            v[u] = __dsub_rn(v[u], tmp);
          }
        }
#pragma unroll
        for (int u = 0; u < S; ++u) {
          double tmp = 0.0;
#pragma unroll
          for (int w_ = 0; w_ < S; ++w_) tmp = __dadd_rn(tmp, __dmul_rn(ce[w_], rm1[u * S + w_]));
          v[u] = __dsub_rn(v[u], tmp);
        }
        st_row<S>(pU + q * QO, 0, v);
        sw_put<S>(K0 + q * QO, v);
#pragma unroll
        for (int u = 0; u < S; ++u) vq[q][u] = v[u];
      }
      pU += gS;
    }
    step_wait(t);
    {
      const double* K1 = Kb + ((y - 1) & (kCsKR - 1)) * KL + ki0;
      double kle[kCsNC][S], kri[kCsNC][S];
#pragma unroll
      for (int q = 0; q < kCsNC; ++q) {
        sw_get<S>(K1 + q * QO - S, kle[q]);
        sw_get<S>(K1 + q * QO + S, kri[q]);
      }
      mb_wait(&mbar[(t + 1) & 7], (unsigned)((t + 1) >> 3) & 1u);
      {
        const double* A0 = Ar + ((y + 1) & (kCsAR - 1)) * AL + ai0;
        const double* Ap = Ar + ((y + 2) & (kCsAR - 1)) * AL + ai0;
        const double* B0 = Br + ((y + 1) & (kCsBR - 1)) * BL + ai0 + (BO - 2) * S;
#pragma unroll
        for (int q = 0; q < kCsNC; ++q) {
          sw_get<S>(A0 + q * QO - S, ale[q]);
          sw_get<S>(A0 + q * QO + S, ari[q]);
          sw_get<S>(Ap + q * QO, adn[q]);
          sw_get<S>(B0 + q * QO, abb[q]);
        }
      }
      double* Z1 = Zs + ((y - 1) & (kCsZR - 1)) * ZL + zi0;
#pragma unroll
      for (int q = 0; q < kCsNC; ++q) {
        double z2[S];
#pragma unroll
        for (int u = 0; u < S; ++u) {
          double a2 = __dadd_rn(0.0, __dmul_rn(rc5[0], kup[q][u]));
          a2 = __dadd_rn(a2, __dmul_rn(rc5[1], kle[q][u]));
          a2 = __dadd_rn(a2, __dmul_rn(rc5[2], kce[q][u]));
          a2 = __dadd_rn(a2, __dmul_rn(rc5[3], kri[q][u]));
          z2[u] = __dadd_rn(a2, __dmul_rn(rc5[4], vq[q][u]));
          kup[q][u] = kce[q][u];
          kce[q][u] = vq[q][u];
        }
        sw_put<S>(Z1 + q * QO, z2);
      }
    }
    step_arrive(t);
  };
  // The halo warp's interior step: its two computing lanes form U_k at columns x0 - 1 and
  // x0 + 512 for the neighbours' stencils (K ring only: no global store, and z' is never
  // needed there, so there is no z-part).
  const int hai = (xs[0] - x0 + 2) * S;
  const unsigned ring_dst = (unsigned)((ca - x0 + 2) * S);
  auto halo_step = [&](int y) {
    const int t = y - ys;
    if (compute) {
      double z[S], v[S], ce[S];
#pragma unroll
      for (int u = 0; u < S; ++u) ce[u] = cce[0][u];
      cs_stencil<S>(rc5, cup[0], ale[0], ce, ari[0], adn[0], z);
#pragma unroll
      for (int u = 0; u < S; ++u) {
        cup[0][u] = ce[u];
        cce[0][u] = adn[0][u];
      }
      norm_row<S>(z, rf1, v);
      if (two) {
#pragma unroll
        for (int u = 0; u < S; ++u) {
          double tmp = 0.0;
#pragma unroll
          for (int w_ = 0; w_ < S; ++w_) tmp = __dadd_rn(tmp, __dmul_rn(abb[0][w_], rm0[u * S + w_]));
          v[u] = __dsub_rn(v[u], tmp);
        }
      }
#pragma unroll
      for (int u = 0; u < S; ++u) {
        double tmp = 0.0;
#pragma unroll
        for (int w_ = 0; w_ < S; ++w_) tmp = __dadd_rn(tmp, __dmul_rn(ce[w_], rm1[u * S + w_]));
        v[u] = __dsub_rn(v[u], tmp);
      }
      if (!cv[0]) {
#pragma unroll
        for (int u = 0; u < S; ++u) v[u] = 0.0;
      }
      sw_put<S>(Kb + (y & (kCsKR - 1)) * KL + hai - S, v);
#pragma unroll
      for (int u = 0; u < S; ++u) {
        kup[0][u] = kce[0][u];
        kce[0][u] = v[u];
      }
    }
    step_wait(t);
#if SK_CS_V3
    if (lane == 0) {  // group t + 3: U_{k-1} line y + 4, U_{k-2} line y + 3 (both inside the grid here)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint64_t* mb = &mbar[(t + 3) & 7];
      mb_expect_arrive(mb, two ? 2u * lbytes : lbytes);
      bulk_g2s(Ar + ((y + 4) & (kCsAR - 1)) * AL + ring_dst, U1 + ((int64_t)(y + 4) * g + ca) * S, lbytes, mb);
      if (two)
        bulk_g2s(Br + ((y + 3) & (kCsBR - 1)) * BL + ring_dst, U0 + ((int64_t)(y + 3) * g + ca) * S, lbytes, mb);
    }
#endif
    if (compute) {
      mb_wait(&mbar[(t + 1) & 7], (unsigned)((t + 1) >> 3) & 1u);
      const double* A0 = Ar + ((y + 1) & (kCsAR - 1)) * AL + hai;
      sw_get<S>(A0 - S, ale[0]);
      sw_get<S>(A0 + S, ari[0]);
      sw_get<S>(Ar + ((y + 2) & (kCsAR - 1)) * AL + hai, adn[0]);
      sw_get<S>(Br + ((y + 1) & (kCsBR - 1)) * BL + hai + (BO - 2) * S, abb[0]);
    }
    step_arrive(t);
  };
  // The reducer warps' interior step (lines y-1 / y-2 inside the range, the prefetched lines
  // y+5 / y+4 inside the grid): wait, one lean bulk-copy issue by the issuer's lane 0, one
  // call of the separately compiled reduction, arrive.
  const int rrole = warp - kCsColWarps - 1;  // 0: self-Gram (and issuer), 1 / 2: raw-Gram slots
  auto red_step = [&](int y) {
    const int t = y - ys;
    step_wait(t);
    if (rrole == 0) {
      if (!SK_CS_V3 && lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        uint64_t* mb = &mbar[(t + 4) & 7];
        mb_expect_arrive(mb, two ? 2u * lbytes : lbytes);
        bulk_g2s(Ar + ((y + 5) & (kCsAR - 1)) * AL + ring_dst, U1 + ((int64_t)(y + 5) * g + ca) * S, lbytes, mb);
        if (two)
          bulk_g2s(Br + ((y + 4) & (kCsBR - 1)) * BL + ring_dst, U0 + ((int64_t)(y + 4) * g + ca) * S, lbytes, mb);
      }
      const int yl = y - 1;
      cs_reduce_self<S>(Kb + (yl & (kCsKR - 1)) * KL + S, gseg + ((int64_t)yl * nstrip + sx) * NE, lane);
    } else {
      const int yl = y - 2;
#ifdef SK_CS_DBG_SLOT0WAIT
      if (rrole == 1) { const int j = t - 3 > 0 ? t - 3 : 0; mb_wait(&mbar[j & 7], (unsigned)(j >> 3) & 1u); }
#endif
      cs_reduce_slot<S>(rrole == 1 ? Ar + (yl & (kCsAR - 1)) * AL + 2 * S : Kb + (yl & (kCsKR - 1)) * KL + S,
                        Zs + (yl & (kCsZR - 1)) * ZL, gseg + ((int64_t)yl * nstrip + sx) * NE + NS + (rrole - 1) * NB, lane);
    }
    step_arrive(t);
  };
#endif
  for (int y = ys; y <= y1 + 1; ++y) {
    const int t = y - ys;
#ifdef SK_CS_DBG_V1LIKE
#ifndef SK_CS_DBG_NOISSUERWAIT
    if (issuer && lane == 0) mb_wait(&mbar[t & 7], (unsigned)(t >> 3) & 1u);
#endif
    __syncthreads();
#endif
#ifdef SK_CS_DBG_ISSUERWAIT
    if (issuer && lane == 0) mb_wait(&mbar[t & 7], (unsigned)(t >> 3) & 1u);
#endif
#if SK_CS_FAST
    // reducers: y-2 >= y0, y-1 < y1, and the issued lines y+5, y+4 in [0, g)
    // reducers: one tight loop over all their interior steps (lines y-1 / y-2 inside the range;
    // without V3 also the issued lines y+5, y+4 inside the grid and wanted: y <= min(y1-3, g-6))
    if (warp > kCsColWarps && y == y0 + 2) {
      const int ylast = SK_CS_V3 ? y1 - 1 : (y1 - 3 < g - 6 ? y1 - 3 : g - 6);
      if (ylast >= y) {
        for (; y <= ylast; ++y) red_step(y);
        --y;
        continue;
      }
    }
    // (V3: the halo warp's lean issue needs lines y + 4 .. y + 6 inside the grid)
    if (warp <= kCsColWarps && y >= y0 + 1 && y + 2 <= y1 - (SK_CS_V3 ? 2 : 1) && (!SK_CS_V3 || y + 6 < g)) {
      if (warp < kCsColWarps) {
        main_step(y);
        main_step(y + 1);
        main_step(y + 2);
      } else {
        halo_step(y);
        halo_step(y + 1);
        halo_step(y + 2);
      }
      y += 2;
      continue;
    }
#endif
    if (warp <= kCsColWarps) {
      const bool act = compute && y <= y1;
      double vq[kCsNC][S];
#ifdef SK_CS_DBG_WAITTOP
      if (t > 0) step_wait(t);
#endif
#ifdef SK_CS_DBG_NOPREF
      if (act && t > 0) {  // operands loaded at the step of use (group t: lines y + 1 / y)
        mb_wait(&mbar[t & 7], (unsigned)(t >> 3) & 1u);
        load_a_ops(y);
      }
#endif
      if (act) {
        double* K0 = Kb + (y & (kCsKR - 1)) * KL;
        const bool wr = inner && y >= y0 && y < y1;
#pragma unroll
        for (int q = 0; q < kCsNC; ++q)
          if (q < nslot) {
            const int ki = (xs[q] - x0 + 1) * S;
            double z[S], v[S], ce[S];
#pragma unroll
            for (int u = 0; u < S; ++u) ce[u] = cce[q][u];
            cs_stencil<S>(sc.scoef, cup[q], ale[q], ce, ari[q], adn[q], z);
#pragma unroll
            for (int u = 0; u < S; ++u) {
              cup[q][u] = ce[u];
              cce[q][u] = adn[q][u];
            }
            norm_row<S>(z, f1s, v);
            if (two) {
#pragma unroll
              for (int u = 0; u < S; ++u) {
                double tmp = 0.0;
#pragma unroll
                for (int w_ = 0; w_ < S; ++w_) tmp = __dadd_rn(tmp, __dmul_rn(abb[q][w_], m0[u * S + w_]));
                v[u] = __dsub_rn(v[u], tmp);
              }
            }
#pragma unroll
            for (int u = 0; u < S; ++u) {
              double tmp = 0.0;
#pragma unroll
              for (int w_ = 0; w_ < S; ++w_) tmp = __dadd_rn(tmp, __dmul_rn(ce[w_], m1[u * S + w_]));
              v[u] = __dsub_rn(v[u], tmp);
            }
            if (!(cv[q] && y >= 0 && y < g)) {
#pragma unroll
              for (int u = 0; u < S; ++u) v[u] = 0.0;
            }
            if (wr) st_row<S>(UK + ((int64_t)y * g + xs[q]) * S, 0, v);
            sw_put<S>(K0 + ki, v);
#pragma unroll
            for (int u = 0; u < S; ++u) vq[q][u] = v[u];
          }
      }
#ifndef SK_CS_DBG_WAITTOP
      if (t > 0) step_wait(t);
#endif
#if SK_CS_V3
      // group t + 3: U_{k-1} line y + 4, U_{k-2} line y + 3 (the slots' last readers, the
      // reducers of step t - 2 included, are done)
      if (issuer && y + 3 <= y1 + 1) issue(t + 3, y + 4, y + 4, y + 3);
#endif
      if (act) {
        const double* K1 = Kb + ((y - 1) & (kCsKR - 1)) * KL;
        double* Z1 = Zs + ((y - 1) & (kCsZR - 1)) * ZL;
        const bool zl = inner && y - 1 >= y0 && y - 1 < y1;
        double kle[kCsNC][S], kri[kCsNC][S];
#pragma unroll
        for (int q = 0; q < kCsNC; ++q)
          if (q < nslot) {
            const int ki = (xs[q] - x0 + 1) * S;
            sw_get<S>(K1 + ki - S, kle[q]);
            sw_get<S>(K1 + ki + S, kri[q]);
          }
#ifndef SK_CS_DBG_NOPREF
        if (y + 1 <= y1) {
          mb_wait(&mbar[(t + 1) & 7], (unsigned)((t + 1) >> 3) & 1u);  // lines y + 2 (U_{k-1}), y + 1 (U_{k-2})
          load_a_ops(y + 1);
        }
#endif
#pragma unroll
        for (int q = 0; q < kCsNC; ++q)
          if (q < nslot) {
            double z2[S];
#pragma unroll
            for (int u = 0; u < S; ++u) {
              double a2 = __dadd_rn(0.0, __dmul_rn(sc.scoef[0], kup[q][u]));
              a2 = __dadd_rn(a2, __dmul_rn(sc.scoef[1], kle[q][u]));
              a2 = __dadd_rn(a2, __dmul_rn(sc.scoef[2], kce[q][u]));
              a2 = __dadd_rn(a2, __dmul_rn(sc.scoef[3], kri[q][u]));
              z2[u] = __dadd_rn(a2, __dmul_rn(sc.scoef[4], vq[q][u]));
              kup[q][u] = kce[q][u];
              kce[q][u] = vq[q][u];
            }
            if (zl) sw_put<S>(Z1 + (xs[q] - x0) * S, z2);
          }
      }
    } else {
      if (t > 0) step_wait(t);
      // group t + 4: U_{k-1} line y + 5, U_{k-2} line y + 4 (consumed from step t + 3 on; the
      // slots' last readers finished step t - 1)
#if !SK_CS_V3
      if (issuer && y + 4 <= y1 + 1) issue(t + 4, y + 5, y + 5, y + 4);
#endif
      const int r = warp - kCsColWarps - 1;
#if SK_CS_NOINLINE_RED
      if (r == 0) {
        const int yl = y - 1;
        if (yl >= y0 && yl < y1)
          cs_reduce_self<S>(Kb + (yl & (kCsKR - 1)) * KL + S, gseg + ((int64_t)yl * nstrip + sx) * NE, lane);
      } else {
        const int yl = y - 2;
#ifdef SK_CS_DBG_SLOT0WAIT
        if (r == 1 && yl >= y0 && yl < y1) { const int j = t - 3 > 0 ? t - 3 : 0; mb_wait(&mbar[j & 7], (unsigned)(j >> 3) & 1u); }
#endif
        if (yl >= y0 && yl < y1)
          cs_reduce_slot<S>(r == 1 ? Ar + (yl & (kCsAR - 1)) * AL + 2 * S : Kb + (yl & (kCsKR - 1)) * KL + S,
                            Zs + (yl & (kCsZR - 1)) * ZL, gseg + ((int64_t)yl * nstrip + sx) * NE + NS + (r - 1) * NB, lane);
      }
#else
      if (r == 0) {
        const int yl = y - 1;
        if (yl >= y0 && yl < y1) {
          const double* K1 = Kb + (yl & (kCsKR - 1)) * KL + S;
          double acc[NS];
#pragma unroll
          for (int e = 0; e < NS; ++e) acc[e] = 0.0;
#pragma unroll 4
          for (int m = 0; m < kLRows; ++m) {
            double vv[S];
            sw_get<S>(K1 + (lane + 32 * m) * S, vv);
            int e = 0;
#pragma unroll
            for (int u = 0; u < S; ++u)
#pragma unroll
              for (int w_ = 0; w_ <= u; ++w_) {
                acc[e] = __dadd_rn(acc[e], __dmul_rn(vv[w_], vv[u]));
                ++e;
              }
          }
#pragma unroll
          for (int e = 0; e < NS; ++e) {
            const double vv = butterfly(acc[e]);
            if (lane == e) gseg[((int64_t)yl * nstrip + sx) * NE + e] = vv;
          }
        }
      } else {
        const int yl = y - 2;
        if (yl >= y0 && yl < y1) {
          const double* src = r == 1 ? Ar + (yl & (kCsAR - 1)) * AL + 2 * S : Kb + (yl & (kCsKR - 1)) * KL + S;
          const double* Z = Zs + (yl & (kCsZR - 1)) * ZL;
          double acc[NB];
#pragma unroll
          for (int e = 0; e < NB; ++e) acc[e] = 0.0;
#pragma unroll 4
          for (int m = 0; m < kLRows; ++m) {
            const int cl = lane + 32 * m;
            double av[S], z[S];
            sw_get<S>(src + cl * S, av);
            sw_get<S>(Z + cl * S, z);
#pragma unroll
            for (int u = 0; u < S; ++u)
#pragma unroll
              for (int w_ = 0; w_ < S; ++w_) acc[u * S + w_] = __dadd_rn(acc[u * S + w_], __dmul_rn(av[w_], z[u]));
          }
#pragma unroll
          for (int e = 0; e < NB; ++e) {
            const double vv = butterfly(acc[e]);
            if (lane == e) gseg[((int64_t)yl * nstrip + sx) * NE + NS + (r - 1) * NB + e] = vv;
          }
        }
      }
#endif
    }
    step_arrive(t);
#ifdef SK_CS_DBG_SYNC
    __syncthreads();
#endif
  }
#else
#ifdef SK_CS_PROF2
  long long pf_wait = 0, pf_work = 0, pf_mb = 0, pf_a = clock64();
#endif
  // steps for lines y0-1 .. y1 (U_k with one halo line each side) + one drain step
  for (int y = ys; y <= y1 + 1; ++y) {
#if SK_CS_TMA
#ifdef SK_CS_PROF2
    const long long pf_m0 = clock64();
#endif
    if (issuer && lane == 0) mb_wait(&mbar[(y - ys) & 7], (unsigned)((y - ys) >> 3) & 1u);
#ifdef SK_CS_PROF2
    pf_mb += clock64() - pf_m0;
#endif
    __syncthreads();
#ifdef SK_CS_PROF2
    const long long pf_b = clock64();
    pf_wait += pf_b - pf_a;
#endif
    // group G(y): U_{k-1} line y + 5, U_{k-2} line y + 4 (consumed at step y + 4;
    // the slots' last readers finished before this step's barrier)
    if (issuer && y + 4 <= y1 + 1) issue(y - ys + 4, y + 5, y + 5, y + 4);
#else
    asm volatile("cp.async.wait_group 3;" ::: "memory");
    __syncthreads();
#endif
    if (warp <= kCsColWarps) {
      if (compute && y <= y1) {
        const double* Am = Ar + ((y - 1) & (kCsAR - 1)) * AL;
        const double* A0 = Ar + (y & (kCsAR - 1)) * AL;
        const double* Ap = Ar + ((y + 1) & (kCsAR - 1)) * AL;
        const double* B0 = Br + (y & (kCsBR - 1)) * BL;
        double* K0 = Kb + (y & (kCsKR - 1)) * KL;
        const double* K1 = Kb + ((y - 1) & (kCsKR - 1)) * KL;
        const double* K2 = Kb + ((y - 2) & (kCsKR - 1)) * KL;
        (void)K2;
        double* Z1 = Zs + ((y - 1) & (kCsZR - 1)) * ZL;
        const bool zl = inner && y - 1 >= y0 && y - 1 < y1;
        const bool wr = inner && y >= y0 && y < y1;
#pragma unroll
        for (int q = 0; q < kCsNC; ++q) {
          if (q < nslot) {
            // branch-free; a point outside the grid (halo line / column) is zeroed
            // after the fact (its stencil sees in-grid neighbours)
            const int ai = (xs[q] - x0 + 2) * S, ki = (xs[q] - x0 + 1) * S;
            double v[S], z2[S];
            {
              double up[S], le[S], ce[S], ri[S];
#if SK_CS_CARRY
#pragma unroll
              for (int t = 0; t < S; ++t) {
                up[t] = kup[q][t];
                ce[t] = kce[q][t];
              }
#else
              sw_get<S>(K2 + ki, up);
              sw_get<S>(K1 + ki, ce);
#endif
              sw_get<S>(K1 + ki - S, le);
              sw_get<S>(K1 + ki + S, ri);
              // z' = op U_k on line y - 1: the first four terms, the down term below
#pragma unroll
              for (int t = 0; t < S; ++t) {
                double a2 = __dadd_rn(0.0, __dmul_rn(sc.scoef[0], up[t]));
                a2 = __dadd_rn(a2, __dmul_rn(sc.scoef[1], le[t]));
                a2 = __dadd_rn(a2, __dmul_rn(sc.scoef[2], ce[t]));
                z2[t] = __dadd_rn(a2, __dmul_rn(sc.scoef[3], ri[t]));
              }
            }
            {
              double up[S], le[S], ce[S], ri[S], dn[S], z[S], bb[S];
#if SK_CS_CARRY
              if (y == ys) {
                sw_get<S>(Am + ai, cup[q]);
                sw_get<S>(A0 + ai, cce[q]);
              }
#pragma unroll
              for (int t = 0; t < S; ++t) {
                up[t] = cup[q][t];
                ce[t] = cce[q][t];
              }
#else
              sw_get<S>(Am + ai, up);
              sw_get<S>(A0 + ai, ce);
#endif
              sw_get<S>(A0 + ai - S, le);
              sw_get<S>(A0 + ai + S, ri);
              sw_get<S>(Ap + ai, dn);
              sw_get<S>(B0 + ai + (BO - 2) * S, bb);
              cs_stencil<S>(sc.scoef, up, le, ce, ri, dn, z);
#if SK_CS_CARRY
#pragma unroll
              for (int t = 0; t < S; ++t) {
                cup[q][t] = ce[t];
                cce[q][t] = dn[t];
              }
#endif
              norm_row<S>(z, f1s, v);
              if (two) {
#pragma unroll
                for (int u = 0; u < S; ++u) {
                  double tmp = 0.0;
#pragma unroll
                  for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(bb[t], m0[u * S + t]));
                  v[u] = __dsub_rn(v[u], tmp);
                }
              }
#pragma unroll
              for (int u = 0; u < S; ++u) {
                double tmp = 0.0;
#pragma unroll
                for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(ce[t], m1[u * S + t]));
                v[u] = __dsub_rn(v[u], tmp);
              }
            }
            if (!(cv[q] && y >= 0 && y < g)) {
#pragma unroll
              for (int t = 0; t < S; ++t) v[t] = 0.0;
            }
            if (wr) st_row<S>(UK + ((int64_t)y * g + xs[q]) * S, 0, v);
            sw_put<S>(K0 + ki, v);
#if SK_CS_CARRY
#pragma unroll
            for (int t = 0; t < S; ++t) {
              kup[q][t] = kce[q][t];
              kce[q][t] = v[t];
            }
#endif
            if (zl) {
#pragma unroll
              for (int t = 0; t < S; ++t) z2[t] = __dadd_rn(z2[t], __dmul_rn(sc.scoef[4], v[t]));
              sw_put<S>(Z1 + (xs[q] - x0) * S, z2);
            }
          }
        }
      }
#if !SK_CS_TMA
      // group G(y): U_{k-1} line y + 5, U_{k-2} line y + 4 (complete at step y + 4)
      if (nslot) copy_a(y + 5);
      if (compute) copy_b(y + 4);
      cs_commit();
#endif
    } else {
      // reducer warps (R1 lane order): self-Gram of line y-1, raw Grams of line y-2
      const int r = warp - kCsColWarps - 1;
#if SK_CS_NOINLINE_RED
      if (r == 0) {
        const int yl = y - 1;
        if (yl >= y0 && yl < y1)
          cs_reduce_self<S>(Kb + (yl & (kCsKR - 1)) * KL + S, gseg + ((int64_t)yl * nstrip + sx) * NE, lane);
      } else if (y - 2 >= y0 && y - 2 < y1) {
        const int yl = y - 2;
        if constexpr (kCsRedWarps == 5) {
          const int slot = (r - 1) >> 1, u = (r - 1) & 1;  // warps 1, 2: slot 0 (U_{k-1}); 3, 4: slot 1 (U_k)
          if (u < S)
            cs_reduce_slot_u<S>(slot == 0 ? Ar + (yl & (kCsAR - 1)) * AL + 2 * S : Kb + (yl & (kCsKR - 1)) * KL + S,
                                Zs + (yl & (kCsZR - 1)) * ZL, u,
                                gseg + ((int64_t)yl * nstrip + sx) * NE + NS + slot * NB + u * S, lane);
        } else {
          cs_reduce_slot<S>(r == 1 ? Ar + (yl & (kCsAR - 1)) * AL + 2 * S : Kb + (yl & (kCsKR - 1)) * KL + S,
                            Zs + (yl & (kCsZR - 1)) * ZL, gseg + ((int64_t)yl * nstrip + sx) * NE + NS + (r - 1) * NB,
                            lane);
        }
      }
      if (true) {  // (the inline loops below are the SK_CS_NOINLINE_RED=0 variant)
      } else if (r == 0) {
#else
      if (r == 0) {
#endif
        const int yl = y - 1;
        if (yl >= y0 && yl < y1) {
          const double* K1 = Kb + (yl & (kCsKR - 1)) * KL + S;
          double acc[NS];
#pragma unroll
          for (int e = 0; e < NS; ++e) acc[e] = 0.0;
#pragma unroll 4
          for (int m = 0; m < kLRows; ++m) {
            double vv[S];
            sw_get<S>(K1 + (lane + 32 * m) * S, vv);
            int e = 0;
#pragma unroll
            for (int u = 0; u < S; ++u)
#pragma unroll
              for (int t = 0; t <= u; ++t) {
                acc[e] = __dadd_rn(acc[e], __dmul_rn(vv[t], vv[u]));
                ++e;
              }
          }
#pragma unroll
          for (int e = 0; e < NS; ++e) {
            const double vv = butterfly(acc[e]);
            if (lane == e) gseg[((int64_t)yl * nstrip + sx) * NE + e] = vv;
          }
        }
      } else {
        const int yl = y - 2;
        if (yl >= y0 && yl < y1) {
          // slot 0: U_{k-1}(yl) . z'(yl); slot 1: U_k(yl) . z'(yl)
          const double* src = r == 1 ? Ar + (yl & (kCsAR - 1)) * AL + 2 * S : Kb + (yl & (kCsKR - 1)) * KL + S;
          const double* Z = Zs + (yl & (kCsZR - 1)) * ZL;
          double acc[NB];
#pragma unroll
          for (int e = 0; e < NB; ++e) acc[e] = 0.0;
#pragma unroll 4
          for (int m = 0; m < kLRows; ++m) {
            const int cl = lane + 32 * m;
            double av[S], z[S];
            sw_get<S>(src + cl * S, av);
            sw_get<S>(Z + cl * S, z);
#pragma unroll
            for (int u = 0; u < S; ++u)
#pragma unroll
              for (int t = 0; t < S; ++t) acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(av[t], z[u]));
          }
#pragma unroll
          for (int e = 0; e < NB; ++e) {
            const double vv = butterfly(acc[e]);
            if (lane == e) gseg[((int64_t)yl * nstrip + sx) * NE + NS + (r - 1) * NB + e] = vv;
          }
        }
      }
    }
#ifdef SK_CS_PROF2
    pf_a = clock64();
    pf_work += pf_a - pf_b;
#endif
  }
#endif  // SK_CS_V2
#if SK_CS_V2
  // every bulk copy issued must have landed before the tail reuses the rings
  if (issuer) {
    const int T = y1 + 2 - ys;
    for (int j = T - 4; j < T; ++j) mb_wait(&mbar[j & 7], (unsigned)(j >> 3) & 1u);
  }
#endif
#if defined(SK_CS_PROF2) && !SK_CS_V2
  if (lane == 0 && blockIdx.x == 5 && side == 0 && (k == 100 || k == 101))
    printf("CSW2 k %lld warp %d steps %d wait %lld (mbarrier %lld) work %lld\n", (long long)k, warp, y1 + 2 - ys,
           pf_wait, pf_mb, pf_work);
#endif
  asm volatile("cp.async.wait_all;" ::: "memory");
  unsigned* ctr = sc.sctr;  // [0..nranges) per range, [nranges] per side
#ifdef SK_CS_PROF
  if (threadIdx.x == 0) g_csprof[blockIdx.y][blockIdx.x][1] = globaltimer();
#endif
  if (!last_cta_arrive(ctr + rg, (unsigned)nstrip)) return;
  // last strip CTA of the range: line nodes (canonical tree over the line's nstrip
  // segment partials) into shared memory, then one node per aligned block of
  // kCsBlk lines to HBM. Both are subtrees of the canonical tree over all segments.
  {
    double* ln = cs_smem;  // [(y1 - y0)][NE]
    const double* gs = gseg + (int64_t)y0 * nstrip * NE;
    const int nitem = (y1 - y0) * NE;
    switch (nstrip) {
      case 1: cs_line_nodes<NE, 1>(gs, nitem, ln); break;
      case 2: cs_line_nodes<NE, 2>(gs, nitem, ln); break;
      case 4: cs_line_nodes<NE, 4>(gs, nitem, ln); break;
      default: cs_line_nodes<NE, 8>(gs, nitem, ln); break;
    }
    __syncthreads();
    const int nb = (y1 - y0) / kCsBlk;
    for (int idx = threadIdx.x; idx < nb * NE; idx += blockDim.x) {
      const int b = idx / NE, e = idx - b * NE;
      double a[kCsBlk];
#pragma unroll
      for (int j = 0; j < kCsBlk; ++j) a[j] = ln[(b * kCsBlk + j) * NE + e];
      lnode[(int64_t)(y0 / kCsBlk + b) * NE + e] = tree_reduce_local(a, kCsBlk);
    }
  }
#ifdef SK_CS_PROF
  __syncthreads();
  if (threadIdx.x == 0) g_csprof[blockIdx.y][blockIdx.x][2] = globaltimer();
#endif
  if (!last_cta_arrive(ctr + nranges, (unsigned)nranges)) return;
  // root: canonical tree over the g / kCsBlk block nodes, one warp per entry:
  // lane l reduces its aligned group of P/32, then pairs of lanes (xor 1, 2, .., 16)
  __shared__ double res[NE];
  if (warp < NE) {
    const int P = g / kCsBlk, per = P / 32;  // g = 512 * 2^j: P >= 64, per = 2^j'
    const double* src = lnode + (int64_t)lane * per * NE + warp;
    double v;
    switch (per) {
      case 2: v = cs_group_tree<2>(src, NE); break;
      case 4: v = cs_group_tree<4>(src, NE); break;
      case 8: v = cs_group_tree<8>(src, NE); break;
      default: v = cs_group_tree<16>(src, NE); break;
    }
#pragma unroll
    for (int d = 1; d <= 16; d <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, d));
    if (lane == 0) res[warp] = v;
  }
  __syncthreads();
#ifdef SK_CS_PROF
  __syncthreads();
  const unsigned long long pft = globaltimer();
#endif
  gram_finish<S>(c, side, res, 0);
  __syncthreads();
  if (st->side[side].stage == ST_GROW_DIRECT) p1_finish<S>(sc, k + 1, res + NS);
#ifdef SK_CS_PROF
  __syncthreads();
  if (threadIdx.x == 0 && (k == 100 || k == 150)) {
    const unsigned long long pend = globaltimer();
    unsigned long long e0 = ~0ull, l0 = ~0ull, l1 = 0, n1 = 0, lsum = 0;
    const int nc = gridDim.x;
    for (int i = 0; i < nc; ++i) {
      const unsigned long long* q = g_csprof[blockIdx.y][i];
      e0 = q[0] < e0 ? q[0] : e0;
      l0 = q[1] < l0 ? q[1] : l0;
      l1 = q[1] > l1 ? q[1] : l1;
      lsum += q[1];
    }
    for (int r = 0; r < nranges; ++r) {
      const unsigned long long* q = g_csprof[blockIdx.y][r * nstrip];
      for (int i = 0; i < nstrip; ++i) {
        const unsigned long long t2 = g_csprof[blockIdx.y][r * nstrip + i][2];
        if (t2 > n1 && t2 >= e0 && t2 < pend) n1 = t2;
      }
      (void)q;
    }
    printf("CSTAIL side %d k %lld ctas %d: loop end min %llu mean %llu max %llu | line nodes done %llu | final tree done %llu | finish done %llu (ns from entry)\n",
           (int)blockIdx.y, (long long)k, nc, l0 - e0, lsum / nc - e0, l1 - e0, n1 - e0, pft - e0, pend - e0);
  }
#endif
}

// Clean-up Gram (rare path): each CTA sweeps all blocks for its row group, so
// the no-op launch stays one CTA per row group.
template <int S>
__global__ void __launch_bounds__(256) k_gram_loop(const __grid_constant__ SolveConst c) {
  constexpr int NB = S * S;
  const int side = blockIdx.z;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.stage != ST_NEED_CLEANUP) return;
  const SideConst& sc = c.side[side];
  const int64_t cta = blockIdx.x;
  if (cta >= sc.ncta) return;
  const int64_t k = ss.blocks;
  const double* __restrict__ x = sc.blocks[k];
  const int lane = threadIdx.x & 31;
  const int64_t n = sc.n;
  const SegGeom g = seg_geom(cta, sc.nseg);
  for (int64_t b = 0; b < k; ++b) {
    const double* __restrict__ ub = sc.blocks[b];
    OwnerVals<NB> segv[kSegsPerWarp];
    for (int q = 0; q < kSegsPerWarp; ++q) {
      double acc[NB];
#pragma unroll
      for (int e = 0; e < NB; ++e) acc[e] = 0.0;
      if (q < g.nvalid_warp) {
        const int64_t base = (g.seg_w0 + q) * kSeg;
        for (int m = 0; m < kLRows; ++m) {
          const int64_t i = base + lane + 32 * m;
          if (i < n) {
            double a[S], y[S];
            ld_raw<S>(ub, i, a);
#pragma unroll
            for (int t = 0; t < S; ++t) y[t] = x[i * S + t];
#pragma unroll
            for (int u = 0; u < S; ++u)
#pragma unroll
              for (int t = 0; t < S; ++t) acc[u * S + t] = __dadd_rn(acc[u * S + t], __dmul_rn(a[t], y[u]));
          }
        }
      }
      seg_butterfly<NB>(acc, segv[q], lane);
    }
    cta_combine<NB>(segv, g.nvalid_warp, g.nvalid_cta, sc.part + (b * sc.ncta + cta) * NB);
    __syncthreads();
  }
  if (!last_cta_arrive(sc.counter + 2, (unsigned)sc.ncta)) return;
  if (sc.dist) {
    for (int64_t b = 0; b < k; ++b)
      dist_emit<NB>(c, side, b, sc.part + b * sc.ncta * NB, sc.ncta, sc.chunk_g, sc.part + k * sc.ncta * NB);
    return;
  }
  for (int64_t b = threadIdx.x; b < k; b += blockDim.x) {
    double G[NB], cb[NB], mb[NB];
    for (int e = 0; e < NB; ++e) G[e] = tree_stream(sc.part + b * sc.ncta * NB + e, sc.ncta, NB);
    block_coefs(sc.nfac + b * (NB + S), G, S, cb, mb);
    for (int e = 0; e < NB; ++e) {
      sc.coef2[b * NB + e] = cb[e];
      sc.mcoef2[b * NB + e] = mb[e];
    }
  }
}

// =====================================================================
// Arnoldi update (many blocks): one thread per row carrying its S column
// chains, y(i,u) = x(i,u) - sum_b [sum_t U_b(i,t) M_b(t,u)] in ascending b
// (same arithmetic per chain as k_update); M and the block pointers staged in
// smem per chunk, 8 block rows in flight per thread.
// =====================================================================
constexpr int kArnThreads = 128;
__device__ __forceinline__ const double* blk_ptr(const SideConst& sc, int64_t b) {
  return reinterpret_cast<const double*>(__ldg(reinterpret_cast<const unsigned long long*>(sc.blocks) + b));
}
template <int S>
__global__ void __launch_bounds__(kArnThreads) k_arn_update(const __grid_constant__ SolveConst c, int mode) {
  constexpr int UN = S <= 2 ? 8 : (S <= 4 ? 4 : 2);   // block rows in flight (registers: 2*UN*S)
  constexpr int CH = (S <= 2 ? 1024 : 4096 / (S * S));  // M chunk (blocks), multiple of UN
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.exhausted || ss.broken) return;
  const SideConst& sc = c.side[side];
  const int64_t k = ss.blocks;
  const double* xin = mode == UM_FIRST ? sc.w : sc.wx;
  double* xout = mode == UM_FIRST ? sc.wx : sc.blocks[k];
  const double* mc = mode == UM_FIRST ? sc.mcoef : sc.mcoef2;
  const int64_t b0 = mode == UM_FIRST ? first_block(c, k) : 0, b1 = k;
  const int64_t n = sc.n;
  if ((int64_t)blockIdx.x * blockDim.x >= n) return;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = g < n;
  const int64_t i = active ? g : n - 1;
  __shared__ double Ms[CH * S * S];
  double y[S];
  ld_raw_cg<S>(xin, i, y);
  double cur[UN][S], nxt[UN][S];
#pragma unroll
  for (int q = 0; q < UN; ++q)
    if (b0 + q < b1) ld_raw<S>(blk_ptr(sc, b0 + q), i, cur[q]);
  int64_t cb = b0 - CH;  // chunk base of the staged M
  for (int64_t bb = b0; bb < b1; bb += UN) {
    if (bb >= cb + CH) {  // restage M (uniform across the CTA)
      cb = bb;
      const int nb = (int)mn64(CH, b1 - cb);
      __syncthreads();
      for (int e = threadIdx.x; e < nb * S * S; e += blockDim.x) Ms[e] = __ldcg(mc + cb * S * S + e);
      __syncthreads();
    }
    // prefetch the next group while this one computes
#pragma unroll
    for (int q = 0; q < UN; ++q)
      if (bb + UN + q < b1) ld_raw<S>(blk_ptr(sc, bb + UN + q), i, nxt[q]);
    const double* m = Ms + (bb - cb) * S * S;
#pragma unroll
    for (int q = 0; q < UN; ++q) {
      if (bb + q < b1) {
#pragma unroll
        for (int u = 0; u < S; ++u) {
          double tmp = 0.0;
#pragma unroll
          for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(cur[q][t], m[q * S * S + u * S + t]));
          y[u] = __dsub_rn(y[u], tmp);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < UN; ++q)
#pragma unroll
      for (int t = 0; t < S; ++t) cur[q][t] = nxt[q][t];
  }
  if (active) st_row<S>(xout, i, y);
}

// R1 self Gram x^T x of the candidate U_k (one warp per segment) + finalise.
template <int S>
__global__ void __launch_bounds__(kFusedThreads) k_self_gram(const __grid_constant__ SolveConst c, int mode) {
  constexpr int NS = S * (S + 1) / 2;
  const int side = blockIdx.z;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  if (ss.exhausted || ss.broken) return;
  const SideConst& sc = c.side[side];
  const int64_t nseg = sc.nseg;
  const int64_t ncta = (nseg + kFusedSegsPerCta - 1) / kFusedSegsPerCta;
  const int64_t cta = blockIdx.x;
  if (cta >= ncta) return;
  const double* __restrict__ x = sc.blocks[ss.blocks];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t seg = cta * kFusedSegsPerCta + warp;
  const int nvalid_cta = (int)mn64(kFusedSegsPerCta, nseg - cta * kFusedSegsPerCta);
  double acc[NS];
#pragma unroll
  for (int e = 0; e < NS; ++e) acc[e] = 0.0;
  if (seg < nseg) {
    const int64_t base = seg * kSeg;
#pragma unroll 4
    for (int m = 0; m < kLRows; ++m) {
      const int64_t i = base + lane + 32 * m;
      if (i < sc.n) {
        double y[S];
        ld_raw_cg<S>(x, i, y);
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
  warp_seg_to_cta<NS>(acc, nvalid_cta, sc.part + cta * NS);
  if (!last_cta_arrive(sc.counter + 1, (unsigned)ncta)) return;
  __shared__ double res[NS];
  final_tree<NS>(sc.part, ncta, res, sc.part + ncta * NS);
  SideState& sst = c.st->side[side];
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    int t, u;
    unpack_tri(e, t, u);
    sst.gbase[u * S + t] = res[e];
    sst.gbase[t * S + u] = res[e];
  }
  __syncthreads();
  if (c.arnoldi) {
    __shared__ double sbuf[1024];
    const double c2 = block_tree(sc.hsq, sst.blocks, sbuf);
    if (threadIdx.x == 0) {
      sst.coeff2 = c2;
      sst.pad = 1;  // coeff2 precomputed for this step
    }
  }
  if (threadIdx.x == 0) finalize_direct(c, side, true, c.st->side[side]);
  (void)mode;
}

// =====================================================================
// x_out = x_in - sum_{b in [b0,b1)} U_b M_b (+ R1 Gram of x_out, finalise)
// =====================================================================

template <int S>
__global__ void __launch_bounds__(256) k_update(const __grid_constant__ SolveConst c, int mode) {
  constexpr int NS = S * (S + 1) / 2;
  const int side = blockIdx.z;
  if (side >= c.nsides) return;
  const DevState* st = c.st;
  if (mode != UM_INIT && st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  const SideConst& sc = c.side[side];
  const int64_t k = ss.blocks;
  const double* xin;
  const double* mc = sc.mcoef;
  double* xout;
  int64_t b0 = 0, b1 = 0;
  bool gram = true;
  switch (mode) {
    case UM_LANCZOS:
      if (ss.exhausted || ss.broken) return;
      xin = sc.w;
      xout = sc.blocks[k];
      b0 = first_block(c, k);
      b1 = k;
      break;
    case UM_FIRST:
      if (ss.exhausted || ss.broken) return;
      xin = sc.w;
      xout = sc.wx;
      b0 = first_block(c, k);
      b1 = k;
      gram = false;
      break;
    case UM_SECOND:
      if (ss.exhausted || ss.broken) return;
      xin = sc.wx;
      xout = sc.blocks[k];
      mc = sc.mcoef2;
      b0 = 0;
      b1 = k;
      break;
    case UM_CLEAN:
      if (ss.stage != ST_NEED_CLEANUP) return;
      xin = sc.blocks[k];
      xout = sc.blocks[k];
      mc = sc.mcoef2;
      b0 = 0;
      b1 = k;
      break;
    default:  // UM_INIT: U_0 = transposed C
      xin = sc.wx;
      xout = sc.blocks[0];
      break;
  }
  const int64_t cta = blockIdx.x;
  if (cta >= sc.ncta) return;
  const int lane = threadIdx.x & 31;
  const int64_t n = sc.n;
  const SegGeom g = seg_geom(cta, sc.nseg);

  OwnerVals<NS> segv[kSegsPerWarp];
#pragma unroll 1
  for (int q = 0; q < kSegsPerWarp; ++q) {
    double acc[NS];
#pragma unroll
    for (int e = 0; e < NS; ++e) acc[e] = 0.0;
    if (q < g.nvalid_warp) {
      const int64_t base = (g.seg_w0 + q) * kSeg;
#pragma unroll 2
      for (int m = 0; m < kLRows; ++m) {
        const int64_t i = base + lane + 32 * m;
        if (i < n) {
          double y[S];
          ld_raw_cg<S>(xin, i, y);
          for (int64_t b = b0; b < b1; ++b) {
            double a[S];
            ld_raw<S>(sc.blocks[b], i, a);
            const double* mb = mc + b * (S * S);
#pragma unroll
            for (int u = 0; u < S; ++u) {
              double tmp = 0.0;
#pragma unroll
              for (int t = 0; t < S; ++t) tmp = __dadd_rn(tmp, __dmul_rn(a[t], __ldg(mb + u * S + t)));
              y[u] = __dsub_rn(y[u], tmp);
            }
          }
          st_row<S>(xout, i, y);
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
  if (!gram) return;
  cta_combine<NS>(segv, g.nvalid_warp, g.nvalid_cta, sc.part + cta * NS);
  if (!last_cta_arrive(sc.counter + 1, (unsigned)sc.ncta)) return;
  if (sc.dist) {
    dist_emit<NS>(c, side, 0, sc.part, sc.ncta, sc.chunk_g, sc.part + sc.ncta * NS);
    return;
  }
  __shared__ double res[NS];
  for (int e = threadIdx.x; e < NS; e += blockDim.x) res[e] = tree_stream(sc.part + e, sc.ncta, NS);
  __syncthreads();
  gram_finish<S>(c, side, res, mode == UM_INIT ? 2 : (mode == UM_CLEAN ? 1 : 0));
}

// =====================================================================
// Rare path: single-CTA Householder QR (decompositions.cpp:16-78 with R1 dots)
// =====================================================================
static __device__ double cta_r1_dot(const double* x, int sx, int cx, const double* y, int sy, int cy,
                                    int64_t n, int64_t row0, double* segbuf) {
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

// which: 0 first-pass NEED_HH, 1 NEED_HH2 after clean-up, 2 init (U_0)
template <int S>
__global__ void __launch_bounds__(1024) k_householder(const __grid_constant__ SolveConst c, int which) {
  const int side = blockIdx.x;
  if (side >= c.nsides) return;
  if (which != 2 && c.st->status != RUNNING) return;
  SideState& st = c.st->side[side];
  const int want = which == 0 ? ST_NEED_HH : (which == 1 ? ST_NEED_HH2 : ST_INIT_HH);
  if (st.stage != want) return;
  const SideConst& sc = c.side[side];
  const int64_t k = which == 2 ? 0 : st.blocks;
  double* cand = sc.blocks[k];
  for (int64_t i = threadIdx.x; i < sc.n * S; i += blockDim.x) sc.hw[i] = cand[i];
  __syncthreads();
  __shared__ double R[kMaxS * kMaxS];
  householder_cta<S>(sc.hw, sc.qh, sc.n, R, sc.part);
  __shared__ int accept;
  if (threadIdx.x == 0) {
    for (int e = 0; e < S * S; ++e) st.R[e] = R[e];
    jacobi_extremes(st.R, S, S, &st.smax, &st.smin);
    if (which == 2) {
      set_nfac(sc, 0, S, st.R, true);
      accept = 1;
    } else {
      if (which == 0) st.paths[1]++;
      classify(c, side, which == 0, ST_GROW_HH, c.st->side[side]);
      accept = st.stage == ST_GROW_HH;
    }
  }
  __syncthreads();
  if (accept)
    for (int64_t i = threadIdx.x; i < sc.n * S; i += blockDim.x) cand[i] = sc.qh[i];
}

// =====================================================================
// Initialisation (block_krylov.cpp:27-52; factorized_solvers.cpp:121-131)
// =====================================================================
template <int S>
__global__ void k_init_transpose(const __grid_constant__ SolveConst c, const double* c1, const double* c2) {
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const SideConst& sc = c.side[side];
  const double* src = side == 0 ? c1 : c2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < sc.n;
       i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int u = 0; u < S; ++u) sc.wx[i * S + u] = src[u * sc.n + i];
}

// R_0 = R_L R_R^T, P_0 = R_0, rho_0 = <R_0,R_0> (R2 contract, one tile)
static __global__ void k_core_init(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  const int s = c.s;
  if (threadIdx.x != 0) return;
  const SideState& a = st->side[0];
  const SideState& b = st->side[c.nsides > 1 ? 1 : 0];
  for (int sd = 0; sd < c.nsides; ++sd) {
    const SideState& x = st->side[sd];
    if (x.smin < __dmul_rn(1e-12, x.smax) || x.smax == 0.0) {
      st->status = RANKDEF;
      return;
    }
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
  double lane[32];
  for (int l = 0; l < 32; ++l) {
    double acc = 0.0;
    if (l < s)
      for (int j = 0; j < s; ++j) acc = __dadd_rn(acc, __dmul_rn(c.R[j * c.ld + l], c.R[j * c.ld + l]));
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
__device__ __forceinline__ double band_at(const double* hband, int s, int64_t i, int64_t l) {
  const int64_t bi = i / s, bl = l / s;
  const int64_t d = bi - bl + 1;
  return hband[(bl * 3 + d) * (s * s) + (l % s) * s + (i % s)];
}

template <int S>
struct CgTile {
  static constexpr int H = 2 * S;
  static constexpr int D = kTile + 2 * H;
};

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

__device__ __forceinline__ double tile_reduce(const double* f, int nrows, int ncols) {
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  if (lane < nrows)
    for (int cc = 0; cc < ncols; ++cc) acc = __dadd_rn(acc, f[cc * kTile + lane]);
  return butterfly(acc);
}

// Canonical pairwise tree over the cnt (<= 32) values held by lanes 0..cnt-1:
// strides 1, 2, 4, ..., a node without a right child passes through.
__device__ __forceinline__ double warp_tree(double v, int cnt) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double o = __shfl_down_sync(0xffffffffu, v, d);
    if ((lane & (2 * d - 1)) == 0 && lane + d < cnt) v = __dadd_rn(v, o);
  }
  return __shfl_sync(0xffffffffu, v, 0);
}
// canonical tree over a[0..n) (stride st) by one warp: aligned groups of 32,
// then the group nodes. GLOBAL: a[] was written by other CTAs (L2 loads);
// otherwise a[] may be shared memory (generic loads).
template <bool GLOBAL>
static __device__ double warp_tree_n(const double* a, int64_t n, int64_t st) {
  const int lane = threadIdx.x & 31;
  auto ld = [&](int64_t i) { return GLOBAL ? __ldcg(a + i * st) : a[i * st]; };
  if (n <= 32) return warp_tree(lane < n ? ld(lane) : 0.0, (int)n);
  const int64_t ng = (n + 31) / 32;
  if (ng <= 32) {
    double node = 0.0;
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t idx = g * 32 + lane;
      const double t = warp_tree(idx < n ? ld(idx) : 0.0, (int)mn64(32, n - g * 32));
      if (lane == g) node = t;
    }
    return warp_tree(node, (int)ng);
  }
  // > 1024 values (not reached for core tiles, r <= 32768): one lane streams
  double v = 0.0;
  if (lane == 0) {
    TreeStream ts;
    ts.init();
    for (int64_t i = 0; i < n; ++i) ts.push(ld(i));
    v = ts.finish();
  }
  return __shfl_sync(0xffffffffu, v, 0);
}
// R2 root: per tile column a canonical tree over its row tiles, then over the
// columns (one warp per column, then one warp over the column nodes)
static __device__ double r2_final(const double* part, int64_t nti, int64_t ntj, double* scratch) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int64_t tj = warp; tj < ntj; tj += nw) {
    const double v = warp_tree_n<true>(part + tj * nti, nti, 1);
    if (lane == 0) scratch[tj] = v;
  }
  __threadfence_block();
  __syncthreads();
  __shared__ double res;
  if (warp == 0) {
    const double v = warp_tree_n<false>(scratch, ntj, 1);
    if (lane == 0) res = v;
  }
  __syncthreads();
  return res;
}

__device__ inline bool any_side_broken(const SolveConst& c) {
  for (int s = 0; s < c.nsides; ++s)
    if (c.st->side[s].broken) return true;
  return false;
}

// ---- CG core tiles (K4) ----
// A CTA owns one 32x32 tile of the core. It stages P with a halo of 2S rows /
// columns, the H-band coefficients of its 32 rows and the G-band coefficients
// of its 32 columns in shared memory (32-bit tile-local indexing), then every
// entry forms image(P)(i,j) = sum_jb [sum_t H(i,l) P(l,j)] + sum_jb [sum_t P(i,l)
// G(j,l)] in exactly image_at's order (jb ascending, t ascending, one partial
// per band block).
template <int S>
struct CoreSmem {
  static constexpr int H = CgTile<S>::H, D = CgTile<S>::D;
  double sp[D * D];
  double hc[3 * S][kTile];  // H(i0+li, (bi-1)S + q)
  double gc[3 * S][kTile];  // G(j0+lj, (bj-1)S + q)
  // tile products f (kTile^2) reuse sp once every entry is formed
  int hlo[kTile], hhi[kTile], glo[kTile], ghi[kTile];  // valid band blocks (absolute)
};
template <int S>
__device__ void stage_bands(CoreSmem<S>& sm, const double* hv, const double* hw, int i0, int j0, int pr,
                            int pc) {
  const int JBr = pr / S, JBc = pc / S;
  for (int idx = threadIdx.x; idx < 3 * S * kTile; idx += blockDim.x) {
    const int q = idx / kTile, li = idx % kTile;
    {
      const int i = i0 + li, bi = i / S;
      const int lo = bi - 1 > 0 ? bi - 1 : 0, hi = bi + 1 < JBr - 1 ? bi + 1 : JBr - 1;
      const int jb = bi - 1 + q / S;
      sm.hc[q][li] = (jb >= lo && jb <= hi) ? band_at(hv, S, i, (int64_t)jb * S + q % S) : 0.0;
      if (q == 0) {
        sm.hlo[li] = lo;
        sm.hhi[li] = hi;
      }
    }
    {
      const int j = j0 + li, bj = j / S;
      const int lo = bj - 1 > 0 ? bj - 1 : 0, hi = bj + 1 < JBc - 1 ? bj + 1 : JBc - 1;
      const int jb = bj - 1 + q / S;
      sm.gc[q][li] = (jb >= lo && jb <= hi) ? band_at(hw, S, j, (int64_t)jb * S + q % S) : 0.0;
      if (q == 0) {
        sm.glo[li] = lo;
        sm.ghi[li] = hi;
      }
    }
  }
}
// image(P) at tile-local (li, lj); i = i0 + li < rows of the window, j = j0 + lj
template <int S>
__device__ __forceinline__ double core_image(const CoreSmem<S>& sm, int li, int lj, int i0, int j0, int pr, int pc) {
  constexpr int H = CgTile<S>::H, D = CgTile<S>::D;
  const int i = i0 + li, j = j0 + lj;
  const bool hasH = j < pc, hasG = i < pr;
  double hpart = 0.0, gpart = 0.0;
  if (hasH) {
    const int bi = i / S, lo = sm.hlo[li], hi = sm.hhi[li];
    const double* pcol = sm.sp + (lj + H) * D + H - i0;  // pcol[l] = P(l, j)
#pragma unroll
    for (int qb = 0; qb < 3; ++qb) {
      const int jb = bi - 1 + qb;
      if (jb >= lo && jb <= hi) {
        double d = 0.0;
#pragma unroll
        for (int t = 0; t < S; ++t) d = __dadd_rn(d, __dmul_rn(sm.hc[qb * S + t][li], pcol[jb * S + t]));
        hpart = __dadd_rn(hpart, d);
      }
    }
  }
  if (hasG) {
    const int bj = j / S, lo = sm.glo[lj], hi = sm.ghi[lj];
    const double* prow = sm.sp + (li + H) + (H - j0) * D;  // prow[l * D] = P(i, l)
#pragma unroll
    for (int qb = 0; qb < 3; ++qb) {
      const int jb = bj - 1 + qb;
      if (jb >= lo && jb <= hi) {
        double d = 0.0;
#pragma unroll
        for (int t = 0; t < S; ++t) d = __dadd_rn(d, __dmul_rn(prow[(jb * S + t) * D], sm.gc[qb * S + t][lj]));
        gpart = __dadd_rn(gpart, d);
      }
    }
  }
  if (hasH && hasG) return __dadd_rn(hpart, gpart);
  return hasH ? hpart : (hasG ? gpart : 0.0);
}
template <int S>
__device__ void stage_p32(CoreSmem<S>& sm, const SolveConst& c, int i0, int j0, int rows_p, int cols_p, int mode,
                          const double* Pprev, const double* Pcur, double beta, bool first) {
  constexpr int H = CgTile<S>::H, D = CgTile<S>::D;
  const int64_t ld = c.ld;
  for (int idx = threadIdx.x; idx < D * D; idx += blockDim.x) {
    const int li = idx % D, lj = idx / D;
    const int i = i0 - H + li, j = j0 - H + lj;
    double v = 0.0;
    if (i >= 0 && j >= 0 && i < rows_p && j < cols_p) {
      const int64_t o = (int64_t)j * ld + i;
      if (mode == 1)
        v = Pcur[o];
      else if (first)
        v = c.R[o];
      else
        v = __dadd_rn(c.R[o], __dmul_rn(beta, Pprev[o]));
    }
    sm.sp[idx] = v;
  }
}
// R2 root with the reduction spread over the tile columns: the last CTA of a
// column reduces that column's tile partials (canonical tree over tile rows),
// the last column to finish reduces the column nodes. True in exactly one CTA.
static __device__ bool r2_columns(const SolveConst& c, int64_t nti, int64_t ntj, int64_t tj, double* root) {
  unsigned int* colctr = c.ccounter + 8;
  double* colnode = c.cpart + nti * ntj;
  if (!last_cta_arrive(colctr + tj, (unsigned)nti)) return false;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const double v = warp_tree_n<true>(c.cpart + tj * nti, nti, 1);
    if (lane == 0) colnode[tj] = v;
  }
  if (!last_cta_arrive(c.ccounter + 0, (unsigned)ntj)) return false;
  __shared__ double res;
  if (warp == 0) {
    const double v = warp_tree_n<true>(colnode, ntj, 1);
    if (lane == 0) res = v;
  }
  __syncthreads();
  *root = res;
  return true;
}

template <int S>
__global__ void __launch_bounds__(256) k_cg_a(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  // pause check (was a kernel of its own, ~4 us per iteration): an extension that asked for a
  // rare path (Householder / clean-up) stops the run here; every CTA takes the same decision
  // from the stages the extension kernel left, one thread publishes it. The host sees PAUSED
  // in the status ring, runs the rare kernels and resumes (sk_driver.cu).
  {
    bool need = false;
    for (int sd = 0; sd < c.nsides; ++sd) {
      const int g = st->side[sd].stage;
      need = need || g == ST_NEED_HH || g == ST_NEED_CLEANUP;
    }
    if (need) {
      if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) st->status = PAUSED;
      return;
    }
  }
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
  const int rows_p = (int)st->rows_p, cols_p = (int)st->cols_p;
  const int64_t nti = (rows_p + kTile - 1) / kTile, ntj = (cols_p + kTile - 1) / kTile;
  const int64_t ti = blockIdx.x, tj = blockIdx.y;
  if (ti >= nti || tj >= ntj) return;
  if (ti == 0 && tj == 0 && threadIdx.x == 0) c.hist_tk[k + 1] = (double)globaltimer();
  constexpr int H = CgTile<S>::H, D = CgTile<S>::D;
  __shared__ CoreSmem<S> sm;
  const int i0 = (int)ti * kTile, j0 = (int)tj * kTile;
  const double* Pprev = c.P[(k + 1) & 1];
  double* Pnew = c.P[k & 1];
  const SideConst& sv = c.side[0];
  const SideConst& sw = c.side[c.nsides > 1 ? 1 : 0];
  stage_p32<S>(sm, c, i0, j0, rows_p, cols_p, 0, Pprev, nullptr, st->beta, k == 0);
  stage_bands<S>(sm, sv.hband, sw.hband, i0, j0, rows_p, cols_p);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = i0 + lane;
  const int64_t ld = c.ld;
  double fv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int lc = warp * 4 + q;
    const int j = j0 + lc;
    fv[q] = 0.0;
    if (i < rows_p && j < cols_p) {
      const double pv = sm.sp[(lc + H) * D + (lane + H)];
      Pnew[(int64_t)j * ld + i] = pv;
      const double qv = core_image<S>(sm, lane, lc, i0, j0, rows_p, cols_p);
      fv[q] = __dmul_rn(c.R[(int64_t)j * ld + i], qv);
    }
  }
  __syncthreads();
  double* f = sm.sp;
#pragma unroll
  for (int q = 0; q < 4; ++q) f[(warp * 4 + q) * kTile + lane] = fv[q];
  __syncthreads();
  if (warp == 0) {
    const int nr = (int)mn64(kTile, rows_p - i0), nc = (int)mn64(kTile, cols_p - j0);
    const double v = tile_reduce(f, nr, nc);
    if (lane == 0) c.cpart[tj * nti + ti] = v;
  }
  double denom;
  if (!r2_columns(c, nti, ntj, tj, &denom)) return;
  if (threadIdx.x == 0) {
    st->denom = denom;
    if (fabs(denom) < __dmul_rn(c.tol, st->rho)) {  // factorized_solvers.cpp:155-160
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
__global__ void __launch_bounds__(256) k_cg_b(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int64_t k = st->k;
  const int rows_p = (int)st->rows_p, cols_p = (int)st->cols_p;
  const int rows_q = (int)st->rows_q, cols_q = (int)st->cols_q;
  const int64_t nti = (rows_q + kTile - 1) / kTile, ntj = (cols_q + kTile - 1) / kTile;
  const int64_t ti = blockIdx.x, tj = blockIdx.y;
  if (ti >= nti || tj >= ntj) return;
  constexpr int D = CgTile<S>::D, H = CgTile<S>::H;
  __shared__ CoreSmem<S> sm;
  const int i0 = (int)ti * kTile, j0 = (int)tj * kTile;
  const double* Pcur = c.P[k & 1];
  const SideConst& sv = c.side[0];
  const SideConst& sw = c.side[c.nsides > 1 ? 1 : 0];
  stage_p32<S>(sm, c, i0, j0, rows_p, cols_p, 1, nullptr, Pcur, 0.0, false);
  stage_bands<S>(sm, sv.hband, sw.hband, i0, j0, rows_p, cols_p);
  __syncthreads();
  const double alpha = st->alpha, nalpha = -alpha;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = i0 + lane;
  const int64_t ld = c.ld;
  double fv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int lc = warp * 4 + q;
    const int j = j0 + lc;
    fv[q] = 0.0;
    if (i < rows_q && j < cols_q) {
      const double qv = core_image<S>(sm, lane, lc, i0, j0, rows_p, cols_p);
      const int64_t o = (int64_t)j * ld + i;
      const bool inp = i < rows_p && j < cols_p;
      const double remb = inp ? c.R[o] : 0.0;
      const double rn = __dadd_rn(remb, __dmul_rn(nalpha, qv));
      c.R[o] = rn;
      fv[q] = __dmul_rn(rn, rn);
      if (inp) {
        const double pv = sm.sp[(lc + H) * D + (lane + H)];
        c.X[o] = __dadd_rn(c.X[o], __dmul_rn(alpha, pv));
      }
    }
  }
  __syncthreads();
  double* f = sm.sp;
#pragma unroll
  for (int q = 0; q < 4; ++q) f[(warp * 4 + q) * kTile + lane] = fv[q];
  __syncthreads();
  if (warp == 0) {
    const int nr = (int)mn64(kTile, rows_q - i0), nc = (int)mn64(kTile, cols_q - j0);
    const double v = tile_reduce(f, nr, nc);
    if (lane == 0) c.cpart[tj * nti + ti] = v;
  }
  double rho_next;
  if (!r2_columns(c, nti, ntj, tj, &rho_next)) return;
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
    if (norm_r <= __dmul_rn(st->norm_r0, c.eps)) {  // factorized_solvers.cpp:173-178
      st->status = CONVERGED;
      return;
    }
    st->beta = __ddiv_rn(rho_next, st->rho);
    st->rho = rho_next;
    if (st->k >= c.max_iter) st->status = MAXITER;
  }
}

// =====================================================================
// standalone kernels: SpMM (parity tests), export with normalisation
// =====================================================================
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
template <int S>
__global__ void k_export_block(const double* blk, const double* nfac, int64_t b, double* out, int64_t n) {
  NF<S> f;
  load_nf<S>(nfac, b, f);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double q[S];
    load_vrow<S>(blk, f, i, q);
#pragma unroll
    for (int u = 0; u < S; ++u) out[u * n + i] = q[u];
  }
}

// =====================================================================
// Row partition: finalisation from the all-gathered chunk nodes (one CTA per
// side; the guards are those of the last CTA it replaces), the pause that hands
// a rare path to the host, and the halo exchange staging of the newest block.
// =====================================================================
enum DistFin : int { DF_P1 = 0, DF_P2 = 1, DF_CGRAM = 2, DF_CSELF = 3 };
template <int S>
__global__ void __launch_bounds__(256) k_dist_fin(const __grid_constant__ SolveConst c, int mode, int64_t msg) {
  constexpr int NB = S * S, NE = 2 * NB, NS = S * (S + 1) / 2;
  const int side = blockIdx.x;
  if (side >= c.nsides) return;
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const SideState& ss = st->side[side];
  const SideConst& sc = c.side[side];
  const int64_t k = ss.blocks;
  if (mode == DF_P1 || mode == DF_P2) {
    if (ss.exhausted || ss.broken) return;
  } else if (ss.stage != ST_NEED_CLEANUP) {
    return;
  }
  __shared__ double res[NE];
  if (mode == DF_P1) {
    dist_root<NE>(c, side, 0, msg, res);
    p1_finish<S>(sc, k, res);
  } else if (mode == DF_P2 || mode == DF_CSELF) {
    dist_root<NS>(c, side, 0, msg, res);
    gram_finish<S>(c, side, res, mode == DF_CSELF ? 1 : 0);
  } else {
    for (int64_t b = threadIdx.x; b < k; b += blockDim.x) {
      double G[NB], cb[NB], mb[NB];
      for (int e = 0; e < NB; ++e) {
        TreeStream ts;
        ts.init();
        for (int r = 0; r < c.world; ++r) {
          const double* base = c.gnodes + r * msg + node_off(c, b, side, 0) + e;
          for (int j = 0; j < c.rank_nch[side * c.world + r]; ++j) ts.push(__ldcg(base + (int64_t)j * c.nex));
        }
        G[e] = ts.finish();
      }
      block_coefs(sc.nfac + b * (NB + S), G, S, cb, mb);
      for (int e = 0; e < NB; ++e) {
        sc.coef2[b * NB + e] = cb[e];
        sc.mcoef2[b * NB + e] = mb[e];
      }
    }
  }
}

// newest block's first / last `halo` local rows -> hsend (lo | hi)
template <int S>
__global__ void k_halo_pack(const __grid_constant__ SolveConst c) {
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const SideConst& sc = c.side[side];
  const int64_t H = sc.halo;
  const int64_t kb = c.st->side[side].blocks;
  if (H == 0 || kb < 1) return;
  const double* src = sc.blocks[kb - 1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < H * S; e += (int64_t)gridDim.x * blockDim.x) {
    sc.hsend[e] = src[e];
    sc.hsend[H * S + e] = src[(sc.n - H) * S + e];
  }
}
// hrecv (from previous | next rank) -> ghost rows of the newest block
template <int S>
__global__ void k_halo_unpack(const __grid_constant__ SolveConst c) {
  const int side = blockIdx.y;
  if (side >= c.nsides) return;
  const SideConst& sc = c.side[side];
  const int64_t H = sc.halo;
  const int64_t kb = c.st->side[side].blocks;
  if (H == 0 || kb < 1) return;
  double* dst = sc.blocks[kb - 1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < H * S; e += (int64_t)gridDim.x * blockDim.x) {
    if (c.rank > 0) dst[e - H * S] = sc.hrecv[e];
    if (c.rank < c.world - 1) dst[sc.n * S + e] = sc.hrecv[H * S + e];
  }
}

static int host_row_mode(const SideConst& sc) {
  if (sc.sdim == 0) return 0;
  return sc.sdim + (sc.sg_pow2 >= 0 ? 10 : 0);
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

// ---- per-S launchers (explicitly instantiated, one translation unit per S) ----
#ifdef SK_INST_COMMON
template <int S>
struct Launch {
  static void init(const SolveConst& c, const double* dc1, const double* dc2, cudaStream_t st);
  static void spmm(const SolveConst& c, cudaStream_t st);
  static void gram(const SolveConst& c, int mode, int64_t nblk, cudaStream_t st);
  static void update(const SolveConst& c, int mode, cudaStream_t st);
  static void householder(const SolveConst& c, int which, cudaStream_t st);
  static void arn_update(const SolveConst& c, int mode, cudaStream_t st);
  static void self_gram(const SolveConst& c, cudaStream_t st);
  static void lanczos_p1(const SolveConst& c, cudaStream_t st);
  static void lanczos_p2(const SolveConst& c, cudaStream_t st);
  static void lanczos_sweep(const SolveConst& c, cudaStream_t st);
  static void gram_loop(const SolveConst& c, cudaStream_t st);
  static void cg_a(const SolveConst& c, int64_t rmax, cudaStream_t st);
  static void cg_b(const SolveConst& c, int64_t rmax, cudaStream_t st);
  static void spmm_plain(const int32_t* rp, const int32_t* ci, const double* val, const double* x,
                         double* y, int64_t n, cudaStream_t st);
  static void export_block(const double* blk, const double* nfac, int64_t b, double* out, int64_t n,
                           cudaStream_t st);
  static void dist_fin(const SolveConst& c, int mode, int64_t msg, cudaStream_t st);
  static void halo(const SolveConst& c, int unpack, int64_t H, cudaStream_t st);
};
#else
template <int S>
struct Launch {
  static void init(const SolveConst& c, const double* dc1, const double* dc2, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    k_init_transpose<S><<<dim3(rows_grid(nmax), c.nsides), 256, 0, st>>>(c, dc1, dc2);
    k_update<S><<<dim3((unsigned)cmax, 1, c.nsides), 256, 0, st>>>(c, (int)UM_INIT);
    k_householder<S><<<c.nsides, 1024, 0, st>>>(c, 2);
  }
  static void spmm(const SolveConst& c, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    k_spmm<S><<<dim3(rows_grid(nmax), c.nsides), 256, 0, st>>>(c);
  }
  static void gram(const SolveConst& c, int mode, int64_t nblk, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    size_t smem = 0;
#if SK_GRAM_RING
    smem = GramRing<S>::BYTES;
    static bool attr = false;
    if (smem > 48 * 1024 && !attr) {
      cudaFuncSetAttribute(k_gram<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
#endif
    k_gram<S><<<dim3((unsigned)((nblk > 0 ? nblk : 1) * GramSplit<S>::H), (unsigned)cmax, c.nsides), 256, smem,
                st>>>(c, mode);
  }
  static void update(const SolveConst& c, int mode, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    k_update<S><<<dim3((unsigned)cmax, 1, c.nsides), 256, 0, st>>>(c, mode);
  }
  static void householder(const SolveConst& c, int which, cudaStream_t st) {
    k_householder<S><<<c.nsides, 1024, 0, st>>>(c, which);
  }
  static void dist_fin(const SolveConst& c, int mode, int64_t msg, cudaStream_t st) {
    k_dist_fin<S><<<c.nsides, 256, 0, st>>>(c, mode, msg);
  }
  static void halo(const SolveConst& c, int unpack, int64_t H, cudaStream_t st) {
    const unsigned g = (unsigned)((H * S + 255) / 256 > 0 ? ((H * S + 255) / 256 < 1184 ? (H * S + 255) / 256 : 1184) : 1);
    if (unpack)
      k_halo_unpack<S><<<dim3(g, c.nsides), 256, 0, st>>>(c);
    else
      k_halo_pack<S><<<dim3(g, c.nsides), 256, 0, st>>>(c);
  }
  static void arn_update(const SolveConst& c, int mode, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    const unsigned g = (unsigned)((nmax + kArnThreads - 1) / kArnThreads);
    k_arn_update<S><<<dim3(g, c.nsides), kArnThreads, 0, st>>>(c, mode);
  }
  static void self_gram(const SolveConst& c, cudaStream_t st) {
    k_self_gram<S><<<dim3(fused_grid(c), 1, c.nsides), kFusedThreads, 0, st>>>(c, 0);
  }
  static unsigned fused_grid(const SolveConst& c) {
    int64_t m = 0;
    for (int s = 0; s < c.nsides; ++s) m = mx64(m, (c.side[s].nseg + kFusedSegsPerCta - 1) / kFusedSegsPerCta);
    return (unsigned)m;
  }
  template <int MODE>
  static void fused_mode(const SolveConst& c, int pass, int side0, int nz, cudaStream_t st) {
    if constexpr (S <= 4) {
      if (pass == 1)
        k_lanczos_p1<S, MODE><<<dim3(fused_grid(c), 1, nz), kFusedThreads, 0, st>>>(c, side0);
      else
        k_lanczos_p2<S, MODE><<<dim3(fused_grid(c), 1, nz), kFusedThreads, 0, st>>>(c, side0);
    }
  }
  static void fused_side(const SolveConst& c, int pass, int mode, int side0, int nz, cudaStream_t st) {
    switch (mode) {
      case 2: fused_mode<2>(c, pass, side0, nz, st); break;
      case 3: fused_mode<3>(c, pass, side0, nz, st); break;
      case 12: fused_mode<12>(c, pass, side0, nz, st); break;
      case 13: fused_mode<13>(c, pass, side0, nz, st); break;
      default: fused_mode<0>(c, pass, side0, nz, st); break;
    }
  }
  static void fused(const SolveConst& c, int pass, cudaStream_t st) {
    const int m0 = host_row_mode(c.side[0]);
    if (c.nsides == 1 || host_row_mode(c.side[1]) == m0) {
      fused_side(c, pass, m0, 0, c.nsides, st);
    } else {
      fused_side(c, pass, m0, 0, 1, st);
      fused_side(c, pass, host_row_mode(c.side[1]), 1, 1, st);
    }
  }
  static void lanczos_p1(const SolveConst& c, cudaStream_t st) { fused(c, 1, st); }
  static void lanczos_p2(const SolveConst& c, cudaStream_t st) { fused(c, 2, st); }
  static int64_t wave_ctas(const SideConst& sc) {
    const int64_t ntile = (sc.nseg + kFusedSegsPerCta - 1) / kFusedSegsPerCta;
    const int64_t trows = (int64_t)kSeg * kFusedSegsPerCta;
    return ntile + 1 + (sc.bw + trows - 1) / trows;
  }
  template <int MODE>
  static void wave_mode(const SolveConst& c, int side0, int interleave, unsigned grid, cudaStream_t st) {
    if constexpr (S <= 4 && MODE != 0) k_lanczos_wave<S, MODE><<<grid, kFusedThreads, 0, st>>>(c, side0, interleave);
  }
  static void wave_side(const SolveConst& c, int side0, int interleave, unsigned grid, cudaStream_t st) {
    switch (host_row_mode(c.side[side0])) {
      case 2: wave_mode<2>(c, side0, interleave, grid, st); break;
      case 3: wave_mode<3>(c, side0, interleave, grid, st); break;
      case 12: wave_mode<12>(c, side0, interleave, grid, st); break;
      case 13: wave_mode<13>(c, side0, interleave, grid, st); break;
      default: break;
    }
  }
  static bool cols_ok(const SideConst& sc) {
    if (S > 2 || sc.sdim != 2 || sc.sg % kSeg != 0 || !sc.spart) return false;
    const int64_t ns = sc.sg / kSeg;
    return ns <= 8 && (ns & (ns - 1)) == 0;
  }
  static int cols_ranges(const SideConst& sc, int nz) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ns = sc.sg / kSeg;
    int64_t r = nsm / (nz * ns);
    r = r < 1 ? 1 : r;
    const int64_t rmin = (sc.sg + kCsMaxLines - 1) / kCsMaxLines;
    if (r < rmin) r = rmin;
    if (r > sc.sg / kCsBlk) r = sc.sg / kCsBlk;
    return (int)r;
  }
  static void cols_launch(const SolveConst& c, int side0, int nz, cudaStream_t st) {
    if constexpr (S <= 2) {
      const SideConst& sc = c.side[side0];
      const int nr = cols_ranges(sc, nz);
      const size_t smem = sizeof(double) * ((kCsAR * kCsA + kCsBR * (SK_CS_TMA ? kCsA : kCsK) + kCsKR * kCsK + kCsZR * kSeg) * S);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_lanczos_cols<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
      }
      k_lanczos_cols<S><<<dim3((unsigned)((sc.sg / kSeg) * nr), nz), kCsThreads, smem, st>>>(c, side0, nr);
    }
  }
  static void lanczos_sweep(const SolveConst& c, cudaStream_t st) {
    if (cols_ok(c.side[0]) && (c.nsides == 1 || cols_ok(c.side[1])) && !getenv("SK_NO_COLS")) {
      if (c.nsides == 2 && c.side[1].sg != c.side[0].sg) {
        cols_launch(c, 0, 1, st);
        cols_launch(c, 1, 1, st);
      } else {
        cols_launch(c, 0, c.nsides, st);
      }
      return;
    }
    const int64_t w0 = wave_ctas(c.side[0]);
    if (c.nsides == 1) {
      wave_side(c, 0, 0, (unsigned)w0, st);
    } else if (wave_ctas(c.side[1]) == w0 && host_row_mode(c.side[1]) == host_row_mode(c.side[0])) {
      wave_side(c, 0, 1, (unsigned)(2 * w0), st);  // tiles of both sides interleaved
    } else {
      wave_side(c, 0, 0, (unsigned)w0, st);
      wave_side(c, 1, 0, (unsigned)wave_ctas(c.side[1]), st);
    }
  }
  static void gram_loop(const SolveConst& c, cudaStream_t st) {
    int64_t nmax, cmax;
    dims(c, nmax, cmax);
    k_gram_loop<S><<<dim3((unsigned)cmax, 1, c.nsides), 256, 0, st>>>(c);
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
  static void export_block(const double* blk, const double* nfac, int64_t b, double* out, int64_t n,
                           cudaStream_t st) {
    k_export_block<S><<<rows_grid(n), 256, 0, st>>>(blk, nfac, b, out, n);
  }
};
#endif  // SK_INST_COMMON

#ifdef SK_INST_S
template struct Launch<SK_INST_S>;
#endif

#ifdef SK_INST_COMMON
// =====================================================================
// BiCGSTAB (factorized_solvers.cpp:220-389) on the device
// =====================================================================
__device__ __forceinline__ double hpacked(const double* hb, int64_t hld, int64_t i, int64_t l) {
  return hb[l * hld + i];
}

// Dense core image with the upper block Hessenberg H (V side) and G (W side):
// q(i,j) = Hpart(i,j) [j < pc] + Gpart(i,j) [i < pr], each part an fma chain over
// the contraction index in ascending order (oracle image(), Arnoldi branch).
// Leading structural zeros are skipped per tile; fma(0, x, acc) = acc for the
// zero padding inside a tile (acc never -0, finite operands).
constexpr int kImT = 64, kImK = 16;
__global__ void __launch_bounds__(256) k_bi_image(const __grid_constant__ SolveConst c, int which) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int s = c.s;
  const double* src = which == 0 ? c.P[0] : c.S;
  double* dst = which == 0 ? c.Q : c.T;
  const int64_t pr = which == 0 ? st->rows_p : st->rows_s, pc = which == 0 ? st->cols_p : st->cols_s;
  const int64_t ro = which == 0 ? st->rows_q : st->rows_t, co = which == 0 ? st->cols_q : st->cols_t;
  const int64_t i0 = (int64_t)blockIdx.x * kImT, j0 = (int64_t)blockIdx.y * kImT;
  if (i0 >= ro || j0 >= co) return;
  const double* hv = c.side[0].hband;
  const double* hw = c.side[c.nsides > 1 ? 1 : 0].hband;
  const int64_t hldv = c.side[0].hld, hldw = c.side[c.nsides > 1 ? 1 : 0].hld;
  __shared__ double As[kImK][kImT + 1], Bs[kImK][kImT + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double accH[4][4], accG[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) accH[a][b] = accG[a][b] = 0.0;
  const int64_t ld = c.ld;
  // H part: rows i (H rows), columns j < pc, contraction l in [lH0, pr)
  if (j0 < pc) {
    const int64_t lH0 = (int64_t)s * mx64(0, i0 / s - 1);
    for (int64_t l0 = lH0; l0 < pr; l0 += kImK) {
      for (int idx = threadIdx.x; idx < kImK * kImT; idx += blockDim.x) {
        const int kk = idx / kImT, ii = idx % kImT;
        const int64_t l = l0 + kk;
        As[kk][ii] = (l < pr && i0 + ii < ro) ? hpacked(hv, hldv, i0 + ii, l) : 0.0;
        Bs[kk][ii] = (l < pr && j0 + ii < pc) ? src[(j0 + ii) * ld + l] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kImK; ++kk) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk][ty * 4 + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx * 4 + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) accH[a][b] = __fma_rn(av[a], bv[b], accH[a][b]);
      }
      __syncthreads();
    }
  }
  // G part: rows i < pr, columns j (G rows), contraction l in [lG0, pc)
  if (i0 < pr) {
    const int64_t lG0 = (int64_t)s * mx64(0, j0 / s - 1);
    for (int64_t l0 = lG0; l0 < pc; l0 += kImK) {
      for (int idx = threadIdx.x; idx < kImK * kImT; idx += blockDim.x) {
        const int kk = idx / kImT, ii = idx % kImT;
        const int64_t l = l0 + kk;
        As[kk][ii] = (l < pc && i0 + ii < pr) ? src[l * ld + i0 + ii] : 0.0;
        Bs[kk][ii] = (l < pc && j0 + ii < co) ? hpacked(hw, hldw, j0 + ii, l) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kImK; ++kk) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk][ty * 4 + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx * 4 + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) accG[a][b] = __fma_rn(av[a], bv[b], accG[a][b]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + ty * 4 + a, j = j0 + tx * 4 + b;
      if (i >= ro || j >= co) continue;
      const bool hj = j < pc, gi = i < pr;
      const double q = (hj && gi) ? __dadd_rn(accH[a][b], accG[a][b]) : (hj ? accH[a][b] : (gi ? accG[a][b] : 0.0));
      dst[j * ld + i] = q;
    }
}

// Register-blocked version: 128x128 output tile, 8x8 outputs per thread,
// BK = 8 chunks double-buffered through registers -> smem. part 0 writes the
// H part (columns j < pc); part 1 adds the G part per the presence rule. The
// fma chain of every output runs over l in ascending order (bitwise the above).
constexpr int kBM = 128, kBK = 8;
__global__ void __launch_bounds__(256, 1) k_bi_image2(const __grid_constant__ SolveConst c, int which, int part) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int s = c.s;
  const double* src = which == 0 ? c.P[0] : c.S;
  double* dst = which == 0 ? c.Q : c.T;
  const int64_t pr = which == 0 ? st->rows_p : st->rows_s, pc = which == 0 ? st->cols_p : st->cols_s;
  const int64_t ro = which == 0 ? st->rows_q : st->rows_t, co = which == 0 ? st->cols_q : st->cols_t;
  const int64_t i0 = (int64_t)blockIdx.x * kBM, j0 = (int64_t)blockIdx.y * kBM;
  if (i0 >= ro || j0 >= co) return;
  const int64_t ld = c.ld;
  const double* hv = c.side[0].hband;
  const double* hw = c.side[c.nsides > 1 ? 1 : 0].hband;
  const int64_t hldv = c.side[0].hld, hldw = c.side[c.nsides > 1 ? 1 : 0].hld;
  // contraction range and operand roles
  int64_t l_begin, l_end;
  bool active;
  if (part == 0) {
    active = j0 < pc;
    l_begin = (int64_t)s * mx64(0, i0 / s - 1);
    l_end = pr;
  } else {
    active = i0 < pr;
    l_begin = (int64_t)s * mx64(0, j0 / s - 1);
    l_end = pc;
  }
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  // row stride 132 doubles: the transposed (kk-fastest) stores below hit each
  // bank pair at most twice per warp (the 2-wavefront minimum for 256 B)
  __shared__ double As[2][kBK][kBM + 4], Bs[2][kBK][kBM + 4];
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  // each thread stages 4 A and 4 B values per chunk (8 x 128 = 1024 each).
  // Operands contiguous along m use idx -> (kk = idx / 128, m = idx % 128); the
  // part-0 B operand (the core, contiguous along l) uses kk = idx % 8, m = idx / 8
  // so a warp reads 4 columns x 64 contiguous bytes.
  double ra[4], rb[4];
  auto fetch = [&](int64_t l0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + 256 * q;
      const int kk = idx / kBM, mm = idx % kBM;
      const int64_t l = l0 + kk;
      const bool lin = l < l_end;
      if (part == 0) {
        const int kt = idx % kBK, mt = idx / kBK;
        const int64_t lt = l0 + kt;
        const int64_t i = i0 + mm, j = j0 + mt;
        ra[q] = (lin && i < ro) ? hpacked(hv, hldv, i, l) : 0.0;
        rb[q] = (lt < l_end && j < pc) ? src[j * ld + lt] : 0.0;
      } else {
        const int64_t i = i0 + mm, j = j0 + mm;
        ra[q] = (lin && i < pr) ? src[l * ld + i] : 0.0;
        rb[q] = (lin && j < co) ? hpacked(hw, hldw, j, l) : 0.0;
      }
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + 256 * q;
      As[buf][idx / kBM][idx % kBM] = ra[q];
      if (part == 0)
        Bs[buf][idx % kBK][idx / kBK] = rb[q];
      else
        Bs[buf][idx / kBM][idx % kBM] = rb[q];
    }
  };
  if (active && l_begin < l_end) {
    fetch(l_begin);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int64_t l0 = l_begin; l0 < l_end; l0 += kBK) {
      const bool more = l0 + kBK < l_end;
      if (more) fetch(l0 + kBK);
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) {
        double av[8], bv[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) av[a] = As[buf][kk][ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 8; ++b) bv[b] = Bs[buf][kk][tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) acc[a][b] = __fma_rn(av[a], bv[b], acc[a][b]);
      }
      if (more) {
        stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int64_t i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      if (i >= ro || j >= co) continue;
      const bool hj = j < pc, gi = i < pr;
      const int64_t o = j * ld + i;
      if (part == 0) {
        if (hj) dst[o] = acc[a][b];
      } else {
        if (hj && gi) dst[o] = __dadd_rn(dst[o], acc[a][b]);
        else if (gi) dst[o] = acc[a][b];
        else if (!hj) dst[o] = 0.0;
      }
    }
}

__device__ inline void bi_breakdown(const SolveConst& c) {
  DevState* st = c.st;
  st->status = BREAKDOWN;
  c.hist_rel[st->k + 1] = c.hist_rel[st->k];
  c.hist_tb[st->k + 1] = (double)globaltimer();
  if (c.hist_tk[st->k + 1] == 0.0) c.hist_tk[st->k + 1] = c.hist_tb[st->k + 1];
  st->nrec = st->k + 2;
}

// after an extension pair: breakdown check and the image window (sched = (2k+2+which)s)
__global__ void k_bi_begin(const __grid_constant__ SolveConst c, int which) {
  DevState* st = c.st;
  if (threadIdx.x != 0 || st->status != RUNNING) return;
  if (any_side_broken(c)) {
    bi_breakdown(c);
    return;
  }
  const int s = c.s;
  const int64_t k = st->k;
  const int64_t sched = (2 * k + 2 + which) * s;
  const int64_t vc = st->side[0].blocks * s, wc = st->side[c.nsides > 1 ? 1 : 0].blocks * s;
  const int64_t r = sched < vc ? sched : vc, cc = sched < wc ? sched : wc;
  if (which == 0) {
    st->rows_q = r;
    st->cols_q = cc;
    c.hist_tk[k + 1] = (double)globaltimer();  // first extension done
  } else {
    st->rows_t = r;
    st->cols_t = cc;
  }
}

// R2 contract over an s x s window (one tile): lane i sums its row, butterfly
__device__ __forceinline__ double r2_small(const double* a, int64_t lda, const double* b, int64_t ldb, int s) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if (lane < s)
    for (int j = 0; j < s; ++j) acc = __dadd_rn(acc, __dmul_rn(a[j * lda + lane], b[j * ldb + lane]));
  return butterfly(acc);
}

// denom = <R~0, Q>_{s x s}, guard on the angle, alpha (factorized_solvers.cpp:292-300)
__global__ void k_bi_alpha(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int s = c.s;
  const double denom = r2_small(c.Rs, s, c.Q, c.ld, s);
  const double qw2 = r2_small(c.Q, c.ld, c.Q, c.ld, s);
  if (threadIdx.x != 0) return;
  const double q_win = __dsqrt_rn(qw2);
  st->denom = denom;
  if (fabs(denom) < __dmul_rn(__dmul_rn(c.tol, st->norm_shadow), q_win)) {
    bi_breakdown(c);
    return;
  }
  st->alpha = __ddiv_rn(st->rho, denom);
  st->rows_s = st->rows_q;
  st->cols_s = st->cols_q;
}

// S = embed(R) - alpha Q over Q's window (factorized_solvers.cpp:301-302)
__global__ void k_bi_s(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int64_t rq = st->rows_q, cq = st->cols_q, rp = st->rows_p, cp = st->cols_p;
  const double na = -st->alpha;
  const int64_t total = rq * cq;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / rq, i = idx - j * rq;
    const int64_t o = j * c.ld + i;
    const double r = (i < rp && j < cp) ? c.R[o] : 0.0;
    c.S[o] = __dadd_rn(r, __dmul_rn(na, c.Q[o]));
  }
}

// tt = <T,T>, ss = <S,S>, st = <S,T>_S (R2 over their windows), omega (:320-336)
__global__ void __launch_bounds__(256) k_bi_omega(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int64_t rt = st->rows_t, ct = st->cols_t, rs = st->rows_s, cs = st->cols_s;
  const int64_t nti = (rt + kTile - 1) / kTile, ntj = (ct + kTile - 1) / kTile;
  const int64_t sti = (rs + kTile - 1) / kTile, stj = (cs + kTile - 1) / kTile;
  const int64_t ti = blockIdx.x, tj = blockIdx.y;
  if (ti >= nti || tj >= ntj) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    const int64_t i = ti * kTile + lane;
    double att = 0.0, ass = 0.0, ast = 0.0;
    if (i < rt)
      for (int q = 0; q < kTile; ++q) {
        const int64_t j = tj * kTile + q;
        if (j >= ct) break;
        const double t = c.T[j * c.ld + i];
        att = __dadd_rn(att, __dmul_rn(t, t));
        if (i < rs && j < cs) {
          const double sv = c.S[j * c.ld + i];
          ass = __dadd_rn(ass, __dmul_rn(sv, sv));
          ast = __dadd_rn(ast, __dmul_rn(sv, t));
        }
      }
    att = butterfly(att);
    ass = butterfly(ass);
    ast = butterfly(ast);
    if (lane == 0) {
      c.cpart[tj * nti + ti] = att;
      if (ti < sti && tj < stj) {
        const int64_t base = nti * ntj + 256;
        c.cpart[base + tj * sti + ti] = ass;
        c.cpart[base + sti * stj + tj * sti + ti] = ast;
      }
    }
  }
  if (!last_cta_arrive(c.ccounter, (unsigned)(nti * ntj))) return;
  __shared__ double scratch[256];
  const int64_t base = nti * ntj + 256;
  double* scr = ntj <= 256 ? scratch : c.cpart + base + 2 * sti * stj;
  const double tt = r2_final(c.cpart, nti, ntj, scr);
  double* scr2 = stj <= 256 ? scratch : c.cpart + base + 2 * sti * stj;
  const double ss = r2_final(c.cpart + base, sti, stj, scr2);
  const double stv = r2_final(c.cpart + base + sti * stj, sti, stj, scr2);
  if (threadIdx.x != 0) return;
  st->tt = tt;
  st->ss = ss;
  st->st = stv;
  if (__dsqrt_rn(ss) <= __dmul_rn(c.eps, st->norm_r0)) {
    st->omega = 0.0;  // converged at the half step
  } else if (tt < __dmul_rn(c.tol, ss)) {
    bi_breakdown(c);
  } else {
    st->omega = __ddiv_rn(stv, tt);
  }
}

// X = (embed(X) + alpha embed(P)) + omega S; R = embed(S) - omega T; ||R||; rho',
// angle guard, beta (factorized_solvers.cpp:338-367)
__global__ void __launch_bounds__(256) k_bi_update(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int64_t rt = st->rows_t, ct = st->cols_t, rs = st->rows_s, cs = st->cols_s;
  const int64_t rp = st->rows_p, cp = st->cols_p;
  const int64_t nti = (rt + kTile - 1) / kTile, ntj = (ct + kTile - 1) / kTile;
  const int64_t ti = blockIdx.x, tj = blockIdx.y;
  if (ti >= nti || tj >= ntj) return;
  const double alpha = st->alpha, omega = st->omega, nom = -omega;
  __shared__ double f[kTile * kTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = ti * kTile + lane;
  for (int q = 0; q < 4; ++q) {
    const int lc = warp * 4 + q;
    const int64_t j = tj * kTile + lc;
    double fv = 0.0;
    if (i < rt && j < ct) {
      const int64_t o = j * c.ld + i;
      const bool ins = i < rs && j < cs;
      const double sv = ins ? c.S[o] : 0.0;
      if (ins) {
        const double pv = (i < rp && j < cp) ? c.P[0][o] : 0.0;
        c.X[o] = __dadd_rn(__dadd_rn(c.X[o], __dmul_rn(alpha, pv)), __dmul_rn(omega, sv));
      }
      const double rn = __dadd_rn(sv, __dmul_rn(nom, c.T[o]));
      c.R[o] = rn;
      fv = __dmul_rn(rn, rn);
    }
    f[lc * kTile + lane] = fv;
  }
  __syncthreads();
  if (warp == 0) {
    const int nr = (int)mn64(kTile, rt - ti * kTile), nc = (int)mn64(kTile, ct - tj * kTile);
    const double v = tile_reduce(f, nr, nc);
    if (lane == 0) c.cpart[tj * nti + ti] = v;
  }
  if (!last_cta_arrive(c.ccounter, (unsigned)(nti * ntj))) return;
  __shared__ double scratch[256];
  double* scr = ntj <= 256 ? scratch : c.cpart + nti * ntj;
  const double rr = r2_final(c.cpart, nti, ntj, scr);
  const int s = c.s;
  double rho_next = 0.0, rw2 = 0.0;
  if (threadIdx.x < 32) {
    rho_next = r2_small(c.Rs, s, c.R, c.ld, s);
    rw2 = r2_small(c.R, c.ld, c.R, c.ld, s);
  }
  if (threadIdx.x != 0) return;
  const int64_t k = st->k;
  const double norm_r = __dsqrt_rn(rr);
  c.hist_rel[k + 1] = __ddiv_rn(norm_r, st->norm_r0);
  c.hist_tb[k + 1] = (double)globaltimer();
  st->nrec = k + 2;
  st->rows_x = rs;
  st->cols_x = cs;
  st->rows_po = rp;
  st->cols_po = cp;
  st->rows_p = rt;
  st->cols_p = ct;
  st->k = k + 1;
  if (norm_r <= __dmul_rn(st->norm_r0, c.eps)) {
    st->status = CONVERGED;
    return;
  }
  const double r_win = __dsqrt_rn(rw2);
  if (fabs(rho_next) < __dmul_rn(__dmul_rn(c.tol, st->norm_shadow), r_win)) {
    st->status = BREAKDOWN;  // record already written for this iteration
    return;
  }
  st->beta = __dmul_rn(__ddiv_rn(alpha, omega), __ddiv_rn(rho_next, st->rho));
  st->rho = rho_next;
  if (st->k >= c.max_iter) st->status = MAXITER;
}

// P = (R + beta embed(P)) + (-beta*omega) embed(Q) over R's window (:369-375)
__global__ void k_bi_p(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (st->status != RUNNING) return;
  const int64_t rt = st->rows_p, ct = st->cols_p, rp = st->rows_po, cp = st->cols_po;
  const int64_t rq = st->rows_q, cq = st->cols_q;
  const double beta = st->beta, nbo = __dmul_rn(-beta, st->omega);
  const int64_t total = rt * ct;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / rt, i = idx - j * rt;
    const int64_t o = j * c.ld + i;
    const double pv = (i < rp && j < cp) ? c.P[0][o] : 0.0;
    const double qv = (i < rq && j < cq) ? c.Q[o] : 0.0;
    c.P[0][o] = __dadd_rn(__dadd_rn(c.R[o], __dmul_rn(beta, pv)), __dmul_rn(nbo, qv));
  }
}
#endif

#ifdef SK_INST_COMMON
static int g_launches = 0;
int launch_count() { return g_launches; }
void launch_count_reset() { g_launches = 0; }

#define SK_DISPATCH_S(s, CALL)      \
  switch (s) {                      \
    case 1: Launch<1>::CALL; break; \
    case 2: Launch<2>::CALL; break; \
    case 3: Launch<3>::CALL; break; \
    case 4: Launch<4>::CALL; break; \
    case 5: Launch<5>::CALL; break; \
    case 6: Launch<6>::CALL; break; \
    case 7: Launch<7>::CALL; break; \
    case 8: Launch<8>::CALL; break; \
    default: break;                 \
  }

void launch_init(const SolveConst& c, const double* dc1, const double* dc2, cudaStream_t st) {
  SK_DISPATCH_S(c.s, init(c, dc1, dc2, st));
  k_core_init<<<1, 32, 0, st>>>(c);
  g_launches += 4;
}
void launch_spmm(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, spmm(c, st));
  g_launches += 1;
}
void launch_lanczos_gram(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, gram(c, (int)GM_J, 2, st));
  g_launches += 1;
}
bool lanczos_fused_ok(const SolveConst& c) { return c.s <= 4 && !c.full_reorth; }
void launch_lanczos_p1(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, lanczos_p1(c, st));
  g_launches += 1;
}
void launch_lanczos_p2(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, lanczos_p2(c, st));
  g_launches += 1;
}
// the wavefront pass applies to matrix-free stencil operators on one GPU
bool lanczos_sweep_ok(const SolveConst& c) {
  if (!lanczos_fused_ok(c) || c.arnoldi || c.world > 1) return false;
  for (int sd = 0; sd < c.nsides; ++sd) {
    const SideConst& sc = c.side[sd];
    if (sc.sdim == 0 || sc.dist || sc.row0 != 0 || !sc.spart || !sc.sctr) return false;
  }
  return true;
}
void launch_lanczos_sweep(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, lanczos_sweep(c, st));
  g_launches += (c.nsides == 2 && (c.side[1].n != c.side[0].n || c.side[1].sdim != c.side[0].sdim)) ? 2 : 1;
}
void launch_lanczos_update(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st) {
  if (c.full_reorth) {
    SK_DISPATCH_S(c.s, update(c, (int)UM_FIRST, st));
    SK_DISPATCH_S(c.s, gram(c, (int)GM_ALL_X, kmax_blocks, st));
    SK_DISPATCH_S(c.s, update(c, (int)UM_SECOND, st));
    g_launches += 3;
  } else {
    SK_DISPATCH_S(c.s, update(c, (int)UM_LANCZOS, st));
    g_launches += 1;
  }
}
void launch_rare(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st) {
  SK_DISPATCH_S(c.s, householder(c, 0, st));
  (void)kmax_blocks;
  SK_DISPATCH_S(c.s, gram_loop(c, st));
  SK_DISPATCH_S(c.s, update(c, (int)UM_CLEAN, st));
  SK_DISPATCH_S(c.s, householder(c, 1, st));
  g_launches += 4;
}
static __global__ void k_dist_pause(const __grid_constant__ SolveConst c) {
  DevState* st = c.st;
  if (threadIdx.x != 0 || st->status != RUNNING) return;
  for (int sd = 0; sd < c.nsides; ++sd) {
    const int g = st->side[sd].stage;
    if (g == ST_NEED_HH || g == ST_NEED_CLEANUP) st->status = PAUSED;
  }
}
static __global__ void k_dist_resume(const __grid_constant__ SolveConst c) {
  if (threadIdx.x == 0 && c.st->status == PAUSED) c.st->status = RUNNING;
}
void launch_dist_fin(const SolveConst& c, int mode, int64_t msg, cudaStream_t st) {
  SK_DISPATCH_S(c.s, dist_fin(c, mode, msg, st));
  g_launches += 1;
}
void launch_dist_pause(const SolveConst& c, cudaStream_t st) {
  k_dist_pause<<<1, 32, 0, st>>>(c);
  g_launches += 1;
}
void launch_dist_resume(const SolveConst& c, cudaStream_t st) {
  k_dist_resume<<<1, 32, 0, st>>>(c);
  g_launches += 1;
}
void launch_halo(const SolveConst& c, int unpack, int64_t H, cudaStream_t st) {
  SK_DISPATCH_S(c.s, halo(c, unpack, H, st));
  g_launches += 1;
}
void launch_householder(const SolveConst& c, int which, cudaStream_t st) {
  SK_DISPATCH_S(c.s, householder(c, which, st));
  g_launches += 1;
}
void launch_gram_loop(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, gram_loop(c, st));
  g_launches += 1;
}
void launch_update_clean(const SolveConst& c, cudaStream_t st) {
  SK_DISPATCH_S(c.s, update(c, (int)UM_CLEAN, st));
  g_launches += 1;
}
void launch_arnoldi_ext(const SolveConst& c, int64_t kmax_blocks, cudaStream_t st) {
  SK_DISPATCH_S(c.s, spmm(c, st));
  SK_DISPATCH_S(c.s, gram(c, (int)GM_ALL_W, kmax_blocks, st));
  SK_DISPATCH_S(c.s, arn_update(c, (int)UM_FIRST, st));
  SK_DISPATCH_S(c.s, gram(c, (int)GM_ALL_X, kmax_blocks, st));
  SK_DISPATCH_S(c.s, arn_update(c, (int)UM_SECOND, st));
  SK_DISPATCH_S(c.s, self_gram(c, st));
  SK_DISPATCH_S(c.s, householder(c, 0, st));
  g_launches += 7;
}
void launch_bicgstab_half(const SolveConst& c, int which, int64_t rmax, cudaStream_t st) {
  k_bi_begin<<<1, 32, 0, st>>>(c, which);
  if (getenv("SK_SIMPLE_IMAGE")) {
    const unsigned nt = (unsigned)((rmax + kImT - 1) / kImT);
    k_bi_image<<<dim3(nt, nt), 256, 0, st>>>(c, which);
  } else {
    const unsigned nt = (unsigned)((rmax + kBM - 1) / kBM);
    k_bi_image2<<<dim3(nt, nt), 256, 0, st>>>(c, which, 0);
    k_bi_image2<<<dim3(nt, nt), 256, 0, st>>>(c, which, 1);
  }
  if (which == 0) {
    k_bi_alpha<<<1, 32, 0, st>>>(c);
    k_bi_s<<<rows_grid(rmax * rmax), 256, 0, st>>>(c);
  } else {
    const unsigned tt = (unsigned)((rmax + kTile - 1) / kTile);
    k_bi_omega<<<dim3(tt, tt), 256, 0, st>>>(c);
    k_bi_update<<<dim3(tt, tt), 256, 0, st>>>(c);
    k_bi_p<<<rows_grid(rmax * rmax), 256, 0, st>>>(c);
  }
  g_launches += which == 0 ? 4 : 5;
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
void launch_export_block(int s, const double* blk, const double* nfac, int64_t b, double* out,
                         int64_t n, cudaStream_t st) {
  SK_DISPATCH_S(s, export_block(blk, nfac, b, out, n, st));
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
