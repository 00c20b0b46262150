// sk_problems.cpp -- problem generators of the product (host C++).
//
// Restates proj/src/problems.cpp:10-96: laplacian_2d, convection_diffusion_3d
// and random_rhs (std::mt19937_64 + Box-Muller with a spare), plus the 2D
// convection-diffusion sibling the BASELINE configs need.
// Rows are emitted directly in CSR order (columns ascending), which is exactly
// what SparseMatrix::from_triplets produces from the reference's triplet stream
// (no duplicates occur), without the O(nnz log nnz) sort.
#include "../../include/sylkrylov_b200.h"

#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

extern "C" {

int64_t sk_gen_stencil_nnz(int32_t kind, int64_t g) {
  if (g < 2) return -1;
  if (kind == 2) return 7 * g * g * g - 6 * g * g;  // 3D: 7 per point minus boundary faces
  return 5 * g * g - 4 * g;                         // 2D
}

sk_status sk_gen_stencil(int32_t kind, int64_t g, const double* wind, int64_t* rp, int64_t* ci,
                         double* val) {
  if (g < 2 || kind < 0 || kind > 2) return SK_ERR_DIMENSION;
  const double h = 1.0 / ((double)g + 1.0);
  const double w0 = wind ? wind[0] : 0.0, w1 = wind ? wind[1] : 0.0, w2 = wind ? wind[2] : 0.0;
  // couplings -1 -/+ w*h/2 per axis (problems.cpp:42-55); Laplacian: w = 0 and diag 4
  const double c0 = w0 * h / 2.0, c1 = w1 * h / 2.0, c2 = w2 * h / 2.0;
  if (kind == 0 || kind == 1) {
    const bool lap = kind == 0;
    const double diag = 4.0;
    const double xm = lap ? -1.0 : -1.0 - c0, xp = lap ? -1.0 : -1.0 + c0;
    const double ym = lap ? -1.0 : -1.0 - c1, yp = lap ? -1.0 : -1.0 + c1;
    // row p = ix + g*iy; nnz before row p is closed-form, so rows fill in parallel
    auto fill_rows = [&](int64_t iy0, int64_t iy1) {
      // nnz of one grid row r: 5g - 2 (x ends) - g at a y boundary
      int64_t nz = 0;
      for (int64_t r = 0; r < iy0; ++r) nz += 5 * g - 2 - ((r == 0 || r == g - 1) ? g : 0);
      for (int64_t iy = iy0; iy < iy1; ++iy) {
        for (int64_t ix = 0; ix < g; ++ix) {
          const int64_t p = ix + g * iy;
          if (iy > 0) ci[nz] = p - g, val[nz++] = ym;
          if (ix > 0) ci[nz] = p - 1, val[nz++] = xm;
          ci[nz] = p, val[nz++] = diag;
          if (ix < g - 1) ci[nz] = p + 1, val[nz++] = xp;
          if (iy < g - 1) ci[nz] = p + g, val[nz++] = yp;
          rp[p + 1] = nz;
        }
      }
    };
    rp[0] = 0;
    const int nt = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (g < 512 || nt == 1) {
      fill_rows(0, g);
    } else {
      std::vector<std::thread> th;
      const int64_t chunk = (g + nt - 1) / nt;
      for (int t = 0; t < nt; ++t) {
        const int64_t a = t * chunk, b = std::min<int64_t>(g, a + chunk);
        if (a < b) th.emplace_back(fill_rows, a, b);
      }
      for (auto& x : th) x.join();
    }
    return SK_OK;
  }
  // 3D (problems.cpp:32-60), p = ix + g*(iy + g*iz)
  const int64_t g2 = g * g;
  int64_t nz = 0;
  rp[0] = 0;
  for (int64_t iz = 0; iz < g; ++iz)
    for (int64_t iy = 0; iy < g; ++iy)
      for (int64_t ix = 0; ix < g; ++ix) {
        const int64_t p = ix + g * (iy + g * iz);
        if (iz > 0) ci[nz] = p - g2, val[nz++] = -1.0 - c2;
        if (iy > 0) ci[nz] = p - g, val[nz++] = -1.0 - c1;
        if (ix > 0) ci[nz] = p - 1, val[nz++] = -1.0 - c0;
        ci[nz] = p, val[nz++] = 6.0;
        if (ix < g - 1) ci[nz] = p + 1, val[nz++] = -1.0 + c0;
        if (iy < g - 1) ci[nz] = p + g, val[nz++] = -1.0 + c1;
        if (iz < g - 1) ci[nz] = p + g2, val[nz++] = -1.0 + c2;
        rp[p + 1] = nz;
      }
  return SK_OK;
}

// random_rhs (problems.cpp:65-96): column-major rows x s, N(0,1) by Box-Muller
sk_status sk_gen_random_rhs(int64_t rows, int64_t s, uint64_t seed, double* out) {
  if (s < 1 || rows < 0) return SK_ERR_DIMENSION;
  std::mt19937_64 gen(seed);
  auto uoc = [&gen]() { return (static_cast<double>(gen() >> 11) + 1.0) * 0x1.0p-53; };
  double spare = 0.0;
  bool have = false;
  const size_t count = (size_t)rows * (size_t)s;
  for (size_t i = 0; i < count; ++i) {
    if (have) {
      out[i] = spare;
      have = false;
    } else {
      const double u1 = uoc(), u2 = uoc();
      const double radius = std::sqrt(-2.0 * std::log(u1));
      const double angle = 2.0 * M_PI * u2;
      out[i] = radius * std::cos(angle);
      spare = radius * std::sin(angle);
      have = true;
    }
  }
  return SK_OK;
}

}  // extern "C"
