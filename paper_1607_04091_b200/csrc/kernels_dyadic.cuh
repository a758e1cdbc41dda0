// kernels_dyadic.cuh -- dyadic-grid evaluation of a reconstruction (front-end
// row SURVEY 8(f)4; restates dyadic.cpp:37-231):
//
//  * k_dy_level  -- one refinement level of every dyadic table at once: the
//    interior scaling function through its dilation equation
//    phi(x) = 2 sum_k h_k phi(2x - k) (dyadic.cpp:57-66) and the p edge
//    functions per side through their coupled equations
//    phi_k(x) = sqrt2 (sum_l H_kl phi_l(2x) + sum_m h_km phi(2x - m))
//    (dyadic.cpp:97-113).  Level r only reads points of levels < r, so one
//    launch per level, all tables in parallel (blockIdx.y = table).
//  * k_dy_ell    -- the scale-J basis sampled on the closed grid of 2^R + 1
//    points as a row-sparse matrix: grid point i -> (column, table value) in
//    ascending column order (left edge columns, the <= 2p interior columns
//    whose support covers i, right edge columns; dyadic.cpp:137-170).
//  * k_dy_weval1 -- 1D: out_i = sum_c (w_c 2^{J/2}) phi_c(i), zero weights
//    skipped, columns ascending (dyadic.cpp:184-199).
//  * k_dy_rows / k_dy_cols -- 2D tensor evaluation out = (B X^T) B^T
//    (dyadic.cpp:201-230) as two banded contractions: Z = B X^T over the
//    coefficient rows (coalesced over the x index), then out(iy, ix) =
//    sum_j Z(iy, j) B(ix, j) with ix fastest (coalesced stores; the output
//    write is the HBM bound).
#pragma once
#include "gs_common.cuh"

#define DY_MAXTAB 17  // interior + 2 x 8 edge functions

struct DyP {
  int p, R, ntab;
  int64_t off[DY_MAXTAB], len[DY_MAXTAB], sb[DY_MAXTAB];
  int side[DY_MAXTAB];  // 0 interior, 1 left edge, 2 right edge
  int kidx[DY_MAXTAB];  // edge function index
  const double* taps;   // 2p, k = -p+1..p
  const double* H[2];   // p x p row-major (left, right)
  const double* h[2];   // p x (2p-1) row-major
};

__device__ __forceinline__ double dy_at(const double* buf, const DyP& P, int t, int64_t num) {
  const int64_t idx = num - (P.sb[t] << P.R);  // FunctionTable::value_at (dyadic.hpp:19-23)
  return (idx < 0 || idx >= P.len[t]) ? 0.0 : buf[P.off[t] + idx];
}

// odd points i = step + 2 step j of level r of table blockIdx.y
__global__ void k_dy_level(DyP P, double* __restrict__ buf, int r) {
  const int t = blockIdx.y;
  const int64_t step = 1LL << (P.R - r);
  const int64_t i = step + 2 * step * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  if (i >= P.len[t]) return;
  const int64_t nx = (P.sb[t] << P.R) + i;
  const int p = P.p;
  double acc = 0.0;
  if (P.side[t] == 0) {
    for (int k = -p + 1; k <= p; ++k) acc += P.taps[k + p - 1] * dy_at(buf, P, 0, 2 * nx - ((int64_t)k << P.R));
    buf[P.off[t] + i] = 2.0 * acc;
    return;
  }
  const int s = P.side[t] - 1, k = P.kidx[t];
  const double* H = P.H[s];
  const double* h = P.h[s];
  const int first = 1 + s * p;  // table id of edge function 0 of this side
  for (int l = 0; l < p; ++l) acc += H[k * p + l] * dy_at(buf, P, first + l, 2 * nx);
  for (int m = p; m <= p + 2 * k; ++m) {
    const int64_t arg = s == 0 ? 2 * nx - ((int64_t)m << P.R) : 2 * nx + ((int64_t)(m + 1) << P.R);
    acc += h[k * (2 * p - 1) + (m - p)] * dy_at(buf, P, 0, arg);
  }
  buf[P.off[t] + i] = sqrt(2.0) * acc;
}

// basis rows of the closed grid: up to km (column, raw table value) pairs per grid point
__global__ void k_dy_ell(DyP P, const double* __restrict__ buf, int J, int Rg, int km, int* __restrict__ cnt,
                         int* __restrict__ col, double* __restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n_grid = 1LL << Rg;
  if (i > n_grid) return;
  const int p = P.p;
  const int64_t n = 1LL << J, unit = 1LL << P.R;  // P.R = tabres = R - J
  int k = 0;
  int* c_out = col + i * km;
  double* v_out = val + i * km;
  auto put = [&](int64_t c, double v) {
    c_out[k] = (int)c;
    v_out[k] = v;
    ++k;
  };
  if (p >= 2)
    for (int c = 0; c < p; ++c)  // left edge functions (support_begin 0)
      if (i <= min(n_grid, (int64_t)(p + c) * unit)) put(c, buf[P.off[1 + c] + i]);
  const int64_t clo = p >= 2 ? p : 0, chi = p >= 2 ? n - p - 1 : n - 1;
  const int64_t q = i / unit;
  for (int64_t c = max(clo, q - p); c <= min(chi, q + p); ++c) {
    const int64_t lo = max((int64_t)0, (c - p + 1) * unit), hi = min(n_grid, (c + p) * unit);
    if (i >= lo && i <= hi) put(c, dy_at(buf, P, 0, i - c * unit));
  }
  if (p >= 2)
    for (int64_t c = n - p; c < n; ++c) {  // right edge functions, j = n - 1 - c
      const int j = (int)(n - 1 - c);
      if (i >= max((int64_t)0, n_grid - (int64_t)(p + j) * unit)) put(c, dy_at(buf, P, 1 + p + j, i - n_grid));
    }
  cnt[i] = k;
}

__global__ void k_dy_weval1(int64_t g, int km, const int* __restrict__ cnt, const int* __restrict__ col,
                            const double* __restrict__ val, const double* __restrict__ w, double amp,
                            double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g) return;
  double acc = 0.0;
  for (int k = 0; k < cnt[i]; ++k) {
    const double wc = w[col[i * km + k]];
    if (wc != 0.0) acc += (wc * amp) * val[i * km + k];
  }
  out[i] = acc;
}

// Z(a, j) = sum_i B(a, i) X(j, i), X(j, i) = coeffs[i n + j]
__global__ void k_dy_rows(int64_t g, int n, int km, const int* __restrict__ cnt, const int* __restrict__ col,
                          const double* __restrict__ val, const double* __restrict__ coeffs, double amp,
                          double* __restrict__ Z) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t a = blockIdx.y;
  if (j >= n) return;
  double acc = 0.0;
  for (int k = 0; k < cnt[a]; ++k) acc += (amp * val[a * km + k]) * coeffs[(int64_t)col[a * km + k] * n + j];
  Z[a * n + j] = acc;
}

// out(a, b) = sum_j Z(a, j) B(b, j)
__global__ void k_dy_cols(int64_t g, int n, int km, const int* __restrict__ cnt, const int* __restrict__ col,
                          const double* __restrict__ val, const double* __restrict__ Z, double amp,
                          double* __restrict__ out) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t a = blockIdx.y;
  if (b >= g) return;
  const double* z = Z + a * n;
  double acc = 0.0;
  for (int k = 0; k < cnt[b]; ++k) acc += z[col[b * km + k]] * (amp * val[b * km + k]);
  out[a * g + b] = acc;
}
