// kernels_ndft.cuh -- direct (exact) NDFT on the FP64 pipe: ndft_forward /
// ndft_adjoint (nufft.cpp:74-132) as a blocked complex-exponential kernel.
//
//   forward  y_m = sum_{k0,k1} x[k0,k1] e^{-2 pi i (k0 xi0_m + k1 xi1_m)}
//   adjoint  z[k0,k1] = sum_m y_m e^{+2 pi i (k0 xi0_m + k1 xi1_m)}
//
// k = -N/2 .. N/2-1 per axis, last axis fastest (1D: one row, k0 = 0).  Modes
// are grouped in "units" of ND_RUN consecutive k1 of one k0 row, so
//   e^{s 2 pi i (k0 xi0 + (k1s + t) xi1)} = G_u(m) * P_t(m),
//   G_u = e^{s 2 pi i (k0 xi0 + k1s xi1)},  P_t = e^{s 2 pi i t xi1}, t < ND_RUN.
// P_t is evaluated exactly once per point (sincospi); per unit and point the
// inner product costs ND_RUN complex FMAs (4 DFMA each), G_u one sincospi
// (adjoint) or one complex multiply along the unit row with an exact restart
// every ND_RESTART units (forward).  ~5-6 FP64 instructions per term.
//
// Forward: a thread owns ND_FPPT points, CTAs stage ND_FTILE units of x in
// shared memory (warp-broadcast reads).  Adjoint: a thread owns ND_AUPT
// consecutive units (their G_u chained by the per-point giant step
// e^{s 2 pi i ND_RUN xi1}), CTAs stage ND_ATILE points with their P_t table.
// Large problems split the other dimension over CTAs (blockIdx.y) into
// partial sums reduced in a fixed order (deterministic, no atomics).
#pragma once
#include "gs_common.cuh"

#define ND_RUN 16
#define ND_RESTART 8
#define ND_FTHREADS 128
#define ND_FPPT 2
#define ND_FTILE 128  // units staged per forward tile (ND_FTILE * ND_RUN complex = 32 KB)
#define ND_ATHREADS 128
#define ND_ATILE 64   // points staged per adjoint tile (P_t table 16 KB)

struct NdGeom {
  int dim;          // 1 or 2
  int N0, N1;       // modes: N0 rows (1 in 1D) x N1 per row
  int runs;         // units per row = ceil(N1 / ND_RUN)
  int64_t M;        // points
  int lo, hi;       // 1D operator use: only k1 indices [lo, hi) of x enter (edge slots zeroed); else 0, N1
  int rh0, kh1;     // k = -N/2 .. N/2-1 with C++ integer division (nufft.cpp:81, 88-91): an odd
                    // length leaves its last index out -> rows < rh0, k1 indices < kh1 are live
};

__device__ __forceinline__ cplx nd_sincospi(double a) {  // e^{i pi a}
  double s, c;
  sincospi(a, &s, &c);
  return mk(c, s);
}
__device__ __forceinline__ cplx cfma(cplx acc, cplx a, cplx b) {  // acc + a b
  return mk(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}

__device__ __forceinline__ void nd_point(const NdGeom& g, const double* __restrict__ pts, int64_t m, double& xi0,
                                         double& xi1) {
  if (g.dim == 1) {
    xi0 = 0.0;
    xi1 = pts[m];
  } else {
    xi0 = pts[2 * m];
    xi1 = pts[2 * m + 1];
  }
}

// ---------------------------------------------------------------- forward
// part[ks][m] (or y[m] when the launch has one k-split and no epilogue):
// sum over the units [u0, u1) of this blockIdx.y.
__global__ void __launch_bounds__(ND_FTHREADS) k_ndft_fwd(NdGeom g, const double* __restrict__ pts,
                                                           const cplx* __restrict__ x, int units_per_split,
                                                           cplx* __restrict__ out) {
  __shared__ cplx xs[ND_FTILE * ND_RUN];
  pts += (int64_t)blockIdx.z * g.M * g.dim;  // batch of independent problems
  x += (int64_t)blockIdx.z * g.N0 * g.N1;
  out += (int64_t)blockIdx.z * gridDim.y * g.M;
  const int nunits = g.N0 * g.runs;
  const int u0 = blockIdx.y * units_per_split;
  const int u1 = min(nunits, u0 + units_per_split);
  const int64_t mbase = (int64_t)blockIdx.x * ND_FTHREADS * ND_FPPT + threadIdx.x;
  double xi0[ND_FPPT], xi1[ND_FPPT];
  cplx P[ND_FPPT][ND_RUN], acc[ND_FPPT], step[ND_FPPT];
#pragma unroll
  for (int j = 0; j < ND_FPPT; ++j) {
    const int64_t m = mbase + j * ND_FTHREADS;
    xi0[j] = xi1[j] = 0.0;
    if (m < g.M) nd_point(g, pts, m, xi0[j], xi1[j]);
#pragma unroll
    for (int t = 0; t < ND_RUN; ++t) P[j][t] = nd_sincospi(-2.0 * (double)t * xi1[j]);
    step[j] = nd_sincospi(-2.0 * (double)ND_RUN * xi1[j]);  // G_{u+1} = G_u step along a row
    acc[j] = mk(0, 0);
  }
  cplx G[ND_FPPT];
  for (int ut = u0; ut < u1; ut += ND_FTILE) {
    const int nu = min(ND_FTILE, u1 - ut);
    __syncthreads();
    for (int i = threadIdx.x; i < nu * ND_RUN; i += ND_FTHREADS) {
      const int u = ut + i / ND_RUN, t = i % ND_RUN;
      const int r = u / g.runs, k1i = (u % g.runs) * ND_RUN + t;
      xs[i] = (k1i >= g.lo && k1i < g.hi && k1i < g.kh1 && r < g.rh0) ? x[(int64_t)r * g.N1 + k1i] : mk(0, 0);
    }
    __syncthreads();
    for (int i = 0; i < nu; ++i) {
      const int u = ut + i;
      const int r = u / g.runs, a = u % g.runs;
      const bool restart = (i == 0) || (a == 0) || (a % ND_RESTART == 0);
      const double k0 = (double)(r - g.N0 / 2), k1s = (double)(a * ND_RUN - g.N1 / 2);
#pragma unroll
      for (int j = 0; j < ND_FPPT; ++j) {
        if (restart) G[j] = nd_sincospi(-2.0 * fma(k0, xi0[j], k1s * xi1[j]));
        else G[j] = cmul(G[j], step[j]);
      }
      cplx in[ND_FPPT];
#pragma unroll
      for (int j = 0; j < ND_FPPT; ++j) in[j] = mk(0, 0);
#pragma unroll
      for (int t = 0; t < ND_RUN; ++t) {
        const cplx xv = xs[i * ND_RUN + t];
#pragma unroll
        for (int j = 0; j < ND_FPPT; ++j) in[j] = cfma(in[j], xv, P[j][t]);
      }
#pragma unroll
      for (int j = 0; j < ND_FPPT; ++j) acc[j] = cfma(acc[j], G[j], in[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < ND_FPPT; ++j) {
    const int64_t m = mbase + j * ND_FTHREADS;
    if (m < g.M) out[(int64_t)blockIdx.y * g.M + m] = acc[j];
  }
}

// fixed-order sum of the k-splits (one warp per output: lane l takes splits
// l, l+32, ..., then a shuffle tree -- deterministic) + optional operator
// epilogue (1D T, freq2wave.cpp:232-236): y_m = D_m acc + sum_c L_mc x_c +
// sum_c R_mc x_{n-p+c}; rec = [D, L_0..L_{p-1}, R_0..R_{p-1}] per point
__device__ __forceinline__ cplx nd_warp_split_sum(const cplx* __restrict__ part, int64_t stride, int nsplit, int64_t i) {
  const int lane = threadIdx.x & 31;
  cplx acc = mk(0, 0);
  for (int s = lane; s < nsplit; s += 32) acc = cadd(acc, part[(int64_t)s * stride + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_down_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_down_sync(0xffffffffu, acc.y, o);
  }
  return acc;
}

__global__ void k_ndft_fwd_reduce(int64_t M, int nsplit, const cplx* __restrict__ part, const cplx* __restrict__ rec,
                                  int p, int edges, const cplx* __restrict__ x, int n, cplx* __restrict__ y) {
  const int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (m >= M) return;
  part += (int64_t)blockIdx.y * nsplit * M;
  y += (int64_t)blockIdx.y * M;
  if (rec) {
    rec += (int64_t)blockIdx.y * M * (1 + (edges ? 2 * p : 0));
    x += (int64_t)blockIdx.y * n;
  }
  cplx acc = nd_warp_split_sum(part, M, nsplit, m);
  if ((threadIdx.x & 31) != 0) return;
  if (rec) {
    const int Rr = 1 + (edges ? 2 * p : 0);
    const cplx* r = rec + m * Rr;
    acc = cmul(r[0], acc);
    if (edges) {
      cplx a = mk(0, 0), c2 = mk(0, 0);
      for (int c = 0; c < p; ++c) a = cadd(a, cmul(r[1 + c], x[c]));
      for (int c = 0; c < p; ++c) c2 = cadd(c2, cmul(r[1 + p + c], x[n - p + c]));
      acc = cadd(acc, cadd(a, c2));
    }
  }
  y[m] = acc;
}

// ---------------------------------------------------------------- adjoint
// part[ms][mode]: a thread owns ND_AUPT consecutive units of one row; the CTA
// walks the points [m0, m1) of this blockIdx.y in staged tiles.
// rec (1D operator use): the staged sample value is conj(D_m) y_m.
template <int ND_AUPT>
__global__ void __launch_bounds__(ND_ATHREADS) k_ndft_adj(NdGeom g, const double* __restrict__ pts,
                                                           const cplx* __restrict__ y, const cplx* __restrict__ rec,
                                                           int Rr, int64_t points_per_split, cplx* __restrict__ out) {
  __shared__ cplx Ps[ND_ATILE * ND_RUN];
  __shared__ cplx vs[ND_ATILE], gs[ND_ATILE];
  __shared__ double x0s[ND_ATILE], x1s[ND_ATILE];
  pts += (int64_t)blockIdx.z * g.M * g.dim;
  y += (int64_t)blockIdx.z * g.M;
  if (rec) rec += (int64_t)blockIdx.z * g.M * Rr;
  out += (int64_t)blockIdx.z * gridDim.y * g.N0 * g.N1;
  const int groups_per_row = (g.runs + ND_AUPT - 1) / ND_AUPT;
  const int grp = blockIdx.x * ND_ATHREADS + threadIdx.x;
  const bool live = grp < g.N0 * groups_per_row;
  const int r = live ? grp / groups_per_row : 0;
  const int a0 = live ? (grp % groups_per_row) * ND_AUPT : 0;
  const double k0 = (double)(r - g.N0 / 2), k1s = (double)(a0 * ND_RUN - g.N1 / 2);
  const int64_t m0 = (int64_t)blockIdx.y * points_per_split;
  const int64_t m1 = min(g.M, m0 + points_per_split);
  cplx acc[ND_AUPT][ND_RUN];
#pragma unroll
  for (int u = 0; u < ND_AUPT; ++u)
#pragma unroll
    for (int t = 0; t < ND_RUN; ++t) acc[u][t] = mk(0, 0);
  for (int64_t mt = m0; mt < m1; mt += ND_ATILE) {
    const int np = (int)min((int64_t)ND_ATILE, m1 - mt);
    __syncthreads();
    for (int i = threadIdx.x; i < np; i += ND_ATHREADS) {
      double a, b;
      nd_point(g, pts, mt + i, a, b);
      x0s[i] = a;
      x1s[i] = b;
      cplx v = y[mt + i];
      if (rec) v = cmul(conj_(rec[(mt + i) * Rr]), v);
      vs[i] = v;
      gs[i] = nd_sincospi(2.0 * (double)ND_RUN * b);  // giant step along the row
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np * ND_RUN; i += ND_ATHREADS) {
      const int pi = i / ND_RUN, t = i % ND_RUN;
      Ps[i] = nd_sincospi(2.0 * (double)t * x1s[pi]);
    }
    __syncthreads();
    if (live) {
      for (int i = 0; i < np; ++i) {
        cplx v = cmul(vs[i], nd_sincospi(2.0 * fma(k0, x0s[i], k1s * x1s[i])));
        const cplx gstep = gs[i];
#pragma unroll
        for (int u = 0; u < ND_AUPT; ++u) {
#pragma unroll
          for (int t = 0; t < ND_RUN; ++t) acc[u][t] = cfma(acc[u][t], v, Ps[i * ND_RUN + t]);
          if (u + 1 < ND_AUPT) v = cmul(v, gstep);
        }
      }
    }
  }
  if (!live) return;
  const int64_t nmodes = (int64_t)g.N0 * g.N1;
#pragma unroll
  for (int u = 0; u < ND_AUPT; ++u)
#pragma unroll
    for (int t = 0; t < ND_RUN; ++t) {
      const int k1i = (a0 + u) * ND_RUN + t;
      if (a0 + u < g.runs && k1i < g.N1)
        out[(int64_t)blockIdx.y * nmodes + (int64_t)r * g.N1 + k1i] =
            (k1i < g.kh1 && r < g.rh0) ? acc[u][t] : mk(0, 0);
    }
}

// fixed-order sum of the point splits (one warp per mode); 1D operator use
// keeps only [lo, hi) (edge slots are filled by k_ndft_adj_edges)
__global__ void k_ndft_adj_reduce(int64_t nmodes, int nsplit, const cplx* __restrict__ part, int lo, int hi,
                                  cplx* __restrict__ z) {
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= nmodes) return;
  if (k < lo || k >= hi) return;
  part += (int64_t)blockIdx.y * nsplit * nmodes;
  z += (int64_t)blockIdx.y * nmodes;
  const cplx acc = nd_warp_split_sum(part, nmodes, nsplit, k);
  if ((threadIdx.x & 31) == 0) z[k] = acc;
}

// edge columns of the 1D adjoint: z_c = sum_m conj(L_mc) y_m, z_{n-p+c} = sum_m conj(R_mc) y_m
// (freq2wave.cpp:318-324); one CTA per edge column, fixed-order block reduction
__global__ void k_ndft_adj_edges(int64_t M, const cplx* __restrict__ rec, int p, const cplx* __restrict__ y, int n,
                                 cplx* __restrict__ z) {
  __shared__ double red[32];
  const int col = blockIdx.x;  // 0..2p-1
  const int Rr = 1 + 2 * p;
  rec += (int64_t)blockIdx.y * M * Rr;
  y += (int64_t)blockIdx.y * M;
  z += (int64_t)blockIdx.y * n;
  cplx acc = mk(0, 0);
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x) acc = cadd(acc, cmul(conj_(rec[m * Rr + 1 + col]), y[m]));
  const double re = block_sum(acc.x, red);
  __syncthreads();
  const double im = block_sum(acc.y, red);
  if (threadIdx.x == 0) z[col < p ? col : n - p + (col - p)] = mk(re, im);
}
