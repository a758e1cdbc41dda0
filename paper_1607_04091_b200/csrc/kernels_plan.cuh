// kernels_plan.cuh -- the lower-level Kaiser-Bessel NfftPlan (nufft.cpp:138-365)
// on the device at any dim / even N / sigma >= 1.25 / w >= 2: deconvolve +
// embed, interpolation and spreading around the general FFT engine
// (kernels_fftg.cuh).  Same per-point tables as the reference: window origin
// base (here wrapped mod n_ov) and 2w+1 weights per axis, deconv per axis.
// Spreading uses FP64 atomics into the oversampled grid (this general path
// trades the fast kernels' owner-computes folds for any window width).
#pragma once
#include "gs_common.cuh"

struct PlanDev {
  int dim;
  int N0, N1;      // modes per axis (N1 = 1 in 1D)
  int n0, n1;      // oversampled lengths (n1 = 1 in 1D)
  int S;           // 2w + 1
  int64_t M;
  int vps;         // vectors per point set: blockIdx.y = set * vps + vector
  int lo, hi;      // embed mask: mode indices [lo, hi) of every axis enter (operator interiors); 0, N
};

// deconvolve and embed I_N into the zeroed oversampled grid (nufft.cpp:247-265)
__global__ void k_plan_embed(PlanDev P, const cplx* __restrict__ x, const double* __restrict__ dec0,
                             const double* __restrict__ dec1, cplx* __restrict__ G) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nm = (int64_t)P.N0 * P.N1;
  if (idx >= nm) return;
  const int b = blockIdx.y;
  x += (int64_t)b * nm;
  G += (int64_t)b * P.n0 * P.n1;
  if (P.dim == 1) {
    const int k = (int)idx - P.N0 / 2;
    const bool in = idx >= P.lo && idx < P.hi;
    G[(k + P.n0) % P.n0] = in ? cscale(x[idx], dec0[idx]) : mk(0, 0);
    return;
  }
  const int i0 = (int)(idx / P.N1), i1 = (int)(idx % P.N1);
  const int k0 = i0 - P.N0 / 2, k1 = i1 - P.N1 / 2;
  const bool in = i0 >= P.lo && i0 < P.hi && i1 >= P.lo && i1 < P.hi;
  G[(int64_t)((k0 + P.n0) % P.n0) * P.n1 + (k1 + P.n1) % P.n1] = in ? cscale(x[idx], dec0[i0] * dec1[i1]) : mk(0, 0);
}

// crop + deconvolve after the backward FFT (nufft.cpp:339-364)
__global__ void k_plan_crop(PlanDev P, const cplx* __restrict__ G, const double* __restrict__ dec0,
                            const double* __restrict__ dec1, cplx* __restrict__ z) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nm = (int64_t)P.N0 * P.N1;
  if (idx >= nm) return;
  const int b = blockIdx.y;
  z += (int64_t)b * nm;
  G += (int64_t)b * P.n0 * P.n1;
  if (P.dim == 1) {
    const int k = (int)idx - P.N0 / 2;
    z[idx] = cscale(G[(k + P.n0) % P.n0], dec0[idx]);
    return;
  }
  const int i0 = (int)(idx / P.N1), i1 = (int)(idx % P.N1);
  const int k0 = i0 - P.N0 / 2, k1 = i1 - P.N1 / 2;
  z[idx] = cscale(G[(int64_t)((k0 + P.n0) % P.n0) * P.n1 + (k1 + P.n1) % P.n1], dec0[i0] * dec1[i1]);
}

// interpolation (nufft.cpp:271-305): base already wrapped into [0, n)
__global__ void k_plan_interp(PlanDev P, const int* __restrict__ base, const double* __restrict__ wts,
                              const cplx* __restrict__ G, cplx* __restrict__ y) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= P.M) return;
  const int b = blockIdx.y;
  base += (int64_t)(b / P.vps) * P.M * P.dim;
  wts += (int64_t)(b / P.vps) * P.M * P.dim * P.S;
  G += (int64_t)b * P.n0 * P.n1;
  y += (int64_t)b * P.M;
  cplx acc = mk(0, 0);
  if (P.dim == 1) {
    const int b0 = base[m];
    const double* w = wts + m * P.S;
    for (int t = 0; t < P.S; ++t) {
      acc = caxpy(acc, w[t], G[(b0 + t) % P.n0]);
    }
  } else {
    const int b0 = base[2 * m], b1 = base[2 * m + 1];
    const double* w0 = wts + (2 * m) * P.S;
    const double* w1 = wts + (2 * m + 1) * P.S;
    for (int t0 = 0; t0 < P.S; ++t0) {
      const cplx* row = G + (int64_t)((b0 + t0) % P.n0) * P.n1;
      cplx ra = mk(0, 0);
      for (int t1 = 0; t1 < P.S; ++t1) ra = caxpy(ra, w1[t1], row[(b1 + t1) % P.n1]);
      acc = caxpy(acc, w0[t0], ra);
    }
  }
  y[m] = acc;
}

__device__ __forceinline__ void atomic_add_c(cplx* p, cplx v) {
  atomicAdd(&p->x, v.x);
  atomicAdd(&p->y, v.y);
}

// spreading (nufft.cpp:313-336), FP64 atomics into the zeroed grid
__global__ void k_plan_spread(PlanDev P, const int* __restrict__ base, const double* __restrict__ wts,
                              const cplx* __restrict__ v, cplx* __restrict__ G) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= P.M) return;
  const int b = blockIdx.y;
  base += (int64_t)(b / P.vps) * P.M * P.dim;
  wts += (int64_t)(b / P.vps) * P.M * P.dim * P.S;
  G += (int64_t)b * P.n0 * P.n1;
  const cplx s = v[(int64_t)b * P.M + m];
  if (P.dim == 1) {
    const int b0 = base[m];
    const double* w = wts + m * P.S;
    for (int t = 0; t < P.S; ++t) {
      atomic_add_c(G + (b0 + t) % P.n0, cscale(s, w[t]));
    }
    return;
  }
  const int b0 = base[2 * m], b1 = base[2 * m + 1];
  const double* w0 = wts + (2 * m) * P.S;
  const double* w1 = wts + (2 * m + 1) * P.S;
  for (int t0 = 0; t0 < P.S; ++t0) {
    const cplx v0 = cscale(s, w0[t0]);
    cplx* row = G + (int64_t)((b0 + t0) % P.n0) * P.n1;
    for (int t1 = 0; t1 < P.S; ++t1) atomic_add_c(row + (b1 + t1) % P.n1, cscale(v0, w1[t1]));
  }
}

// KB window of plan points (already scaled to [-1/2, 1/2); nufft.cpp:208-223),
// per point and axis: base = (llround(pos) - w) mod n_ov, S weights
__global__ void k_plan_window(const double* __restrict__ pts, int64_t count, int dim, int n0, int n1, int w,
                              double beta, int* __restrict__ base, double* __restrict__ wts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // point * dim + axis
  if (i >= count) return;
  const int axis = dim == 2 ? (int)(i % 2) : 0;
  const int n = axis == 0 ? n0 : n1;
  const int S = 2 * w + 1;
  const double pos = pts[i] * (double)n;
  const long long j0 = llround(pos);
  const long long b = j0 - w;
  base[i] = (int)(((b % n) + n) % n);
  for (int t = 0; t < S; ++t) {
    const double u = pos - (double)(j0 - w + t);
    const double q = 1.0 - (u / w) * (u / w);
    wts[i * S + t] = q < 0 ? 0.0 : cyl_bessel_i0(beta * sqrt(q));
  }
}
