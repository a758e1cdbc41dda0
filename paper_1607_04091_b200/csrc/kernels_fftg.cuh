// kernels_fftg.cuh -- general-length FFT engine (any length, any radix) for
// the generic routes: the lower-level NfftPlan of nufft.cpp:138-365 at any
// sigma >= 1.25 / even N / kernel width, and the uniform-grid reduction
// (nufft.cpp:383-459) at any DFT length q N / epsilon.  The power-of-two
// fused kernels of the configs stay in kernels_nfft*.cuh / kernels_uniform.cuh.
//
// One CTA transforms G whole lines held in shared memory (two ping-pong
// buffers): mixed-radix Stockham autosort, L = p_1 p_2 ... p_s, stage radix p
// processed as L/p butterflies whose twiddle and DFT_p factors come from ONE
// table entry tw[(r (k L/(Ns p) + q L/p)) mod L] = e^{-2 pi i (...)/L}
// (correctly rounded host table), so any prime radix needs no special code.
// Lines are gathered / scattered with arbitrary element / line strides and an
// optional per-element twiddle pre-multiply (the four-step decomposition of
// lengths beyond one CTA: L = L1 L2, FFT_L1 on strided columns, twiddle,
// FFT_L2 on rows written transposed).
#pragma once
#include "gs_common.cuh"

#define FG_MAXF 32
#define FG_THREADS 256

struct FgLines {
  int L;             // line length
  int nf;            // number of radices
  int f[FG_MAXF];    // radices (product = L)
  const cplx* tw;    // tw[k] = e^{-2 pi i k / L}, k < L
  int sign;          // -1 forward (FFTW_FORWARD), +1 backward
  int G;             // lines per CTA
  int64_t nlines;    // lines in the launch
  // element (line l, index j) of the input: in + (l / per) * bstride + (l % per) * lstride + j * estride
  int64_t per, bstride, lstride, estride;
  int64_t obstride, olstride, oestride;  // same for the output
  // optional pre-twiddle of the four-step: element (l, j) *= e^{sign 2 pi i (l % per) j / Lpre}
  const cplx* pretw;  // table of length Lpre (tw of the full length), or nullptr
  int64_t Lpre;
};

__device__ __forceinline__ cplx fg_tw(const cplx* __restrict__ tw, int64_t idx, int sign) {
  cplx w = __ldg(tw + idx);
  if (sign > 0) w.y = -w.y;
  return w;
}

__global__ void __launch_bounds__(FG_THREADS) k_fftg_lines(FgLines P, const cplx* __restrict__ in,
                                                           cplx* __restrict__ out) {
  extern __shared__ cplx fg_sm[];
  const int L = P.L, G = P.G;
  cplx* b0 = fg_sm;
  cplx* b1 = fg_sm + (size_t)G * L;
  const int64_t l0 = (int64_t)blockIdx.x * G;
  const int ng = (int)min((int64_t)G, P.nlines - l0);
  // gather: consecutive threads take consecutive lines first (coalesced for column lines)
  for (int t = threadIdx.x; t < ng * L; t += blockDim.x) {
    const int gl = t % ng, j = t / ng;
    const int64_t l = l0 + gl;
    const int64_t b = l / P.per, lp = l % P.per;
    cplx v = in[b * P.bstride + lp * P.lstride + (int64_t)j * P.estride];
    if (P.pretw) v = cmul(v, fg_tw(P.pretw, (lp * j) % P.Lpre, P.sign));
    b0[(size_t)gl * L + j] = v;
  }
  __syncthreads();
  int Ns = 1;
  cplx* src = b0;
  cplx* dst = b1;
  for (int s = 0; s < P.nf; ++s) {
    const int p = P.f[s];
    const int Lp = L / p;
    const int step_k = L / (Ns * p);  // twiddle stride of k
    for (int t = threadIdx.x; t < ng * Lp; t += blockDim.x) {
      const int gl = t / Lp, j = t - gl * Lp;
      const int k = j % Ns;
      const cplx* a = src + (size_t)gl * L;
      cplx* o = dst + (size_t)gl * L + (j / Ns) * Ns * p + k;
      if (p == 2) {
        const cplx u = a[j];
        const cplx v = k ? cmul(a[j + Lp], fg_tw(P.tw, (int64_t)k * step_k, P.sign)) : a[j + Lp];
        o[0] = cadd(u, v);
        o[Ns] = csub(u, v);
      } else {
        for (int q = 0; q < p; ++q) {
          cplx acc = a[j];
          const int64_t base = (int64_t)k * step_k + (int64_t)q * Lp;  // per unit r
          for (int r = 1; r < p; ++r) acc = cadd(acc, cmul(a[j + r * Lp], fg_tw(P.tw, (r * base) % L, P.sign)));
          o[q * Ns] = acc;
        }
      }
    }
    __syncthreads();
    Ns *= p;
    cplx* tmp = src;
    src = dst;
    dst = tmp;
  }
  for (int t = threadIdx.x; t < ng * L; t += blockDim.x) {
    const int gl = t % ng, j = t / ng;
    const int64_t l = l0 + gl;
    const int64_t b = l / P.per, lp = l % P.per;
    out[b * P.obstride + lp * P.olstride + (int64_t)j * P.oestride] = src[(size_t)gl * L + j];
  }
}
