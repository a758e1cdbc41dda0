// gs_common.cuh -- complex128 helpers, shared-memory FFT, block reductions.
// Everything here is FP64: the path computes in complex128 (BASELINE north star).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define GS_PI 3.141592653589793238462643383279502884
#define GS_TWO_PI (2.0 * GS_PI)

typedef double2 cplx;

__host__ __device__ __forceinline__ cplx mk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
// (a.x + i a.y)(b.x + i b.y): same operation order as the textbook formula
// libstdc++ uses on the fast path (ac - bd, ad + bc).
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ cplx conj_(cplx a) { return mk(a.x, -a.y); }
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return mk(a.x * s, a.y * s); }
// acc += w * v  (real weight)
__host__ __device__ __forceinline__ cplx caxpy(cplx acc, double w, cplx v) {
  return mk(fma(w, v.x, acc.x), fma(w, v.y, acc.y));
}
__device__ __forceinline__ cplx polar1(double theta) {  // std::polar(1.0, theta)
  double s, c;
  sincos(theta, &s, &c);
  return mk(c, s);
}
__device__ __forceinline__ cplx ldg2(const cplx* p) { return __ldg(p); }

// ---------------------------------------------------------------------------
// In-place radix-2 DIT FFT in shared memory over `count` independent lines of
// length L = 2^logL stored at buf + c*lstride (element stride 1), input already
// in bit-reversed order.  Unnormalised; sign -1 = FFTW_FORWARD, +1 = BACKWARD
// (nufft.cpp:51-54 semantics).  tw[k] = exp(-2 pi i k / Lmax), k < Lmax/2.
// Each stage pairs radix-2 butterflies across all threads of the block.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void block_fft_bitrev(cplx* buf, int logL, int count, int lstride,
                                                 const cplx* __restrict__ tw, int logLmax, int sign) {
  const int L = 1 << logL;
  const int half = L >> 1;
  const int total = count * half;
  for (int s = 1; s <= logL; ++s) {
    const int h = 1 << (s - 1);           // half-size of current sub-transforms
    const int twshift = logLmax - s;      // twiddle index stride = Lmax / (2h)
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int c = t / half;
      const int j = t - c * half;
      const int k = j & (h - 1);
      const int i0 = ((j >> (s - 1)) << s) + k;
      cplx* base = buf + c * lstride;
      cplx w = ldg2(tw + (k << twshift));
      if (sign > 0) w.y = -w.y;
      cplx u = base[i0];
      cplx v = cmul(base[i0 + h], w);
      base[i0] = cadd(u, v);
      base[i0 + h] = csub(u, v);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Same transform as block_fft_bitrev (bit-reversed input, natural output,
// identical butterflies and twiddles in the same stage order -> bit-identical
// results) with three radix-2 stages fused per pass in registers: a thread
// loads 8 elements at stride h, runs stages s, s+1, s+2 on them and stores
// them back, so a 512-point line takes 3 shared-memory round trips and 3
// barriers instead of 9.  Element i of line c lives at buf[c*lstride + fpad(i)]
// (one pad slot per 8 elements keeps the stride-8 first pass conflict-free).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int fpad(int i) { return i + (i >> 3); }
__host__ __device__ __forceinline__ int fpad_len(int L) { return L + (L >> 3); }

// TWS: tw points to shared memory (staged table; a generic load, since
// ld.global.nc on a shared address faults) instead of the global table
template <int NST, bool TWS = false>
__device__ __forceinline__ void fft_fused_pass(cplx* buf, int logL, int s, int count, int lstride,
                                               const cplx* __restrict__ tw, int logLmax, int sign) {
  constexpr int G = 1 << NST;
  const int h = 1 << (s - 1);
  const int per = (1 << logL) / G;
  const int groups = count * per;
  for (int t = threadIdx.x; t < groups; t += blockDim.x) {
    const int c = t / per, j = t - c * per;
    const int jh = j & (h - 1);
    const int i0 = (j >> (s - 1)) * (G * h) + jh;
    cplx* base = buf + c * lstride;
    cplx v[G];
#pragma unroll
    for (int m = 0; m < G; ++m) v[m] = base[fpad(i0 + m * h)];
#pragma unroll
    for (int q = 0; q < NST; ++q) {
      const int twshift = logLmax - (s + q);
#pragma unroll
      for (int m = 0; m < G; ++m) {
        if ((m >> q) & 1) continue;
        const int k = jh + (m & ((1 << q) - 1)) * h;
        cplx w = TWS ? tw[k << twshift] : ldg2(tw + (k << twshift));
        if (sign > 0) w.y = -w.y;
        const cplx u = v[m], x = cmul(v[m + (1 << q)], w);
        v[m] = cadd(u, x);
        v[m + (1 << q)] = csub(u, x);
      }
    }
#pragma unroll
    for (int m = 0; m < G; ++m) base[fpad(i0 + m * h)] = v[m];
  }
}

template <bool TWS = false>
__device__ __forceinline__ void block_fft_padded(cplx* buf, int logL, int count, int lstride,
                                                 const cplx* __restrict__ tw, int logLmax, int sign) {
  int s = 1;
  while (s <= logL) {
    const int nst = logL - s + 1 >= 3 ? 3 : logL - s + 1;
    if (nst == 3) fft_fused_pass<3, TWS>(buf, logL, s, count, lstride, tw, logLmax, sign);
    else if (nst == 2) fft_fused_pass<2, TWS>(buf, logL, s, count, lstride, tw, logLmax, sign);
    else fft_fused_pass<1, TWS>(buf, logL, s, count, lstride, tw, logLmax, sign);
    __syncthreads();
    s += nst;
  }
}

// compact twiddle table of one FFT length 2^logL (entries k < 2^logL / 2) out of
// the 2^logLmax device table, for block_fft_padded(..., tws, logL, ...) from
// shared memory (caller synchronises before use)
__device__ __forceinline__ void stage_twiddles(cplx* tws, const cplx* __restrict__ tw, int logL, int logLmax) {
  for (int k = threadIdx.x; k < (1 << logL) / 2; k += blockDim.x) tws[k] = ldg2(tw + ((int64_t)k << (logLmax - logL)));
}

__device__ __forceinline__ int bitrev(int i, int logL) { return (int)(__brev((unsigned)i) >> (32 - logL)); }

// Direct DFT fallback (non power-of-two lengths, uniform route only):
// out[k] = sum_j in[j] exp(sign 2 pi i jk / L).
__device__ inline void block_dft(const cplx* in, cplx* out, int L, int sign) {
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    cplx acc = mk(0, 0);
    for (int j = 0; j < L; ++j) {
      long long jk = ((long long)j * k) % L;
      cplx w = polar1(sign * GS_TWO_PI * (double)jk / (double)L);
      acc = cadd(acc, cmul(in[j], w));
    }
    out[k] = acc;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Block reduction of a double (deterministic order for a fixed launch shape).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline double block_sum(double v, double* scratch /* >= 32 doubles */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  if (threadIdx.x == 0) scratch[0] = r;
  __syncthreads();
  r = scratch[0];
  __syncthreads();
  return r;
}
