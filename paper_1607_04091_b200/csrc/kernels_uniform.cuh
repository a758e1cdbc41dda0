// kernels_uniform.cuh -- exact uniform-grid route (K-U / K-U*):
// one CTA per vector does embed+phase -> shared-memory FFT of length N2 ->
// output phase -> D (+ L/R edge terms) entirely on chip.  Restates
// uniform_ndft_fft / uniform_ndft_adjoint_fft (nufft.cpp:383-459) fused with
// the 1D apply_forward / apply_adjoint bodies (freq2wave.cpp:223-238, 313-326).
// Strided in/out lets the same kernels run both passes of the exact 2D tensor
// route T = T_x (x) T_y on a uniform tensor grid.
#pragma once
#include "gs_common.cuh"
#include "kernels_vec.cuh"

struct UniP {
  int n;          // coefficients per vector (N = 2^J)
  int M;          // samples per vector
  int q, N2, logN2;  // zero-embedding factor, DFT length, log2 (or -1: direct DFT)
  int p, edges;   // family p, edges = p >= 2
  double eps;     // uniform_epsilon
  double phase_step;  // pi * eps * M / N  (nufft.cpp:412)
  // phase tables built at construction (host libm, same arguments as the reference):
  // ph_in[l] = e^{i phase_step l} (nufft.cpp:414), ph_out[m] = e^{i pi N xi_m} (nufft.cpp:427)
  const cplx* ph_in;
  const cplx* ph_out;
};

constexpr int UNI_MAX_WARPS = 16;  // k_uni_* run 256 threads, the fused CGLS iteration 512

struct Strided {
  int64_t prob, vec, elem;  // strides in complex elements
};

// y = D o (e^{i pi N xi} FFT_{-}(z)) + L x_head + R x_tail
// (device body: one CTA per (vec, prob); the caller owns the shared buffer sm)
__device__ __forceinline__ void uni_fwd_body(const UniP& P, const cplx* __restrict__ x, Strided xs,
                                             const cplx* __restrict__ rec, int64_t rec_prob, cplx* __restrict__ y,
                                             Strided ys, const double* __restrict__ post, int64_t post_prob,
                                             const cplx* __restrict__ tw, int logLmax, int vec, int prob, cplx* sm) {
  x += prob * xs.prob + vec * xs.vec;
  y += prob * ys.prob + vec * ys.vec;
  rec += prob * rec_prob;
  if (post) post += prob * post_prob + vec * ys.vec;
  const bool pow2 = P.logN2 >= 0;
  const int R = 1 + (P.edges ? 2 * P.p : 0);
  const int slots = pow2 ? fpad_len(P.N2) : P.N2;  // power-of-two lengths use the padded FFT layout
  for (int i = threadIdx.x; i < slots; i += blockDim.x) sm[i] = mk(0, 0);
  __syncthreads();
  for (int l = threadIdx.x; l < P.n; l += blockDim.x) {
    cplx v = x[l * xs.elem];
    if (P.edges && (l < P.p || l >= P.n - P.p)) v = mk(0, 0);  // freq2wave.cpp:224-230
    cplx z = cmul(v, ldg2(P.ph_in + l));
    int pos = P.q * l;
    sm[pow2 ? fpad(bitrev(pos, P.logN2)) : pos] = z;
  }
  __syncthreads();
  cplx* Z = sm;
  if (pow2) {
    block_fft_padded<true>(sm, P.logN2, 1, 0, tw, logLmax, -1);  // tw: the staged table
  } else {
    block_dft(sm, sm + P.N2, P.N2, -1);
    Z = sm + P.N2;
  }
  cplx xh[8], xt[8];  // fixed-trip unrolled loops with a p predicate keep these in registers
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const bool on = P.edges && c < P.p;
    xh[c] = on ? x[c * xs.elem] : mk(0, 0);
    xt[c] = on ? x[(P.n - P.p + c) * xs.elem] : mk(0, 0);
  }
  for (int m = threadIdx.x; m < P.M; m += blockDim.x) {
    cplx o = cmul(ldg2(P.ph_out + m), Z[pow2 ? fpad(m) : m]);
    const cplx* r = rec + (int64_t)m * R;
    cplx ym = cmul(r[0], o);
    if (P.edges) {
      cplx a = mk(0, 0), b = mk(0, 0);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < P.p) a = cadd(a, cmul(r[1 + c], xh[c]));
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < P.p) b = cadd(b, cmul(r[1 + P.p + c], xt[c]));
      ym = cadd(ym, cadd(a, b));
    }
    if (post) ym = cscale(ym, post[m * ys.elem]);
    y[m * ys.elem] = ym;
  }
}

// <= 128 registers: 2 CTAs of 256 or 4 of 128 threads per SM (the tensor route
// launches 256-512 CTAs of 128 threads: one wave on 148 SMs)
__global__ void __launch_bounds__(256, 2) k_uni_fwd(UniP P, const cplx* __restrict__ x, Strided xs, const cplx* __restrict__ rec,
                          int64_t rec_prob, cplx* __restrict__ y, Strided ys, const double* __restrict__ post,
                          int64_t post_prob, const cplx* __restrict__ tw, int logLmax, double* npart,
                          UniPre upd) {
  extern __shared__ cplx sm[];  // FFT buffer + (power-of-two N2) N2/2 staged twiddles
  if (upd.st) {  // CGLS update of the vector this CTA owns (its input when mode 1)
    uni_pre_apply(upd, blockIdx.x, blockIdx.y);
    __syncthreads();
  }
  const cplx* twf = tw;
  if (P.logN2 >= 0) {  // visible after the body's first barrier
    stage_twiddles(sm + fpad_len(P.N2), tw, P.logN2, logLmax);
    twf = sm + fpad_len(P.N2);
    logLmax = P.logN2;
  }
  uni_fwd_body(P, x, xs, rec, rec_prob, y, ys, post, post_prob, twf, logLmax, blockIdx.x, blockIdx.y, sm);
  if (npart) {  // ||y_vec||^2 of this CTA's output vector (each thread re-reads the entries it wrote)
    __shared__ double red[32];
    const cplx* yv = y + blockIdx.y * ys.prob + blockIdx.x * ys.vec;
    double acc = 0.0;
    for (int m = threadIdx.x; m < P.M; m += blockDim.x) {
      const cplx a = yv[m * ys.elem];
      acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
    const double v = block_sum(acc, red);
    if (threadIdx.x == 0) npart[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = v;
  }
}

// z = gather_q(FFT_{+}(e^{-i pi N xi} conj(D) o u)) e^{-i phase l}, edge slots
// replaced by L^H u / R^H u.   u = pre o y  (pre = sqrt(mu) on the tensor route)
__device__ __forceinline__ void uni_adj_body(const UniP& P, const cplx* __restrict__ y, Strided ys,
                                             const double* __restrict__ pre, int64_t pre_prob,
                                             const cplx* __restrict__ rec, int64_t rec_prob, cplx* __restrict__ z,
                                             Strided zs, const cplx* __restrict__ tw, int logLmax, int vec, int prob,
                                             cplx* sm, double* ered) {
  y += prob * ys.prob + vec * ys.vec;
  z += prob * zs.prob + vec * zs.vec;
  rec += prob * rec_prob;
  if (pre) pre += prob * pre_prob + vec * ys.vec;
  const bool pow2 = P.logN2 >= 0;
  const int R = 1 + (P.edges ? 2 * P.p : 0);
  const int slots = pow2 ? fpad_len(P.N2) : P.N2;
  for (int i = threadIdx.x; i < slots; i += blockDim.x) sm[i] = mk(0, 0);
  __syncthreads();
  cplx eh[8], et[8];
  for (int c = 0; c < 8; ++c) eh[c] = et[c] = mk(0, 0);
  for (int m = threadIdx.x; m < P.M; m += blockDim.x) {
    cplx u = y[m * ys.elem];
    if (pre) u = cscale(u, pre[m * ys.elem]);
    const cplx* r = rec + (int64_t)m * R;
    cplx v = cmul(conj_(r[0]), u);  // freq2wave.cpp:315
    cplx val = cmul(v, conj_(ldg2(P.ph_out + m)));  // e^{-i pi N xi_m}, nufft.cpp:443-445
    sm[pow2 ? fpad(bitrev(m, P.logN2)) : m] = val;
    if (P.edges)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < P.p) {
          eh[c] = cadd(eh[c], cmul(conj_(r[1 + c]), u));
          et[c] = cadd(et[c], cmul(conj_(r[1 + P.p + c]), u));
        }
  }
  __syncthreads();
  cplx* Z = sm;
  if (pow2) {
    block_fft_padded<true>(sm, P.logN2, 1, 0, tw, logLmax, +1);  // tw: the staged table
  } else {
    block_dft(sm, sm + P.N2, P.N2, +1);
    Z = sm + P.N2;
  }
  for (int l = threadIdx.x; l < P.n; l += blockDim.x) {
    cplx v = cmul(Z[pow2 ? fpad(P.q * l) : P.q * l], conj_(ldg2(P.ph_in + l)));
    if (P.edges && (l < P.p || l >= P.n - P.p)) v = mk(0, 0);  // freq2wave.cpp:318-321
    z[l * zs.elem] = v;
  }
  if (P.edges) {
    // block reductions of L^H u, R^H u (freq2wave.cpp:323-324): warp sums of
    // all 4p components, one barrier, then thread k < 4p folds component k
    // over the warps in a fixed order (ered: >= 32 doubles per warp)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < P.p) {
        const double v0 = warp_sum(eh[c].x), v1 = warp_sum(eh[c].y);
        const double v2 = warp_sum(et[c].x), v3 = warp_sum(et[c].y);
        if (lane == 0) {
          ered[wid * 32 + 4 * c + 0] = v0;
          ered[wid * 32 + 4 * c + 1] = v1;
          ered[wid * 32 + 4 * c + 2] = v2;
          ered[wid * 32 + 4 * c + 3] = v3;
        }
      }
    __syncthreads();  // also orders the zero writes of the edge slots above before the sums below
    if (threadIdx.x < 4 * P.p) {
      double a = 0.0;
      for (int w = 0; w < nw; ++w) a += ered[w * 32 + threadIdx.x];
      const int c = threadIdx.x >> 2, comp = threadIdx.x & 3;
      const int idx = comp < 2 ? c : P.n - P.p + c;
      reinterpret_cast<double*>(z + idx * zs.elem)[comp & 1] = a;
    }
  }
}

__global__ void __launch_bounds__(256, 2) k_uni_adj(UniP P, const cplx* __restrict__ y, Strided ys, const double* __restrict__ pre,
                          int64_t pre_prob, const cplx* __restrict__ rec, int64_t rec_prob,
                          cplx* __restrict__ z, Strided zs, const cplx* __restrict__ tw, int logLmax,
                          double* npart, UniPre upd) {
  extern __shared__ cplx sm[];  // FFT buffer + (power-of-two N2) N2/2 staged twiddles
  __shared__ double ered[UNI_MAX_WARPS * 32];
  if (upd.st) {  // CGLS update of a vector this CTA owns (its input when mode 2)
    uni_pre_apply(upd, blockIdx.x, blockIdx.y);
    __syncthreads();
  }
  const cplx* twf = tw;
  if (P.logN2 >= 0) {  // visible after the body's first barrier
    stage_twiddles(sm + fpad_len(P.N2), tw, P.logN2, logLmax);
    twf = sm + fpad_len(P.N2);
    logLmax = P.logN2;
  }
  uni_adj_body(P, y, ys, pre, pre_prob, rec, rec_prob, z, zs, twf, logLmax, blockIdx.x, blockIdx.y, sm, ered);
  if (npart) {  // ||z_vec||^2 of this CTA's output vector
    __syncthreads();  // edge slots written by other threads
    const cplx* zv = z + blockIdx.y * zs.prob + blockIdx.x * zs.vec;
    double acc = 0.0;
    for (int l = threadIdx.x; l < P.n; l += blockDim.x) {
      const cplx a = zv[l * zs.elem];
      acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
    const double v = block_sum(acc, ered);
    if (threadIdx.x == 0) npart[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = v;
  }
}
