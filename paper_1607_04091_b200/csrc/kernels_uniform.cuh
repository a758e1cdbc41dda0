// kernels_uniform.cuh -- exact uniform-grid route (K-U / K-U*):
// one CTA per vector does embed+phase -> shared-memory FFT of length N2 ->
// output phase -> D (+ L/R edge terms) entirely on chip.  Restates
// uniform_ndft_fft / uniform_ndft_adjoint_fft (nufft.cpp:383-459) fused with
// the 1D apply_forward / apply_adjoint bodies (freq2wave.cpp:223-238, 313-326).
// Strided in/out lets the same kernels run both passes of the exact 2D tensor
// route T = T_x (x) T_y on a uniform tensor grid.
#pragma once
#include "gs_common.cuh"

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

struct Strided {
  int64_t prob, vec, elem;  // strides in complex elements
};

// y = D o (e^{i pi N xi} FFT_{-}(z)) + L x_head + R x_tail
__global__ void k_uni_fwd(UniP P, const cplx* __restrict__ x, Strided xs, const cplx* __restrict__ rec,
                          int64_t rec_prob, cplx* __restrict__ y, Strided ys, const double* __restrict__ post,
                          int64_t post_prob, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  const int vec = blockIdx.x, prob = blockIdx.y;
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
    block_fft_padded(sm, P.logN2, 1, 0, tw, logLmax, -1);
  } else {
    block_dft(sm, sm + P.N2, P.N2, -1);
    Z = sm + P.N2;
  }
  cplx xh[8], xt[8];
  if (P.edges)
    for (int c = 0; c < P.p; ++c) {
      xh[c] = x[c * xs.elem];
      xt[c] = x[(P.n - P.p + c) * xs.elem];
    }
  for (int m = threadIdx.x; m < P.M; m += blockDim.x) {
    cplx o = cmul(ldg2(P.ph_out + m), Z[pow2 ? fpad(m) : m]);
    const cplx* r = rec + (int64_t)m * R;
    cplx ym = cmul(r[0], o);
    if (P.edges) {
      cplx a = mk(0, 0), b = mk(0, 0);
      for (int c = 0; c < P.p; ++c) a = cadd(a, cmul(r[1 + c], xh[c]));
      for (int c = 0; c < P.p; ++c) b = cadd(b, cmul(r[1 + P.p + c], xt[c]));
      ym = cadd(ym, cadd(a, b));
    }
    if (post) ym = cscale(ym, post[m * ys.elem]);
    y[m * ys.elem] = ym;
  }
}

// z = gather_q(FFT_{+}(e^{-i pi N xi} conj(D) o u)) e^{-i phase l}, edge slots
// replaced by L^H u / R^H u.   u = pre o y  (pre = sqrt(mu) on the tensor route)
__global__ void k_uni_adj(UniP P, const cplx* __restrict__ y, Strided ys, const double* __restrict__ pre,
                          int64_t pre_prob, const cplx* __restrict__ rec, int64_t rec_prob,
                          cplx* __restrict__ z, Strided zs, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  __shared__ double red[32];
  const int vec = blockIdx.x, prob = blockIdx.y;
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
      for (int c = 0; c < P.p; ++c) {
        eh[c] = cadd(eh[c], cmul(conj_(r[1 + c]), u));
        et[c] = cadd(et[c], cmul(conj_(r[1 + P.p + c]), u));
      }
  }
  __syncthreads();
  cplx* Z = sm;
  if (pow2) {
    block_fft_padded(sm, P.logN2, 1, 0, tw, logLmax, +1);
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
    // block reductions of L^H u, R^H u (freq2wave.cpp:323-324); all threads
    // participate in every block_sum, thread 0 writes after the last one.
    __syncthreads();
    for (int c = 0; c < P.p; ++c) {
      double hr = block_sum(eh[c].x, red), hi = block_sum(eh[c].y, red);
      double tr = block_sum(et[c].x, red), ti = block_sum(et[c].y, red);
      if (threadIdx.x == 0) {
        z[c * zs.elem] = mk(hr, hi);
        z[(P.n - P.p + c) * zs.elem] = mk(tr, ti);
      }
    }
  }
}
