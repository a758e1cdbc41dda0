// kernels_cgls_fused.cuh -- a whole CGLS iteration (solver.cpp:70-88) in ONE
// launch for the 1D uniform route: one CTA per problem runs
//   q = T p, qq = ||q||^2, alpha = gamma / qq, x += alpha p, r -= alpha q,
//   s = T* r, gamma' = ||s||^2, history / tolerance, beta, p = s + beta p
// with the T / T* bodies of kernels_uniform.cuh (shared-memory FFT) and the
// scalar steps of kernels_vec.cuh (same CgState semantics as k_cg_alpha /
// k_cg_beta / k_axpy_alpha / k_pupdate).  A 1D problem is a few KB-MB that
// one SM holds; the ~11 dependent launches of the generic iteration cost more
// than the arithmetic, so the graph-captured iteration becomes one kernel.
#pragma once
#include "kernels_uniform.cuh"
#include "kernels_vec.cuh"

constexpr int UNI_CG_THREADS = 512;
// (the q-step / s-step device functions live in kernels_vec.cuh)

// `iters` whole 1D-uniform iterations, one CTA per problem, in one launch:
// the twiddles of the length-N2 FFT are staged in shared memory once and the
// problem's vectors stay L1/L2-hot between iterations; a problem that stops
// (tolerance, qq == 0) leaves the loop with its state written like the
// generic kernels would.  Dynamic smem: uni_smem(P) + N2/2 twiddles.
__global__ void __launch_bounds__(UNI_CG_THREADS)
k_uni_cgls_iter(UniP P, const cplx* __restrict__ rec, int64_t rec_prob, cplx* __restrict__ x, cplx* __restrict__ p,
                cplx* __restrict__ s, cplx* __restrict__ r, cplx* __restrict__ q, CgState* st, double tol,
                double* hist, int hist_stride, const cplx* __restrict__ tw, int logLmax, int iters) {
  extern __shared__ cplx sm[];
  __shared__ double red[UNI_MAX_WARPS * 32];
  const int prob = blockIdx.x;
  CgState cs = st[prob];  // every thread holds the same state: the branches below are CTA-uniform
  if (!cs.active) return;
  const int n = P.n, M = P.M;
  const bool pow2 = P.logN2 >= 0;
  const cplx* twf = tw;
  int logTw = logLmax;
  if (pow2) {  // compact twiddle table of length N2/2 after the FFT buffer
    cplx* tws = sm + fpad_len(P.N2);
    stage_twiddles(tws, tw, P.logN2, logLmax);
    __syncthreads();
    twf = tws;
    logTw = P.logN2;
  }
  cplx* pp = p + (int64_t)prob * n;
  cplx* sp = s + (int64_t)prob * n;
  double* hrow = hist ? hist + (int64_t)prob * hist_stride : nullptr;
  for (int it = 0; it < iters && cs.active; ++it) {
    // q = T p   (k_uni_fwd); the q-step reads back only the q entries each thread wrote
    uni_fwd_body(P, p, Strided{n, 0, 1}, rec, rec_prob, q, Strided{M, 0, 1}, nullptr, 0, twf, logTw, 0, prob, sm);
    if (!cg_qstep_dev(cs, st + prob, q + (int64_t)prob * M, r + (int64_t)prob * M, x + (int64_t)prob * n, pp, M, n,
                      red))
      return;
    __syncthreads();  // shared buffer reuse (and r written block-wide before the adjoint reads it)
    // s = T* r   (k_uni_adj)
    uni_adj_body(P, r, Strided{M, 0, 1}, nullptr, 0, rec, rec_prob, s, Strided{n, 0, 1}, twf, logTw, 0, prob, sm,
                 red);
    __syncthreads();  // edge slots of s visible block-wide
    cg_sstep_dev(cs, st + prob, sp, pp, n, tol, hrow, hist_stride, red);
    __syncthreads();  // p complete before the next forward; shared buffer reuse
  }
}
