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
// the twiddles of the length-N2 FFT are staged in shared memory once; with
// `resident` (host-checked: it fits) the problem's vectors p, x, r and its
// factor records also live in shared memory for the whole launch (q and s are
// produced there) and are written back at the end, so an iteration touches no
// global memory but the phase tables, history and state.  A problem that
// stops (tolerance, qq == 0) leaves the loop with its state written like the
// generic kernels would.  Dynamic smem: uni_smem_tw(P) [+ resident vectors].
__global__ void __launch_bounds__(UNI_CG_THREADS)
k_uni_cgls_iter(UniP P, const cplx* __restrict__ rec, int64_t rec_prob, cplx* __restrict__ x, cplx* __restrict__ p,
                cplx* __restrict__ s, cplx* __restrict__ r, cplx* __restrict__ q, CgState* st, double tol,
                double* hist, int hist_stride, const cplx* __restrict__ tw, int logLmax, int iters, int resident) {
  extern __shared__ cplx sm[];
  __shared__ double red[UNI_MAX_WARPS * 32];
  const int prob = blockIdx.x;
  CgState cs = st[prob];  // every thread holds the same state: the branches below are CTA-uniform
  if (!cs.active) return;
  const int n = P.n, M = P.M;
  const int R = 1 + (P.edges ? 2 * P.p : 0);
  const bool pow2 = P.logN2 >= 0;
  const cplx* twf = tw;
  int logTw = logLmax;
  const int buf = pow2 ? fpad_len(P.N2) + P.N2 / 2 : 2 * P.N2;  // FFT buffer (+ twiddles)
  if (pow2) {  // compact twiddle table of length N2/2 after the FFT buffer
    cplx* tws = sm + fpad_len(P.N2);
    stage_twiddles(tws, tw, P.logN2, logLmax);
    twf = tws;
    logTw = P.logN2;
  }
  cplx* gp = p + (int64_t)prob * n;
  cplx* gx = x + (int64_t)prob * n;
  cplx* gs = s + (int64_t)prob * n;
  cplx* gr = r + (int64_t)prob * M;
  cplx* gq = q + (int64_t)prob * M;
  const cplx* grec = rec + prob * rec_prob;
  cplx *vp = gp, *vx = gx, *vs = gs, *vr = gr, *vq = gq;
  const cplx* vrec = grec;
  if (resident) {
    vp = sm + buf;
    vx = vp + n;
    vs = vx + n;
    vr = vs + n;
    vq = vr + M;
    cplx* srec = vq + M;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      vp[i] = gp[i];
      vx[i] = gx[i];
    }
    for (int i = threadIdx.x; i < M; i += blockDim.x) vr[i] = gr[i];
    for (int i = threadIdx.x; i < M * R; i += blockDim.x) srec[i] = grec[i];
    vrec = srec;
  }
  __syncthreads();
  double* hrow = hist ? hist + (int64_t)prob * hist_stride : nullptr;
  bool wrote_q = false, wrote_s = false;
  for (int it = 0; it < iters && cs.active; ++it) {
    // q = T p   (k_uni_fwd); the q-step reads back only the q entries each thread wrote
    uni_fwd_body(P, vp, Strided{0, 0, 1}, vrec, 0, vq, Strided{0, 0, 1}, nullptr, 0, twf, logTw, 0, 0, sm);
    wrote_q = true;
    if (!cg_qstep_dev(cs, st + prob, vq, vr, vx, vp, M, n, red)) break;
    __syncthreads();  // shared buffer reuse (and r written block-wide before the adjoint reads it)
    // s = T* r   (k_uni_adj)
    uni_adj_body(P, vr, Strided{0, 0, 1}, nullptr, 0, vrec, 0, vs, Strided{0, 0, 1}, twf, logTw, 0, 0, sm, red);
    wrote_s = true;
    __syncthreads();  // edge slots of s visible block-wide
    cg_sstep_dev(cs, st + prob, vs, vp, n, tol, hrow, hist_stride, red);
    __syncthreads();  // p complete before the next forward; shared buffer reuse
  }
  if (resident) {  // write the session vectors back
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      gp[i] = vp[i];
      gx[i] = vx[i];
      if (wrote_s) gs[i] = vs[i];
    }
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      gr[i] = vr[i];
      if (wrote_q) gq[i] = vq[i];
    }
  }
}
