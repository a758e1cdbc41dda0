// kernels_vec.cuh -- CGLS vector algebra kept on the device (solver.cpp:19-91):
// per-problem norms (deterministic block reductions), the alpha / beta scalar
// steps, and the fused axpys.  Every kernel is batched over independent
// problems and honours the per-problem `active` flag, so converged problems
// freeze while the rest of the batch keeps iterating with no host round trip.
#pragma once
#include "gs_common.cuh"

struct CgState {
  double ref;      // ||T* b||
  double gamma;    // ||s||^2 of the current residual
  double gamma_new;
  double qq;
  double alpha, beta;
  int active;      // 1 while iterating
  int iterations;
  int converged;
  int hist_len;
  double pend_alpha;  // 1D NFFT fused q-step: alpha of the r update the next interpolation applies
  double pend_beta;   // tensor route: p = s + pend_beta p still to apply (pend_p) by the next x-pass
  int pend_p;
};

// a vector update one CTA of a tensor-route pass applies to the vector it owns
// before its transform (the CGLS axpys without launches of their own):
//   mode 1: v = w + pend_beta v (if pend_p)     -- p = s + beta p, deferred
//   mode 2: v = v - alpha w     (if active)     -- r -= alpha q
//   mode 3: v = v + alpha w     (if active)     -- x += alpha p
struct UniPre {
  const CgState* st;
  int mode;
  cplx* v;
  const cplx* w;
  int64_t sprob, svec, selem;  // strides of v and w (same layout)
  int len;
};
__device__ __forceinline__ void uni_pre_apply(const UniPre& u, int vec, int prob) {
  const CgState& c = u.st[prob];
  double a;
  if (u.mode == 1) {
    if (!c.pend_p) return;
    a = c.pend_beta;
  } else {
    if (!c.active) return;
    a = u.mode == 2 ? -c.alpha : c.alpha;
  }
  cplx* v = u.v + prob * u.sprob + vec * u.svec;
  const cplx* w = u.w + prob * u.sprob + vec * u.svec;
  for (int i = threadIdx.x; i < u.len; i += blockDim.x) {
    const cplx vv = v[i * u.selem], ww = w[i * u.selem];
    v[i * u.selem] = u.mode == 1 ? mk(fma(a, vv.x, ww.x), fma(a, vv.y, ww.y))
                                 : mk(fma(a, ww.x, vv.x), fma(a, ww.y, vv.y));
  }
}

// out[prob] = sum |v|^2 over len entries (one block per problem; fixed order)
__global__ void k_norm2(const cplx* __restrict__ v, int64_t len, double* __restrict__ out) {
  __shared__ double red[32];
  const int prob = blockIdx.x;
  v += prob * len;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
    cplx a = v[i];
    acc = fma(a.x, a.x, fma(a.y, a.y, acc));
  }
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) out[prob] = s;
}

// two-level variant for long vectors: partial sums per (prob, chunk)
__global__ void k_norm2_part(const cplx* __restrict__ v, int64_t len, int chunks, double* __restrict__ part) {
  __shared__ double red[32];
  const int prob = blockIdx.y, ch = blockIdx.x;
  const int64_t per = (len + chunks - 1) / chunks;
  const int64_t lo = ch * per, hi = min(len, lo + per);
  v += prob * len;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    cplx a = v[i];
    acc = fma(a.x, a.x, fma(a.y, a.y, acc));
  }
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[(int64_t)prob * chunks + ch] = s;
}
__global__ void k_norm2_fold(const double* __restrict__ part, int chunks, int B, double* __restrict__ out) {
  const int prob = blockIdx.x * blockDim.x + threadIdx.x;
  if (prob >= B) return;
  double a = 0.0;  // sequential fold keeps the order fixed
  for (int c = 0; c < chunks; ++c) a += part[(int64_t)prob * chunks + c];
  out[prob] = a;
}

// b_s[prob][s] = sqrtw_s * b_raw[prob][perm[s]]  (solver.cpp:30-33, sorted order)
__global__ void k_gather_scale(const cplx* __restrict__ b, const int* __restrict__ perm, const double* __restrict__ sw,
                               int64_t M, int B, cplx* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * B) return;
  const int64_t prob = i / M;
  const int64_t src = perm ? prob * M + perm[i] : i;
  cplx v = b[src];
  if (sw) v = cscale(v, sw[i]);
  out[i] = v;
}

// r = b - tx
__global__ void k_sub(const cplx* __restrict__ b, const cplx* __restrict__ tx, int64_t n, cplx* __restrict__ r) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) r[i] = csub(b[i], tx[i]);
}

// preamble: ref = sqrt(n2[0]); state init   (solver.cpp:42-48)
__global__ void k_cg_ref(CgState* st, const double* __restrict__ n2, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  CgState s;
  s.ref = sqrt(n2[b]);
  s.gamma = s.gamma_new = s.qq = s.alpha = s.beta = s.pend_alpha = s.pend_beta = 0.0;
  s.pend_p = 0;
  s.iterations = 0;
  s.converged = 0;
  s.hist_len = 0;
  s.active = 1;
  if (s.ref == 0.0) {  // zero data -> zero solution, converged, history {0}
    s.active = 0;
    s.converged = 1;
    s.hist_len = 1;
  }
  st[b] = s;
}

// gamma = ||s||^2; history[0]; tolerance test  (solver.cpp:55-62)
__global__ void k_cg_gamma0(CgState* st, const double* __restrict__ n2, double tol, double* hist, int hist_stride, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  CgState s = st[b];
  if (!s.active) {
    if (s.ref == 0.0 && hist) hist[(int64_t)b * hist_stride] = 0.0;
    return;
  }
  s.gamma = n2[b];
  double h = sqrt(s.gamma) / s.ref;
  if (hist) hist[(int64_t)b * hist_stride] = h;
  s.hist_len = 1;
  if (h <= tol) {
    s.converged = 1;
    s.active = 0;
  }
  st[b] = s;
}

// qq = ||q||^2; break on qq == 0; alpha = gamma / qq  (solver.cpp:71-74)
__device__ __forceinline__ void cg_alpha_dev(CgState& s, double qq) {
  s.qq = qq;
  if (s.qq == 0.0) {
    s.active = 0;  // search direction in the numerical null space
    s.alpha = 0.0;
  } else {
    s.alpha = s.gamma / s.qq;
  }
}
__global__ void k_cg_alpha(CgState* st, const double* __restrict__ n2, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  CgState s = st[b];
  if (!s.active) return;
  cg_alpha_dev(s, n2[b]);
  st[b] = s;
}

// gamma' = ||s||^2; history; tolerance; beta  (solver.cpp:77-87)
// (the iteration number lives on the device, so one captured CUDA graph replays
// every iteration)
__device__ __forceinline__ void cg_beta_dev(CgState& s, double gn, double tol, double* hist, int hist_stride, int b) {
  const int it = s.iterations + 1;
  s.iterations = it;
  double h = sqrt(gn) / s.ref;
  if (hist) hist[(int64_t)b * hist_stride + (it < hist_stride ? it : hist_stride - 1)] = h;
  s.hist_len = (it < hist_stride ? it : hist_stride - 1) + 1;
  if (h <= tol) {
    s.converged = 1;
    s.active = 0;
    s.beta = 0.0;
  } else {
    s.beta = gn / s.gamma;
    s.gamma = gn;
  }
}
__global__ void k_cg_beta(CgState* st, const double* __restrict__ n2, double tol, double* hist, int hist_stride,
                          int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  CgState s = st[b];
  if (!s.active) return;
  cg_beta_dev(s, n2[b], tol, hist, hist_stride, b);
  st[b] = s;
}

// the two-level norm's fold fused with the alpha / beta step (one launch less each)
__global__ void k_norm2_fold_alpha(const double* __restrict__ part, int chunks, int B, CgState* st) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  CgState s = st[b];
  if (!s.active) return;
  double a = 0.0;  // same sequential order as k_norm2_fold
  for (int c = 0; c < chunks; ++c) a += part[(int64_t)b * chunks + c];
  cg_alpha_dev(s, a);
  st[b] = s;
}
__global__ void k_norm2_fold_beta(const double* __restrict__ part, int chunks, int B, CgState* st, double tol,
                                  double* hist, int hist_stride) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  CgState s = st[b];
  if (!s.active) return;
  double a = 0.0;
  for (int c = 0; c < chunks; ++c) a += part[(int64_t)b * chunks + c];
  cg_beta_dev(s, a, tol, hist, hist_stride, b);
  st[b] = s;
}

// many-partial folds (the tensor route's per-vector norms): one warp per
// problem, lane-strided sums then a fixed-order warp reduction
__device__ __forceinline__ double fold_warp(const double* __restrict__ part, int chunks) {
  double a = 0.0;
  for (int c = threadIdx.x; c < chunks; c += 32) a += part[c];
  return warp_sum(a);
}
__global__ void k_fold_alpha_w(const double* __restrict__ part, int chunks, CgState* st) {
  const int b = blockIdx.x;
  const double qq = fold_warp(part + (int64_t)b * chunks, chunks);
  if (threadIdx.x) return;
  CgState s = st[b];
  s.pend_p = 0;  // the x-pass of this iteration has applied it
  if (s.active) cg_alpha_dev(s, qq);
  st[b] = s;
}
__global__ void k_fold_beta_w(const double* __restrict__ part, int chunks, CgState* st, double tol, double* hist,
                              int hist_stride) {
  const int b = blockIdx.x;
  const double gn = fold_warp(part + (int64_t)b * chunks, chunks);
  if (threadIdx.x) return;
  CgState s = st[b];
  if (!s.active) return;
  cg_beta_dev(s, gn, tol, hist, hist_stride, b);
  s.pend_p = s.active;  // p = s + beta p, applied by the next x-pass (k_uni_fwd UniPre mode 1)
  s.pend_beta = s.beta;
  st[b] = s;
}

// x += alpha p (first lenx * B entries of the grid) and r -= alpha q (the next
// lenr * B) in one launch -- k_axpy_alpha twice
__global__ void k_axpy_xr(cplx* __restrict__ x, const cplx* __restrict__ p, int64_t lenx, cplx* __restrict__ r,
                          const cplx* __restrict__ q, int64_t lenr, int B, const CgState* st) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  cplx* v;
  const cplx* w;
  int64_t len;
  double sign;
  if (i < lenx * B) {
    v = x; w = p; len = lenx; sign = 1.0;
  } else {
    i -= lenx * B;
    if (i >= lenr * B) return;
    v = r; w = q; len = lenr; sign = -1.0;
  }
  const CgState& s = st[i / len];
  if (!s.active) return;
  const double a = sign * s.alpha;
  cplx a0 = v[i], b0 = w[i];
  v[i] = mk(fma(a, b0.x, a0.x), fma(a, b0.y, a0.y));
}

// v += alpha w   (x += alpha p,  solver.cpp:75)  -- only while the problem is active
// and its alpha was set this iteration (flag snapshot taken before k_cg_alpha)
__global__ void k_axpy_alpha(cplx* __restrict__ v, const cplx* __restrict__ w, int64_t len, int B, const CgState* st,
                             double sign) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len * B) return;
  const CgState& s = st[i / len];
  if (!s.active) return;
  const double a = sign * s.alpha;
  cplx a0 = v[i], b0 = w[i];
  v[i] = mk(fma(a, b0.x, a0.x), fma(a, b0.y, a0.y));
}

// p = s + beta p  (solver.cpp:87)
__global__ void k_pupdate(cplx* __restrict__ p, const cplx* __restrict__ s, int64_t len, int B, const CgState* st) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len * B) return;
  const CgState& c = st[i / len];
  if (!c.active) return;
  cplx pv = p[i], sv = s[i];
  p[i] = mk(fma(c.beta, pv.x, sv.x), fma(c.beta, pv.y, sv.y));
}

// any problem still active?  (host polls this every chunk of iterations)
__global__ void k_any_active(const CgState* st, int B, int* flag) {
  int a = 0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) a |= st[b].active;
  a = __syncthreads_or(a);
  if (threadIdx.x == 0) *flag = a;
}

// zero the solution of zero-data problems (ref == 0): x = 0 (solver.cpp:43-47)
__global__ void k_zero_if_ref0(cplx* __restrict__ x, int64_t len, int B, const CgState* st) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len * B) return;
  if (st[i / len].ref == 0.0) x[i] = mk(0, 0);
}

// ---------------------------------------------------------------------------
// One-CTA-per-problem forms of the scalar / vector phases (fused CGLS paths)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double norm2_local(const cplx* __restrict__ v, int len) {
  double acc = 0.0;  // same per-entry fma order as k_norm2
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const cplx a = v[i];
    acc = fma(a.x, a.x, fma(a.y, a.y, acc));
  }
  return acc;
}

// qq = ||q||^2; alpha or stop; x += alpha p; r -= alpha q   (k_cg_alpha +
// k_axpy_alpha x2).  One CTA owns the problem; returns false when it stopped.
__device__ __forceinline__ bool cg_qstep_dev(CgState& cs, CgState* stp, const cplx* __restrict__ qp,
                                             cplx* __restrict__ rp, cplx* __restrict__ xp,
                                             const cplx* __restrict__ pp, int M, int n, double* red) {
  const double qq = block_sum(norm2_local(qp, M), red);
  cs.qq = qq;
  if (qq == 0.0) {  // search direction in the numerical null space
    cs.active = 0;
    cs.alpha = 0.0;
    if (threadIdx.x == 0) *stp = cs;
    return false;
  }
  const double alpha = cs.gamma / qq;
  cs.alpha = alpha;
  for (int l = threadIdx.x; l < n; l += blockDim.x) {
    const cplx a0 = xp[l], b0 = pp[l];
    xp[l] = mk(fma(alpha, b0.x, a0.x), fma(alpha, b0.y, a0.y));
  }
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const cplx a0 = rp[m], b0 = qp[m];
    rp[m] = mk(fma(-alpha, b0.x, a0.x), fma(-alpha, b0.y, a0.y));
  }
  return true;
}

// gamma' = ||s||^2; history; tolerance; beta; p = s + beta p   (k_cg_beta +
// k_pupdate).  s must be complete block-wide (barrier before the call).
__device__ __forceinline__ void cg_sstep_dev(CgState& cs, CgState* stp, const cplx* __restrict__ sp,
                                             cplx* __restrict__ pp, int n, double tol, double* hist,
                                             int hist_stride, double* red) {
  const double gn = block_sum(norm2_local(sp, n), red);
  const int it = cs.iterations + 1;
  const double h = sqrt(gn) / cs.ref;
  cs.iterations = it;
  cs.hist_len = (it < hist_stride ? it : hist_stride - 1) + 1;
  const bool stop = h <= tol;
  if (stop) {
    cs.converged = 1;
    cs.active = 0;
    cs.beta = 0.0;
  } else {
    cs.beta = gn / cs.gamma;
    cs.gamma = gn;
  }
  if (threadIdx.x == 0) {
    if (hist) hist[it < hist_stride ? it : hist_stride - 1] = h;
    *stp = cs;
  }
  if (stop) return;
  const double beta = cs.beta;
  for (int l = threadIdx.x; l < n; l += blockDim.x) {
    const cplx pv = pp[l], sv = sp[l];
    pp[l] = mk(fma(beta, pv.x, sv.x), fma(beta, pv.y, sv.y));
  }
}

constexpr int CG_STEP_THREADS = 1024;

// the two scalar/vector phases of the generic iteration for problems whose
// vectors one CTA reduces (Session chunks == 1): 2 launches instead of 7
__global__ void __launch_bounds__(CG_STEP_THREADS)
k_cg_qstep(CgState* st, const cplx* __restrict__ q, cplx* __restrict__ r, cplx* __restrict__ x,
           const cplx* __restrict__ p, int64_t M, int64_t n) {
  __shared__ double red[32];
  const int prob = blockIdx.x;
  CgState cs = st[prob];
  if (!cs.active) return;
  cg_qstep_dev(cs, st + prob, q + prob * M, r + prob * M, x + prob * n, p + prob * n, (int)M, (int)n, red);
  if (threadIdx.x == 0 && cs.active) st[prob] = cs;  // alpha, qq
}

__global__ void __launch_bounds__(CG_STEP_THREADS)
k_cg_sstep(CgState* st, const cplx* __restrict__ s, cplx* __restrict__ p, int64_t n, double tol, double* hist,
           int hist_stride) {
  __shared__ double red[32];
  const int prob = blockIdx.x;
  CgState cs = st[prob];
  if (!cs.active) return;
  cg_sstep_dev(cs, st + prob, s + prob * n, p + prob * n, (int)n, tol, hist ? hist + (int64_t)prob * hist_stride : nullptr,
               hist_stride, red);
}

