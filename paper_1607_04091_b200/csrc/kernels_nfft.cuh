// kernels_nfft.cuh -- Kaiser-Bessel gridding routes (K-N1 / K-N2 / K-F / K-DC /
// K-D / K-S of SURVEY 2.3), restating NfftPlan::forward / ::adjoint
// (nufft.cpp:244-365) fused with the 1D and 9-block 2D operator algebra of
// apply_forward / apply_adjoint (freq2wave.cpp:215-387).
//
// Sample-space data (base cell, 13 window weights, D/L/R record) is held in
// bin-sorted order ("s" index); perm[s] maps back to the caller's order.
// Spreading (the adjoint) is output-owned, never a global atomic:
//   1D  -- 16 lanes per oversampled cell (one per tap) gather from the
//          sorted bins and fold by shuffles;
//   2D  -- per-chunk partial regions (generic k2_spread here, the DMMA
//          kernels in kernels_nfft2d_fast.cuh), folded per tile from a
//          source list (k2_fold_src) so every grid cell is written once.
#pragma once
#include "gs_common.cuh"
#include "kernels_vec.cuh"

struct NfP {
  int n;        // modes per axis (2^J)
  int n_ov;     // oversampled length per axis (power of two)
  int log_nov;
  int p, edges; // family, edges = p >= 2
  int S;        // 2w+1 taps
  int64_t M;    // samples per problem
  // 2D tiling
  int T, R, nt; // tile edge, region edge = T + S - 1, tiles per axis
  int CW;       // columns per CTA in the column-FFT kernels
  int RW;       // rows per CTA in the row-FFT kernels (n_ov * RW / 8 = one 8-point group per thread)
};

// ============================================================== 1D route
// deconvolve + embed + FFT_{-}  (nufft.cpp:247-269), edge slots zeroed (freq2wave.cpp:224-230)
__global__ void k_n1_embed_fft(NfP P, const cplx* __restrict__ x, const double* __restrict__ deconv,
                               cplx* __restrict__ G, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  const int prob = blockIdx.x;
  x += (int64_t)prob * P.n;
  G += (int64_t)prob * P.n_ov;
  cplx* tws = sm + fpad_len(P.n_ov);  // twiddles staged in shared memory (dynamic smem: + n_ov / 2)
  for (int i = threadIdx.x; i < fpad_len(P.n_ov); i += blockDim.x) sm[i] = mk(0, 0);
  stage_twiddles(tws, tw, P.log_nov, logLmax);
  __syncthreads();
  for (int idx = threadIdx.x; idx < P.n; idx += blockDim.x) {
    int k = idx - P.n / 2;
    cplx v = x[idx];
    if (P.edges && (idx < P.p || idx >= P.n - P.p)) v = mk(0, 0);
    int pos = (k + P.n_ov) & (P.n_ov - 1);
    sm[fpad(bitrev(pos, P.log_nov))] = cscale(v, deconv[idx]);
  }
  __syncthreads();
  block_fft_padded<true>(sm, P.log_nov, 1, 0, tws, P.log_nov, -1);
  for (int i = threadIdx.x; i < P.n_ov; i += blockDim.x) G[i] = sm[fpad(i)];
}

// CGLS q-step split over the two 1D gridding kernels (k_cg_qstep's work, no
// launch of its own).  k_n1_spread: qq from the interpolation's per-CTA
// partials (the same fixed-order fold in every CTA), alpha, the adjoint's input
// r - alpha q formed as the samples are read, x <- x + alpha p grid-strided;
// CTA 0 stores the state with pend_alpha = alpha.  r itself is updated one
// kernel later, by the next iteration's k_n1_interp: the thread of sample s
// applies r[s] -= pend_alpha q[s] before it overwrites q[s] (13 spreading CTAs
// read each r[s], so the spreading cannot store it).
struct N1QStep {
  double* qpart;
  int nqpart;
  const cplx* q;
  cplx* r;
  CgState* st;
  cplx* x;
  const cplx* p;
};

// interpolation + D + L/R  (nufft.cpp:273-284, freq2wave.cpp:232-236);
// inside CGLS (qpart != nullptr) each CTA also writes its partial ||q||^2
// (qpart[prob][blockIdx.x]) for the q-step fused into k_n1_spread
__global__ void k_n1_interp(NfP P, const int* __restrict__ base, const double* __restrict__ wts,
                            const cplx* __restrict__ rec, const cplx* __restrict__ G, const cplx* __restrict__ x,
                            const int* __restrict__ out_perm, cplx* __restrict__ y, N1QStep qs) {
  const int prob = blockIdx.y;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double nq = 0.0;
  const double pend = qs.st ? qs.st[prob].pend_alpha : 0.0;
  if (s < P.M) {
    if (pend != 0.0) {  // previous iteration's r -= alpha q (sorted order: y[s] is q[s])
      const int64_t gi = prob * P.M + s;
      const cplx qv = y[gi], rv = qs.r[gi];
      qs.r[gi] = mk(fma(-pend, qv.x, rv.x), fma(-pend, qv.y, rv.y));
    }
    const int64_t gs = prob * P.M + s;
    const int Rr = 1 + (P.edges ? 2 * P.p : 0);
    const cplx* g = G + (int64_t)prob * P.n_ov;
    const int b = base[gs];
    const double* w = wts + gs * P.S;
    cplx acc = mk(0, 0);
    for (int t = 0; t < P.S; ++t) acc = caxpy(acc, w[t], ldg2(g + ((b + t) & (P.n_ov - 1))));
    const cplx* r = rec + gs * Rr;
    cplx ym = cmul(r[0], acc);
    if (P.edges) {
      const cplx* xp = x + (int64_t)prob * P.n;
      cplx a = mk(0, 0), c2 = mk(0, 0);
      for (int c = 0; c < P.p; ++c) a = cadd(a, cmul(r[1 + c], ldg2(xp + c)));
      for (int c = 0; c < P.p; ++c) c2 = cadd(c2, cmul(r[1 + P.p + c], ldg2(xp + P.n - P.p + c)));
      ym = cadd(ym, cadd(a, c2));
    }
    const int64_t o = out_perm ? (int64_t)out_perm[gs] : s;
    y[prob * P.M + o] = ym;
    nq = fma(ym.x, ym.x, ym.y * ym.y);
  }
  if (qs.st) {
    __shared__ double red[32];
    const double v = block_sum(nq, red);
    if (threadIdx.x == 0) qs.qpart[(int64_t)prob * gridDim.x + blockIdx.x] = v;
  }
}


// spreading, owner-computes: cell j sums w_s[t] conj(D_s) y_s over the points
// whose window base is (j - t) mod n_ov  (transpose of nufft.cpp:313-322).
// 16 lanes per cell, lane t < S takes tap t (S <= 15), so a thread walks the
// ~M/n_ov samples of one cell instead of S cells; the lanes' sums are folded
// by shuffles in a fixed order.  Lane 0 (tap 0) visits every sample of its
// own cell, i.e. every sample exactly once over the grid: it also
// accumulates the edge sums L^H y, R^H y (freq2wave.cpp:323-324), reduced per
// CTA into edge_part[prob][blockIdx.x][2p] (summed by k_n1_ifft_crop).
constexpr int N1_SPREAD_THREADS = 128;
constexpr int N1_SPREAD_CELLS = N1_SPREAD_THREADS / 16;
__global__ void __launch_bounds__(N1_SPREAD_THREADS)
k_n1_spread(NfP P, const int* __restrict__ cell_start, const double* __restrict__ wts,
            const cplx* __restrict__ rec, const cplx* __restrict__ yin, const int* __restrict__ in_perm,
            cplx* __restrict__ line, cplx* __restrict__ edge_part, N1QStep qs) {
  __shared__ cplx esm[N1_SPREAD_THREADS / 32][16];
  __shared__ double s_alpha;
  const int prob = blockIdx.y;
  double alpha = 0.0;  // nonzero only while a fused q-step updates r
  if (qs.st) {
    if (threadIdx.x < 32) {
      double a = 0.0;
      const double* qp = qs.qpart + (int64_t)prob * qs.nqpart;
      for (int k = threadIdx.x; k < qs.nqpart; k += 32) a += qp[k];
      a = warp_sum(a);
      if (threadIdx.x == 0) {
        CgState cs = qs.st[prob];
        double al = 0.0;
        if (cs.active) {
          cg_alpha_dev(cs, a);  // stops the problem when qq == 0 (no update)
          if (cs.active) al = cs.alpha;
        }
        cs.pend_alpha = al;  // r's deferred update (0: none)
        if (blockIdx.x == 0) qs.st[prob] = cs;
        s_alpha = al;
      }
    }
    __syncthreads();
    alpha = s_alpha;
    if (alpha != 0.0) {
      cplx* xp = qs.x + (int64_t)prob * P.n;
      const cplx* pp = qs.p + (int64_t)prob * P.n;
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        const cplx a0 = xp[i], b0 = pp[i];
        xp[i] = mk(fma(alpha, b0.x, a0.x), fma(alpha, b0.y, a0.y));
      }
    }
  }
  const int lane16 = threadIdx.x & 15;
  const int j = blockIdx.x * N1_SPREAD_CELLS + (threadIdx.x >> 4);  // n_ov is a multiple of the cells per CTA
  const int Rr = 1 + (P.edges ? 2 * P.p : 0);
  const int* cs = cell_start + (int64_t)prob * (P.n_ov + 1);
  const cplx* yp = yin + (int64_t)prob * P.M;
  cplx acc = mk(0, 0);
  cplx e[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) e[c] = mk(0, 0);
  if (lane16 < P.S) {
    const int t = lane16;
    const int cell = (j - t + P.n_ov) & (P.n_ov - 1);
    const int s1 = cs[cell + 1];
    for (int s = cs[cell]; s < s1; ++s) {
      const int64_t gs = prob * P.M + s;
      cplx yv = ldg2(yp + (in_perm ? (int64_t)in_perm[gs] : s));
      if (alpha != 0.0) {  // r - alpha q (k_axpy_alpha's arithmetic); in CGLS the order is internal
        const cplx qv = ldg2(qs.q + gs);
        yv = mk(fma(-alpha, qv.x, yv.x), fma(-alpha, qv.y, yv.y));
      }
      const cplx* r = rec + gs * Rr;
      const cplx v = cmul(conj_(ldg2(r)), yv);
      acc = caxpy(acc, __ldg(wts + gs * P.S + t), v);
      if (P.edges && t == 0) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c < 2 * P.p) e[c] = cadd(e[c], cmul(conj_(ldg2(r + 1 + c)), yv));
      }
    }
  }
  // fold the 16 taps of the cell: lane t += lane t + 8, + 4, + 2, + 1
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    acc.x += __shfl_down_sync(0xffffffffu, acc.x, o, 16);
    acc.y += __shfl_down_sync(0xffffffffu, acc.y, o, 16);
  }
  if (lane16 == 0) line[(int64_t)prob * P.n_ov + j] = acc;
  if (!P.edges) return;
  // edge sums: lanes 0 and 16 of each warp hold them; fold the pair, then the warps
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (c >= 2 * P.p) break;
    e[c].x += __shfl_down_sync(0xffffffffu, e[c].x, 16);
    e[c].y += __shfl_down_sync(0xffffffffu, e[c].y, 16);
    if (lane == 0) esm[warp][c] = e[c];
  }
  __syncthreads();
  if (threadIdx.x < 2 * P.p) {
    cplx sum = esm[0][threadIdx.x];
    for (int w = 1; w < N1_SPREAD_THREADS / 32; ++w) sum = cadd(sum, esm[w][threadIdx.x]);
    edge_part[((int64_t)prob * gridDim.x + blockIdx.x) * (2 * P.p) + threadIdx.x] = sum;
  }
}

// FFT_{+}, crop, deconvolve (nufft.cpp:340-350); edge slots <- L^H y, R^H y
// (freq2wave.cpp:317-325) from the nparts per-CTA partials of k_n1_spread,
// one warp per edge column summing them in a fixed order.  Inside CGLS
// (cst != nullptr) the CTA that owns the problem's s also runs the s-step
// (gamma', history, beta, p = s + beta p: k_cg_beta + k_pupdate).
__global__ void k_n1_ifft_crop(NfP P, const cplx* __restrict__ line, const double* __restrict__ deconv,
                               const cplx* __restrict__ edge_part, int nparts, cplx* __restrict__ z,
                               const cplx* __restrict__ tw, int logLmax, CgState* cst, cplx* __restrict__ pvec,
                               double tol, double* hist, int hist_stride) {
  extern __shared__ cplx sm[];
  __shared__ double red[32];
  const int prob = blockIdx.x;
  line += (int64_t)prob * P.n_ov;
  z += (int64_t)prob * P.n;
  cplx* tws = sm + fpad_len(P.n_ov);  // dynamic smem: + n_ov / 2 twiddles
  for (int i = threadIdx.x; i < P.n_ov; i += blockDim.x) sm[fpad(bitrev(i, P.log_nov))] = line[i];
  stage_twiddles(tws, tw, P.log_nov, logLmax);
  __syncthreads();
  block_fft_padded<true>(sm, P.log_nov, 1, 0, tws, P.log_nov, +1);
  for (int idx = threadIdx.x; idx < P.n; idx += blockDim.x) {
    int k = idx - P.n / 2;
    if (P.edges && (idx < P.p || idx >= P.n - P.p)) continue;  // edge slots: written below
    z[idx] = cscale(sm[fpad((k + P.n_ov) & (P.n_ov - 1))], deconv[idx]);
  }
  if (P.edges) {
    const int lane = threadIdx.x & 31, E = 2 * P.p;
    const cplx* ep = edge_part + (int64_t)prob * nparts * E;
    for (int c = threadIdx.x >> 5; c < E; c += blockDim.x >> 5) {
      cplx a = mk(0, 0);
      for (int k = lane; k < nparts; k += 32) a = cadd(a, ep[(int64_t)k * E + c]);
      const double re = warp_sum(a.x), im = warp_sum(a.y);
      if (lane == 0) z[c < P.p ? c : P.n - 2 * P.p + c] = mk(re, im);
    }
  }
  if (!cst) return;
  CgState cs = cst[prob];
  if (!cs.active) return;
  __syncthreads();  // s complete block-wide
  cg_sstep_dev(cs, cst + prob, z, pvec + (int64_t)prob * P.n, P.n, tol,
               hist ? hist + (int64_t)prob * hist_stride : nullptr, hist_stride, red);
}

// ============================================================== 2D route
// Grid layout: G[prob][r][c], axis0 (rows) = y, axis1 (cols) = x, last axis
// fastest (freq2wave.cpp:183-190).  Coefficients X(i, j) = x[j*n + i], i = x.

// rows of the embedded interior block, deconvolved, FFT_{-} along x
// (nufft.cpp:253-266 row part + freq2wave.cpp:246-254); RW rows per CTA
__global__ void k2_rows_embed_fft(NfP P, const cplx* __restrict__ x, const double* __restrict__ deconv,
                                  cplx* __restrict__ G, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  const int j0 = blockIdx.x * P.RW, prob = blockIdx.y;
  const int ls = fpad_len(P.n_ov) + 1, nr = min(P.RW, P.n - j0);
  for (int i = threadIdx.x; i < P.RW * ls; i += blockDim.x) sm[i] = mk(0, 0);
  __syncthreads();
  for (int t = threadIdx.x; t < nr * P.n; t += blockDim.x) {
    const int rr = t / P.n, i = t - rr * P.n, j = j0 + rr;
    if (P.edges && (j < P.p || j >= P.n - P.p || i < P.p || i >= P.n - P.p)) continue;  // edge rows / slots stay 0
    const cplx v = x[(int64_t)prob * P.n * P.n + (int64_t)j * P.n + i];
    const int pos = (i - P.n / 2 + P.n_ov) & (P.n_ov - 1);
    sm[rr * ls + fpad(bitrev(pos, P.log_nov))] = cscale(v, deconv[j] * deconv[i]);
  }
  __syncthreads();
  block_fft_padded(sm, P.log_nov, P.RW, ls, tw, logLmax, -1);
  for (int t = threadIdx.x; t < nr * P.n_ov; t += blockDim.x) {
    const int rr = t / P.n_ov, i = t - rr * P.n_ov;
    const int r = (j0 + rr - P.n / 2 + P.n_ov) & (P.n_ov - 1);
    G[((int64_t)prob * P.n_ov + r) * P.n_ov + i] = sm[rr * ls + fpad(i)];
  }
}

// FFT_{-} along y of CW columns; only the n rows carrying data are loaded
__global__ void k2_cols_fft(NfP P, cplx* __restrict__ G, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  const int c0 = blockIdx.x * P.CW, prob = blockIdx.y;
  const int ls = fpad_len(P.n_ov) + 1;
  cplx* g = G + (int64_t)prob * P.n_ov * P.n_ov;
  for (int i = threadIdx.x; i < P.CW * ls; i += blockDim.x) sm[i] = mk(0, 0);
  __syncthreads();
  for (int t = threadIdx.x; t < P.n * P.CW; t += blockDim.x) {
    const int jj = t / P.CW, cc = t - jj * P.CW;
    const int r = (jj - P.n / 2 + P.n_ov) & (P.n_ov - 1);
    sm[cc * ls + fpad(bitrev(r, P.log_nov))] = g[(int64_t)r * P.n_ov + c0 + cc];
  }
  __syncthreads();
  block_fft_padded(sm, P.log_nov, P.CW, ls, tw, logLmax, -1);
  for (int t = threadIdx.x; t < P.n_ov * P.CW; t += blockDim.x) {
    const int r = t / P.CW, cc = t - r * P.CW;
    g[(int64_t)r * P.n_ov + c0 + cc] = sm[cc * ls + fpad(r)];
  }
}

// The 4p side lines (freq2wave.cpp:272-301): line e < 2p runs along y at the
// x-edge index i_e (rows 0..p-1, n-p..n-1 of X), e >= 2p along x at the
// y-edge index j_e.  Interior entries only, deconvolved, FFT_{-}.
__device__ __forceinline__ int edge_index(int e, int n, int p) { return e < p ? e : n - 2 * p + e; }

__global__ void k2_lines_fft(NfP P, const cplx* __restrict__ x, const double* __restrict__ deconv,
                             cplx* __restrict__ lines, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  const int L = blockIdx.x, prob = blockIdx.y;
  const int twop = 2 * P.p;
  const bool yline = L < twop;
  const int e = yline ? L : L - twop;
  const int fixed = edge_index(e, P.n, P.p);
  const cplx* X = x + (int64_t)prob * P.n * P.n;
  cplx* tws = sm + fpad_len(P.n_ov);  // dynamic smem: + n_ov / 2 staged twiddles
  for (int i = threadIdx.x; i < fpad_len(P.n_ov); i += blockDim.x) sm[i] = mk(0, 0);
  stage_twiddles(tws, tw, P.log_nov, logLmax);
  __syncthreads();
  for (int v = P.p + threadIdx.x; v < P.n - P.p; v += blockDim.x) {
    cplx val = yline ? X[(int64_t)v * P.n + fixed] : X[(int64_t)fixed * P.n + v];
    int pos = (v - P.n / 2 + P.n_ov) & (P.n_ov - 1);
    sm[fpad(bitrev(pos, P.log_nov))] = cscale(val, deconv[v]);
  }
  __syncthreads();
  block_fft_padded<true>(sm, P.log_nov, 1, 0, tws, P.log_nov, -1);
  cplx* out = lines + ((int64_t)prob * 2 * twop + L) * P.n_ov;
  for (int i = threadIdx.x; i < P.n_ov; i += blockDim.x) out[i] = sm[fpad(i)];
}

// Per-point forward: 2D interpolation (nufft.cpp:287-303) scaled by Dx Dy,
// 4 corner blocks (freq2wave.cpp:260-270), 4p side interpolations
// (freq2wave.cpp:272-301).  axis 0 = x, 1 = y in the sorted arrays.
__global__ void k2_interp(NfP P, const int* __restrict__ base_x, const int* __restrict__ base_y,
                          const double* __restrict__ wx_all, const double* __restrict__ wy_all,
                          const cplx* __restrict__ recx_all, const cplx* __restrict__ recy_all,
                          const cplx* __restrict__ G, const cplx* __restrict__ lines, const cplx* __restrict__ x,
                          const int* __restrict__ out_perm, cplx* __restrict__ y) {
  const int prob = blockIdx.y;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= P.M) return;
  const int64_t gs = prob * P.M + s;
  const int S = P.S, mask = P.n_ov - 1, p = P.p;
  const int Rr = 1 + (P.edges ? 2 * p : 0);
  const int by = base_y[gs], bx = base_x[gs];
  const double* wy = wy_all + gs * S;
  const double* wx = wx_all + gs * S;
  double wyr[16], wxr[16];
  for (int t = 0; t < S; ++t) {
    wyr[t] = wy[t];
    wxr[t] = wx[t];
  }
  const cplx* g = G + (int64_t)prob * P.n_ov * P.n_ov;
  cplx acc = mk(0, 0);
  for (int t0 = 0; t0 < S; ++t0) {
    const cplx* row = g + (int64_t)((by + t0) & mask) * P.n_ov;
    cplx ra = mk(0, 0);
    for (int t1 = 0; t1 < S; ++t1) ra = caxpy(ra, wxr[t1], ldg2(row + ((bx + t1) & mask)));
    acc = caxpy(acc, wyr[t0], ra);
  }
  const cplx* rx = recx_all + gs * Rr;
  const cplx* ry = recy_all + gs * Rr;
  const cplx Dx = rx[0], Dy = ry[0];
  cplx out = cmul(cmul(Dx, Dy), acc);
  if (P.edges) {
    const cplx* X = x + (int64_t)prob * P.n * P.n;
    const int n = P.n, np = n - p;
    // corners: (Lx,Ly) (Lx,Ry) (Rx,Ly) (Rx,Ry)
    for (int k = 0; k < 4; ++k) {
      const int ax = (k < 2) ? 1 : 1 + p;        // record offset of Ax columns
      const int by_ = (k % 2 == 0) ? 1 : 1 + p;  // record offset of By columns
      const int row0 = (k < 2) ? 0 : np, col0 = (k % 2 == 0) ? 0 : np;
      cplx sum = mk(0, 0);
      for (int j = 0; j < p; ++j) {
        cplx t = mk(0, 0);
        for (int i = 0; i < p; ++i) t = cadd(t, cmul(rx[ax + i], ldg2(X + (int64_t)(col0 + j) * n + row0 + i)));
        sum = cadd(sum, cmul(t, ry[by_ + j]));
      }
      out = cadd(out, sum);
    }
    const cplx* LY = lines + (int64_t)prob * 4 * p * P.n_ov;
    const cplx* LX = LY + (int64_t)2 * p * P.n_ov;
    // side_x_edge (Lx then Rx): y-lines, weights along y
    for (int e = 0; e < 2 * p; ++e) {
      const cplx* ln = LY + (int64_t)e * P.n_ov;
      cplx u = mk(0, 0);
      for (int t = 0; t < S; ++t) u = caxpy(u, wyr[t], ldg2(ln + ((by + t) & mask)));
      out = cadd(out, cmul(cmul(rx[1 + e], Dy), u));
    }
    // side_y_edge (Ly then Ry): x-lines, weights along x
    for (int e = 0; e < 2 * p; ++e) {
      const cplx* ln = LX + (int64_t)e * P.n_ov;
      cplx u = mk(0, 0);
      for (int t = 0; t < S; ++t) u = caxpy(u, wxr[t], ldg2(ln + ((bx + t) & mask)));
      out = cadd(out, cmul(cmul(ry[1 + e], Dx), u));
    }
  }
  const int64_t o = out_perm ? (int64_t)out_perm[gs] : s;
  y[prob * P.M + o] = out;
}

// Adjoint spreading of one tile: 4 warps, each with a private shared-memory
// copy of the (T+S-1)^2 region and of the 2 x 2p line segments; one point per
// warp at a time, lanes over the window cells (no two lanes share a cell).
// Output: the region (TB), the line segments (TL) and the corner partial sums
// (TC) of this tile -- each written exactly once.
#define K2_WARPS 4
__global__ void __launch_bounds__(32 * K2_WARPS)
k2_spread(NfP P, const int* __restrict__ tile_start, const int* __restrict__ base_x, const int* __restrict__ base_y,
          const double* __restrict__ wx_all, const double* __restrict__ wy_all, const cplx* __restrict__ recx_all,
          const cplx* __restrict__ recy_all, const cplx* __restrict__ yin, const int* __restrict__ in_perm,
          cplx* __restrict__ TB, cplx* __restrict__ TL, cplx* __restrict__ TC) {
  extern __shared__ cplx sm[];
  const int tile = blockIdx.x, prob = blockIdx.y;
  const int ntiles = P.nt * P.nt;
  const int ty = tile / P.nt, tx = tile - ty * P.nt;
  const int R = P.R, S = P.S, p = P.p, twop = 2 * p;
  const int nreg = R * R;
  const int nlin = P.edges ? 2 * twop * R : 0;
  const int per_warp = nreg + nlin;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < per_warp * K2_WARPS; i += blockDim.x) sm[i] = mk(0, 0);
  __syncthreads();
  cplx* reg = sm + warp * per_warp;
  cplx* lin = reg + nreg;  // [2][2p][R]: y-lines then x-lines
  const int Rr = 1 + (P.edges ? twop : 0);
  const int ncorner = P.edges ? 4 * p * p : 0;
  cplx cacc[8];
  for (int u = 0; u < 8; ++u) cacc[u] = mk(0, 0);
  const int* ts = tile_start + (int64_t)prob * (ntiles + 1);
  const int s0 = ts[tile], s1 = ts[tile + 1];
  const cplx* yp = yin + (int64_t)prob * P.M;
  for (int s = s0 + warp; s < s1; s += K2_WARPS) {
    const int64_t gs = prob * P.M + s;
    const int oy = base_y[gs] - ty * P.T, ox = base_x[gs] - tx * P.T;
    const double wyl = lane < S ? wy_all[gs * S + lane] : 0.0;
    const double wxl = lane < S ? wx_all[gs * S + lane] : 0.0;
    const cplx ys = ldg2(yp + (in_perm ? (int64_t)in_perm[gs] : s));
    const cplx* rx = recx_all + gs * Rr;
    const cplx* ry = recy_all + gs * Rr;
    const cplx Dx = ldg2(rx), Dy = ldg2(ry);
    const cplx v2 = cmul(conj_(cmul(Dx, Dy)), ys);  // freq2wave.cpp:335
    for (int base = 0; base < S * S; base += 32) {
      const int idx = base + lane;
      const int t0 = idx / S, t1 = idx - t0 * S;
      const double w0 = __shfl_sync(0xffffffffu, wyl, t0 < S ? t0 : 0);
      const double w1 = __shfl_sync(0xffffffffu, wxl, t1);
      if (idx < S * S) {
        cplx* cell = reg + (oy + t0) * R + (ox + t1);
        const cplx v0 = cscale(v2, w0);  // v0 = w0[t0] * y (nufft.cpp:328)
        *cell = caxpy(*cell, w1, v0);
      }
    }
    if (P.edges) {
      for (int base = 0; base < twop * S; base += 32) {
        const int idx = base + lane;
        const int e = idx / S, t = idx - e * S;
        const double wyt = __shfl_sync(0xffffffffu, wyl, t);
        const double wxt = __shfl_sync(0xffffffffu, wxl, t);
        if (idx < twop * S) {
          // side_x_edge: v = conj(Ax(m,e) Dy) y along y; side_y_edge: conj(By(m,e) Dx) y along x
          const cplx vy = cmul(conj_(cmul(ldg2(rx + 1 + e), Dy)), ys);
          const cplx vx = cmul(conj_(cmul(ldg2(ry + 1 + e), Dx)), ys);
          cplx* ly = lin + e * R + oy + t;
          cplx* lx = lin + (twop + e) * R + ox + t;
          *ly = caxpy(*ly, wyt, vy);
          *lx = caxpy(*lx, wxt, vx);
        }
      }
      // corners: Z(row0+i, col0+j) += conj(Ax(m,i)) (y conj(By(m,j)))  (freq2wave.cpp:349-353)
      for (int u = 0; u < 8; ++u) {
        const int q = lane + 32 * u;
        if (q < ncorner) {
          const int k = q / (p * p), rem = q - k * p * p, i = rem / p, j = rem - i * p;
          const int ax = (k < 2) ? 1 : 1 + p, byo = (k % 2 == 0) ? 1 : 1 + p;
          cacc[u] = cadd(cacc[u], cmul(conj_(ldg2(rx + ax + i)), cmul(ys, conj_(ldg2(ry + byo + j)))));
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
  // fold the warp copies and write the tile's region / lines once
  cplx* tb = TB + ((int64_t)prob * ntiles + tile) * nreg;
  for (int i = threadIdx.x; i < nreg; i += blockDim.x) {
    cplx a = sm[i];
    for (int w = 1; w < K2_WARPS; ++w) a = cadd(a, sm[w * per_warp + i]);
    tb[i] = a;
  }
  if (P.edges) {
    cplx* tl = TL + ((int64_t)prob * ntiles + tile) * nlin;
    for (int i = threadIdx.x; i < nlin; i += blockDim.x) {
      cplx a = sm[nreg + i];
      for (int w = 1; w < K2_WARPS; ++w) a = cadd(a, sm[w * per_warp + nreg + i]);
      tl[i] = a;
    }
    __syncthreads();
    // corner partials: reuse the region smem of warp 0 as [K2_WARPS][ncorner]
    for (int u = 0; u < 8; ++u) {
      const int q = lane + 32 * u;
      if (q < ncorner) sm[warp * ncorner + q] = cacc[u];
    }
    __syncthreads();
    cplx* tc = TC + ((int64_t)prob * ntiles + tile) * ncorner;
    for (int q = threadIdx.x; q < ncorner; q += blockDim.x) {
      cplx a = sm[q];
      for (int w = 1; w < K2_WARPS; ++w) a = cadd(a, sm[w * ncorner + q]);
      tc[q] = a;
    }
  }
}

// Tiles whose (T+S-1)-wide region covers global index r along one axis, as
// (tile, local offset) pairs: region of tile t spans [t*T, t*T + R) mod n_ov;
// the last tile may be partial (n_ov need not be a multiple of T).
#define MAX_COVER 8
__host__ __device__ __forceinline__ int cover(int r, int T, int R, int nt, int n_ov, int* tl, int* ll) {
  int k = 0;
  const int dmax = (R + T - 1) / T;
  for (int d = 0; d <= dmax && d < nt; ++d) {
    const int t = ((r / T - d) % nt + nt) % nt;
    for (int l = ((r - t * T) % n_ov + n_ov) % n_ov; l < R && k < MAX_COVER; l += n_ov) {
      tl[k] = t;
      ll[k] = l;
      ++k;
    }
  }
  return k;
}

// Fold the per-chunk adjoint partials into the oversampled grid: one CTA per
// (tile, problem) writes the tile's T x T core cells of G, each the sum over
// every chunk of every tile whose (T+S-1)^2 region covers the cell (coverage
// per coordinate precomputed in cov / covn, same order as cover()).  Reads of
// the partial rows are contiguous along x; every G cell is written once.
__global__ void k2_fold_tiles(NfP P, const cplx* __restrict__ TB, const int* __restrict__ tcs_all, int cap,
                              const int2* __restrict__ cov, const int* __restrict__ covn, cplx* __restrict__ G) {
  const int tile = blockIdx.x, prob = blockIdx.y;
  const int ty = tile / P.nt, tx = tile - ty * P.nt;
  const cplx* TBp = TB + (int64_t)prob * cap * P.R * P.R;
  const int* tcs = tcs_all + (int64_t)prob * (P.nt * P.nt + 1);
  cplx* g = G + (int64_t)prob * P.n_ov * P.n_ov;
  for (int q = threadIdx.x; q < P.T * P.T; q += blockDim.x) {
    const int r = ty * P.T + q / P.T, c = tx * P.T + q % P.T;
    if (r >= P.n_ov || c >= P.n_ov) continue;
    cplx a = mk(0, 0);
    const int ny = covn[r], nx = covn[c];
    for (int i = 0; i < ny; ++i) {
      const int2 yv = cov[r * MAX_COVER + i];
      for (int j = 0; j < nx; ++j) {
        const int2 xv = cov[c * MAX_COVER + j];
        const int tl = yv.x * P.nt + xv.x;
        for (int ch = tcs[tl]; ch < tcs[tl + 1]; ++ch)
          a = cadd(a, ldg2(TBp + ((int64_t)ch * P.R + yv.y) * P.R + xv.y));
      }
    }
    g[(int64_t)r * P.n_ov + c] = a;
  }
}

// FFT_{+} along y for CW columns of G; only the rows the crop keeps are written
// Same fold, driven by a per-tile source list built at construction
// (gs_capi.cu): entry (chunk, oy, ox) adds partial chunk[(oy + a) mod n_ov]
// [(ox + b) mod n_ov] to core cell (a, b) where that lies inside the chunk's
// region, in the order k2_fold_tiles sums them (row cover, column cover,
// chunk).  The list sits in shared memory, so each thread's partial loads are
// independent and issue back to back instead of behind the coverage lookups.
#define K2_FOLD_SRC 64
__global__ void k2_fold_src(NfP P, const cplx* __restrict__ TB, const int* __restrict__ fs_start,
                            const int4* __restrict__ fsrc, int cap, cplx* __restrict__ G) {
  __shared__ int4 src[K2_FOLD_SRC];
  const int tile = blockIdx.x, prob = blockIdx.y, ntl = P.nt * P.nt;
  const int ty = tile / P.nt, tx = tile - ty * P.nt;
  const cplx* TBp = TB + (int64_t)prob * cap * P.R * P.R;
  const int f0 = fs_start[(int64_t)prob * (ntl + 1) + tile], f1 = fs_start[(int64_t)prob * (ntl + 1) + tile + 1];
  const int q = threadIdx.x, a = q / P.T, b = q - (q / P.T) * P.T;
  const int r = ty * P.T + a, c = tx * P.T + b;
  const bool live = q < P.T * P.T && r < P.n_ov && c < P.n_ov;
  cplx acc = mk(0, 0);
  for (int base = f0; base < f1; base += K2_FOLD_SRC) {
    const int ns = min(K2_FOLD_SRC, f1 - base);
    __syncthreads();
    for (int i = threadIdx.x; i < ns; i += blockDim.x) src[i] = fsrc[base + i];
    __syncthreads();
    if (!live) continue;
    for (int i0 = 0; i0 < ns; i0 += 4) {
      cplx v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = mk(0, 0);
        if (i0 + k < ns) {
          const int4 e = src[i0 + k];
          int la = e.y + a, lb = e.z + b;
          if (la >= P.n_ov) la -= P.n_ov;
          if (lb >= P.n_ov) lb -= P.n_ov;
          if (la < P.R && lb < P.R) v[k] = ldg2(TBp + ((int64_t)e.x * P.R + la) * P.R + lb);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i0 + k < ns) acc = cadd(acc, v[k]);
    }
  }
  if (live) G[((int64_t)prob * P.n_ov + r) * P.n_ov + c] = acc;
}

__global__ void k2_cols_ifft(NfP P, cplx* __restrict__ G, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  const int c0 = blockIdx.x * P.CW, prob = blockIdx.y;
  const int ls = fpad_len(P.n_ov) + 1;
  cplx* g = G + (int64_t)prob * P.n_ov * P.n_ov;
  for (int t = threadIdx.x; t < P.n_ov * P.CW; t += blockDim.x) {
    const int r = t / P.CW, cc = t - r * P.CW;
    sm[cc * ls + fpad(bitrev(r, P.log_nov))] = g[(int64_t)r * P.n_ov + c0 + cc];
  }
  __syncthreads();
  block_fft_padded(sm, P.log_nov, P.CW, ls, tw, logLmax, +1);
  for (int t = threadIdx.x; t < P.n * P.CW; t += blockDim.x) {
    const int jj = t / P.CW, cc = t - jj * P.CW;
    const int r = (jj - P.n / 2 + P.n_ov) & (P.n_ov - 1);
    g[(int64_t)r * P.n_ov + c0 + cc] = sm[cc * ls + fpad(r)];
  }
}

// FFT_{+} along x of the kept rows, crop, deconvolve -> interior block of Z;
// every edge entry of Z is zeroed here (filled by k2_edges).
__global__ void k2_rows_ifft_crop(NfP P, const cplx* __restrict__ G, const double* __restrict__ deconv,
                                  cplx* __restrict__ z, const cplx* __restrict__ tw, int logLmax) {
  extern __shared__ cplx sm[];
  const int j0 = blockIdx.x * P.RW, prob = blockIdx.y;
  const int ls = fpad_len(P.n_ov) + 1, nr = min(P.RW, P.n - j0);
  for (int t = threadIdx.x; t < P.RW * P.n_ov; t += blockDim.x) {
    const int rr = t / P.n_ov, i = t - rr * P.n_ov;
    cplx v = mk(0, 0);
    if (rr < nr) {
      const int r = (j0 + rr - P.n / 2 + P.n_ov) & (P.n_ov - 1);
      v = G[((int64_t)prob * P.n_ov + r) * P.n_ov + i];
    }
    sm[rr * ls + fpad(bitrev(i, P.log_nov))] = v;
  }
  __syncthreads();
  block_fft_padded(sm, P.log_nov, P.RW, ls, tw, logLmax, +1);
  for (int t = threadIdx.x; t < nr * P.n; t += blockDim.x) {
    const int rr = t / P.n, i = t - rr * P.n, j = j0 + rr;
    cplx v = cscale(sm[rr * ls + fpad((i - P.n / 2 + P.n_ov) & (P.n_ov - 1))], deconv[j] * deconv[i]);
    if (P.edges && (j < P.p || j >= P.n - P.p || i < P.p || i >= P.n - P.p)) v = mk(0, 0);
    z[(int64_t)prob * P.n * P.n + (int64_t)j * P.n + i] = v;
  }
}

// Side lines (gather of the tile line segments, FFT_{+}, crop, deconvolve,
// add into the edge rows / columns of Z, freq2wave.cpp:359-385) and, in the
// extra block per problem, the corner sums (freq2wave.cpp:349-357).
// Fold the side-line partials of every chunk along the tile row (y-lines) or
// tile column (x-lines) they belong to: TLF[prob][axis][t][e][l], one thread
// per (t, e, l) -- a fully parallel first level of the line gather.
// per (axis, tile line t, edge column e, region offset l): the sum of the
// side-line partials of every chunk on that tile line.  A CTA takes 32
// consecutive outputs (one per lane: coalesced partial rows) and splits the
// nt tiles of the line over K2_FL_SPLIT warps, folded through shared memory
// in a fixed order -- a single problem (C4) gets nt / K2_FL_SPLIT dependent
// loads per thread instead of nt.
#define K2_FL_SPLIT 8
__global__ void __launch_bounds__(32 * K2_FL_SPLIT)
k2_fold_lines(NfP P, const cplx* __restrict__ TL, const int* __restrict__ tcs_all, int cap, cplx* __restrict__ TLF) {
  __shared__ cplx part[K2_FL_SPLIT][32];
  const int prob = blockIdx.z, axis = blockIdx.y;
  const int twop = 2 * P.p, R = P.R, nt = P.nt;
  const int per = nt * twop * R;
  const int lane = threadIdx.x & 31, sp = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  cplx a = mk(0, 0);
  if (i < per) {
    const int t = i / (twop * R), rem = i - t * twop * R;  // rem = e * R + l
    const int nlin = 2 * twop * R;
    const int* tcs = tcs_all + (int64_t)prob * (nt * nt + 1);
    const cplx* TLp = TL + (int64_t)prob * cap * nlin + (axis ? twop * R : 0) + rem;
    for (int o = sp; o < nt; o += K2_FL_SPLIT) {
      const int tile = axis == 0 ? t * nt + o : o * nt + t;
      for (int ch = tcs[tile]; ch < tcs[tile + 1]; ++ch) a = cadd(a, ldg2(TLp + (int64_t)ch * nlin));
    }
  }
  part[sp][lane] = a;
  __syncthreads();
  if (sp == 0 && i < per) {
    for (int k = 1; k < K2_FL_SPLIT; ++k) a = cadd(a, part[k][lane]);
    const int t = i / (twop * R), rem = i - t * twop * R;
    TLF[(((int64_t)prob * 2 + axis) * nt + t) * twop * R + rem] = a;
  }
}

// First level of the corner reduction: TCF[prob][g][q] = sum of the corner
// partials of chunks g*64 .. g*64+63 (fixed order).
#define K2_CGROUP 16
__global__ void k2_fold_corners(NfP P, const cplx* __restrict__ TC, const int* __restrict__ ch_count, int cap,
                                int ngroups, cplx* __restrict__ TCF) {
  const int prob = blockIdx.y;
  const int ncorner = 4 * P.p * P.p;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ngroups * ncorner) return;
  const int g = i / ncorner, q = i - g * ncorner;
  const int nch = ch_count[prob];
  const cplx* tc = TC + (int64_t)prob * cap * ncorner + q;
  cplx a = mk(0, 0);
  for (int c = g * K2_CGROUP; c < min(nch, (g + 1) * K2_CGROUP); ++c) a = cadd(a, ldg2(tc + (int64_t)c * ncorner));
  TCF[((int64_t)prob * ngroups + g) * ncorner + q] = a;
}

__global__ void k2_edges(NfP P, const cplx* __restrict__ TLF, const cplx* __restrict__ TC,
                         const int* __restrict__ tcs_all, const int* __restrict__ ch_count, int cap,
                         const double* __restrict__ deconv, cplx* __restrict__ z, const cplx* __restrict__ tw,
                         int logLmax) {
  extern __shared__ cplx sm[];
  const int L = blockIdx.x, prob = blockIdx.y;
  const int p = P.p, twop = 2 * p, n = P.n, T = P.T, R = P.R, nt = P.nt;
  const int nlin = 2 * twop * R;
  const int* tcs = tcs_all + (int64_t)prob * (nt * nt + 1);
  cplx* Z = z + (int64_t)prob * n * n;
  if (L == 2 * twop) {  // corners: fixed-order sum of the chunk-group partials (TC = TCF here),
    // the groups split over blockDim / ncorner thread slices folded in shared memory
    const int ncorner = 4 * p * p;
    const int ngroups = (cap + K2_CGROUP - 1) / K2_CGROUP;
    const cplx* tc = TC + (int64_t)prob * ngroups * ncorner;
    const int nch = (ch_count[prob] + K2_CGROUP - 1) / K2_CGROUP;
    const int nsl = max(1, (int)blockDim.x / ncorner);  // slices (ncorner <= 256 for p <= 8)
    const int q = threadIdx.x % ncorner, sl = threadIdx.x / ncorner;
    cplx a = mk(0, 0);
    if (sl < nsl)
      for (int t = sl; t < nch; t += nsl) a = cadd(a, tc[(int64_t)t * ncorner + q]);
    if (sl < nsl) sm[sl * ncorner + q] = a;
    __syncthreads();
    if (sl == 0) {
      for (int k = 1; k < nsl; ++k) a = cadd(a, sm[k * ncorner + q]);
      const int k = q / (p * p), rem = q - k * p * p, i = rem / p, j = rem - i * p;
      const int row0 = (k < 2) ? 0 : n - p, col0 = (k % 2 == 0) ? 0 : n - p;
      Z[(int64_t)(col0 + j) * n + row0 + i] = a;
    }
    return;
  }
  const bool yline = L < twop;
  const int e = yline ? L : L - twop;
  const cplx* TLFp = TLF + ((int64_t)prob * 2 + (yline ? 0 : 1)) * nt * twop * R;
  (void)nlin;
  (void)tcs;
  cplx* tws = sm + fpad_len(P.n_ov);  // dynamic smem: + n_ov / 2 staged twiddles
  stage_twiddles(tws, tw, P.log_nov, logLmax);
  for (int pos = threadIdx.x; pos < P.n_ov; pos += blockDim.x) {
    cplx a = mk(0, 0);
    int tk[MAX_COVER], lk[MAX_COVER];
    const int nc = cover(pos, T, R, nt, P.n_ov, tk, lk);
    for (int i = 0; i < nc; ++i) a = cadd(a, TLFp[((int64_t)tk[i] * twop + e) * R + lk[i]]);
    sm[fpad(bitrev(pos, P.log_nov))] = a;
  }
  __syncthreads();
  block_fft_padded<true>(sm, P.log_nov, 1, 0, tws, P.log_nov, +1);
  const int fixed = edge_index(e, n, p);
  for (int v = p + threadIdx.x; v < n - p; v += blockDim.x) {
    cplx val = cscale(sm[fpad((v - n / 2 + P.n_ov) & (P.n_ov - 1))], deconv[v]);
    if (yline) Z[(int64_t)v * n + fixed] = val;  // Z(i_e, j)
    else Z[(int64_t)fixed * n + v] = val;        // Z(i, j_e)
  }
}

// ------------------------------------------------------------------ column FFTs, radix-8 passes with global I/O
// Same transform as k2_cols_fft / k2_cols_ifft (radix-2 DIT on bit-reversed
// input, three stages fused per pass) for n_ov = 8^k: the first pass gathers
// its 8 bit-reversed rows straight from global memory into registers and the
// last pass stores its 8 rows straight back, so a 512-point column costs two
// shared-memory round trips instead of four plus the load / store copies; the
// twiddles sit in shared memory.  Thread (j, cc): column c0 + cc, lanes run
// along the CW columns so every row access is a CW x 16 B segment.
// FWD: forward (FFT_-), only the n rows carrying data are read (the zero rows
// of the embedded block are skipped); else inverse (FFT_+), only the n rows
// the crop keeps are stored.
#ifndef F_COLS_QW
#define F_COLS_QW 1  // quarter-wave twiddle table in the column FFTs: 2 KB less shared memory, 3 CTAs of 8 columns per SM
#endif
// QW: tws holds the first quarter of the table only (k < 2^L / 4);
// exp(-2 pi i (k + 2^L / 4) / 2^L) = -i exp(-2 pi i k / 2^L)
template <bool FWD, int NST, bool QW = false>
__device__ __forceinline__ void r8_pass(cplx* v, int jh, int h, const cplx* __restrict__ tws, int L, int s) {
  constexpr int GN = 1 << NST;
#pragma unroll
  for (int q = 0; q < NST; ++q) {
#pragma unroll
    for (int m = 0; m < GN; ++m) {
      if ((m >> q) & 1) continue;
      const int k = jh + (m & ((1 << q) - 1)) * h;
      const int idx = k << (L - (s + q));
      cplx w;
      if (QW) {
        const int qn = 1 << (L - 2);
        const bool hi = idx >= qn;
        const cplx t = tws[hi ? idx - qn : idx];
        w = hi ? mk(t.y, -t.x) : t;
      } else {
        w = tws[idx];
      }
      if (!FWD) w.y = -w.y;
      const cplx u = v[m], x = cmul(v[m + (1 << q)], w);
      v[m] = cadd(u, x);
      v[m + (1 << q)] = csub(u, x);
    }
  }
}

// one pass of NST fused stages starting at stage s over the CTA's CW columns
template <bool FWD, int NST>
__device__ __forceinline__ void cols_pass(const NfP& P, cplx* __restrict__ g, cplx* sm, const cplx* __restrict__ tws,
                                          int ls, int c0, int s, bool first, bool last) {
  constexpr int GN = 1 << NST;
  const int L = P.log_nov, N = P.n_ov, CW = P.CW, half = P.n / 2;
  const int h = 1 << (s - 1);
  const int nthr = (N / GN) * CW;
  for (int tix = threadIdx.x; tix < nthr; tix += blockDim.x) {
    const int cc = tix % CW, j = tix / CW;
    const int jh = j & (h - 1);
    const int i0 = (j >> (s - 1)) * (GN * h) + jh;
    cplx* base = sm + cc * ls;
    cplx v[GN];
    if (first) {
#pragma unroll
      for (int m = 0; m < GN; ++m) {
        const int r = bitrev(i0 + m, L);  // input row of bit-reversed position i0 + m
        v[m] = (!FWD || r < half || r >= N - half) ? g[(int64_t)r * N + c0 + cc] : mk(0, 0);
      }
    } else {
#pragma unroll
      for (int m = 0; m < GN; ++m) v[m] = base[fpad(i0 + m * h)];
    }
    r8_pass<FWD, NST, F_COLS_QW != 0>(v, jh, h, tws, L, s);
    if (last) {
#pragma unroll
      for (int m = 0; m < GN; ++m) {
        const int r = i0 + m * h;
        if (FWD || r < half || r >= N - half) g[(int64_t)r * N + c0 + cc] = v[m];
      }
    } else {
#pragma unroll
      for (int m = 0; m < GN; ++m) base[fpad(i0 + m * h)] = v[m];
    }
  }
}

#ifndef F_COLS_THREADS
#define F_COLS_THREADS 256  // threads of a column-FFT CTA
#endif
#ifndef F_COLS_QW
#define F_COLS_QW 1  // quarter-wave twiddle table in the column FFTs: 2 KB less shared memory, 3 CTAs of 8 columns per SM
#endif
#ifndef F_COLS_MINB
#define F_COLS_MINB (F_COLS_QW ? 3 : 2)
#endif
template <bool FWD>
__global__ void __launch_bounds__(F_COLS_THREADS, F_COLS_MINB) k2_cols_fft8(NfP P, cplx* __restrict__ G, const cplx* __restrict__ tw) {
  extern __shared__ cplx sm[];
  const int L = P.log_nov, N = P.n_ov, CW = P.CW;
  const int ls = fpad_len(N) + 1;
  cplx* tws = sm + CW * ls;  // N / 2 twiddles (N / 4 with F_COLS_QW)
  const int c0 = blockIdx.x * CW, prob = blockIdx.y;
  cplx* g = G + (int64_t)prob * N * N;
  for (int i = threadIdx.x; i < (F_COLS_QW ? N / 4 : N / 2); i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  for (int s = 1; s <= L;) {
    const int nst = L - s + 1 >= 3 ? 3 : L - s + 1;
    const bool first = s == 1, last = s + nst > L;
    if (nst == 3) cols_pass<FWD, 3>(P, g, sm, tws, ls, c0, s, first, last);
    else if (nst == 2) cols_pass<FWD, 2>(P, g, sm, tws, ls, c0, s, first, last);
    else cols_pass<FWD, 1>(P, g, sm, tws, ls, c0, s, first, last);
    __syncthreads();
    s += nst;
  }
}

// ------------------------------------------------------------------ row FFTs with global I/O in the first / last pass
// k2_rows_embed_fft / k2_rows_ifft_crop restated the same way as k2_cols_fft8:
// the first pass gathers its bit-reversed inputs from global memory (the
// embedded, deconvolved row of X for the forward; the row of G for the
// inverse) and the last pass writes its outputs (the whole row of G; the
// cropped, deconvolved row of Z), twiddles in shared memory.
// Row-FFT shared-memory layout: one pad per 8 and per 64 elements, so that the
// first pass's stores (groups in bit-reversed order, F_ROWS_COAL) as well as the
// strided accesses of the later passes spread over the 16-B bank groups.
#ifndef F_ROWS_COAL
#define F_ROWS_COAL 1  // coalesced first-pass loads of the row FFTs
#endif
__host__ __device__ __forceinline__ int rpad(int i) { return i + (i >> 3) + (i >> 6); }
__host__ __device__ __forceinline__ int rpad_len(int L) { return L + (L >> 3) + (L >> 6); }
template <bool FWD, int NST>
__device__ __forceinline__ void rows_pass(const NfP& P, const cplx* __restrict__ src, cplx* __restrict__ dst,
                                          const double* __restrict__ deconv, cplx* sm, const cplx* __restrict__ tws,
                                          int ls, int j0, int nr, int s, bool first, bool last) {
  constexpr int GN = 1 << NST;
  const int L = P.log_nov, N = P.n_ov, n = P.n, half = n / 2;
  const int h = 1 << (s - 1);
  const int groups = N / GN, nthr = groups * P.RW;
  for (int tix = threadIdx.x; tix < nthr; tix += blockDim.x) {
    const int rr = tix / groups, jn = tix - rr * groups;
    // first pass: thread jn takes the group whose 8 bit-reversed input positions are
    // rev3(m) * groups + jn, so a warp's loads cover contiguous segments of the row
    const int j = (F_ROWS_COAL && first) ? bitrev(jn, L - NST) : jn;
    const int jy = j0 + rr;  // coefficient row (y index) of this line
    const int jh = j & (h - 1);
    const int i0 = (j >> (s - 1)) * (GN * h) + jh;
    cplx* base = sm + rr * ls;
    cplx v[GN];
    if (first) {
#pragma unroll
      for (int m = 0; m < GN; ++m) {
        const int pos = bitrev(i0 + m, L);  // grid column held by bit-reversed position i0 + m
        cplx a = mk(0, 0);
        if (rr < nr) {
          if (FWD) {  // embedded X(i, jy) deconvolved, edge rows / slots zero
            const int i = (pos + half) & (N - 1);
            if (i < n && !(P.edges && (jy < P.p || jy >= n - P.p || i < P.p || i >= n - P.p)))
              a = cscale(src[(int64_t)jy * n + i], deconv[jy] * deconv[i]);
          } else {
            a = src[(int64_t)((jy - half + N) & (N - 1)) * N + pos];
          }
        }
        v[m] = a;
      }
    } else {
#pragma unroll
      for (int m = 0; m < GN; ++m) v[m] = base[rpad(i0 + m * h)];
    }
    r8_pass<FWD, NST>(v, jh, h, tws, L, s);
    if (last) {
      if (rr < nr) {
#pragma unroll
        for (int m = 0; m < GN; ++m) {
          const int pos = i0 + m * h;
          if (FWD) {
            dst[(int64_t)((jy - half + N) & (N - 1)) * N + pos] = v[m];
          } else {
            const int i = (pos + half) & (N - 1);  // crop: grid column pos -> coefficient index i
            if (i < n) {
              cplx z = cscale(v[m], deconv[jy] * deconv[i]);
              if (P.edges && (jy < P.p || jy >= n - P.p || i < P.p || i >= n - P.p)) z = mk(0, 0);
              dst[(int64_t)jy * n + i] = z;
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < GN; ++m) base[rpad(i0 + m * h)] = v[m];
    }
  }
}

#ifndef F_ROWS_MINB
#define F_ROWS_MINB 4  // resident row-FFT CTAs per SM the register budget is sized for
#endif
template <bool FWD>
__global__ void __launch_bounds__(256, F_ROWS_MINB) k2_rows_fft8(NfP P, const cplx* __restrict__ src, const double* __restrict__ deconv,
                             cplx* __restrict__ dst, const cplx* __restrict__ tw) {
  extern __shared__ cplx sm[];
  const int L = P.log_nov, N = P.n_ov;
  const int ls = rpad_len(N) + 1;
  cplx* tws = sm + P.RW * ls;
  const int j0 = blockIdx.x * P.RW, prob = blockIdx.y, nr = min(P.RW, P.n - j0);
  const cplx* s = FWD ? src + (int64_t)prob * P.n * P.n : src + (int64_t)prob * N * N;
  cplx* d = FWD ? dst + (int64_t)prob * N * N : dst + (int64_t)prob * P.n * P.n;
  for (int i = threadIdx.x; i < N / 2; i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  for (int st = 1; st <= L;) {
    const int nst = L - st + 1 >= 3 ? 3 : L - st + 1;
    const bool first = st == 1, last = st + nst > L;
    if (nst == 3) rows_pass<FWD, 3>(P, s, d, deconv, sm, tws, ls, j0, nr, st, first, last);
    else if (nst == 2) rows_pass<FWD, 2>(P, s, d, deconv, sm, tws, ls, j0, nr, st, first, last);
    else rows_pass<FWD, 1>(P, s, d, deconv, sm, tws, ls, j0, nr, st, first, last);
    __syncthreads();
    st += nst;
  }
}
