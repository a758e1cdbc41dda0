// general_route.cuh -- the operator's general routes: T / T* composed exactly
// as the reference composes them (freq2wave.cpp:215-387) from the device
// NfftPlan and the uniform reduction at ANY length (plan.h: general FFT
// engine), for the option values the fused kernels of the configs do not take
// (non-power-of-two or > 4096 oversampled lengths -- sigma != 2 --, kernel
// half-widths w > 7, uniform DFT lengths > 8192 or non-power-of-two > 4096).
//   1D: y = D o F(x~) + L x[0:p] + R x[n-p:n];  z = F^H(conj(D) o y) (edges zeroed) + L^H y, R^H y
//   2D: interior 2D plan x Dx Dy, 4 corners, 2p side lines per axis through the 1D plans.
// Samples stay in the caller's order (no bin sort); the spreading of the
// general plan uses FP64 atomics.  Included by gs_capi.cu after struct gs_op.
#pragma once

// v = conj(D) o y (1D adjoint input, freq2wave.cpp:315); rec [B][M][Rr]
__global__ void k_g_conjd(int64_t M, int Rr, const cplx* __restrict__ rec, const cplx* __restrict__ y,
                          cplx* __restrict__ v) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int64_t i = (int64_t)blockIdx.y * M + m;
  v[i] = cmul(conj_(rec[i * Rr]), y[i]);
}

// side-line inputs of the 2D forward (freq2wave.cpp:273-301): for c < 2p,
// ly[b][c][j] = X(row_c, j) and lx[b][c][i] = X(i, col_c) on the interior
// [p, n-p), 0 elsewhere; row_c / col_c = c (< p) or n - 2p + c; X(i, j) = x[j n + i]
__global__ void k_g2_lines_in(int n, int p, const cplx* __restrict__ x, cplx* __restrict__ ly,
                              cplx* __restrict__ lx) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // c * n + k
  const int E = 2 * p;
  if (t >= (int64_t)E * n) return;
  const int b = blockIdx.y;
  const int c = (int)(t / n), k = (int)(t % n);
  const int e = c < p ? c : n - 2 * p + c;
  x += (int64_t)b * n * n;
  const bool in = k >= p && k < n - p;
  ly[((int64_t)b * E + c) * n + k] = in ? x[(int64_t)k * n + e] : mk(0, 0);
  lx[((int64_t)b * E + c) * n + k] = in ? x[(int64_t)e * n + k] : mk(0, 0);
}

// y_m = Dx Dy u2 + corners + sum_c Ax_c Dy uy_c + sum_c By_c Dx ux_c
// (freq2wave.cpp:252-301); rec = [D, L_0..L_{p-1}, R_0..R_{p-1}] so A_c = rec[1 + c], c < 2p
__global__ void k_g2_fwd_combine(int64_t M, int n, int p, int Rr, const cplx* __restrict__ recx,
                                 const cplx* __restrict__ recy, const cplx* __restrict__ u2,
                                 const cplx* __restrict__ uy, const cplx* __restrict__ ux, const cplx* __restrict__ x,
                                 cplx* __restrict__ y) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int b = blockIdx.y;
  const int64_t gi = (int64_t)b * M + m;
  const cplx* rx = recx + gi * Rr;
  const cplx* ry = recy + gi * Rr;
  const cplx Dx = rx[0], Dy = ry[0];
  cplx acc = cmul(cmul(Dx, Dy), u2[gi]);
  if (p >= 2) {
    const int E = 2 * p;
    x += (int64_t)b * n * n;
    for (int ci = 0; ci < 2; ++ci)      // corners: row block (Lx | Rx) x column block (Ly | Ry)
      for (int cj = 0; cj < 2; ++cj) {
        const int row0 = ci ? n - p : 0, col0 = cj ? n - p : 0;
        for (int c = 0; c < p; ++c) {
          cplx t = mk(0, 0);
          for (int r = 0; r < p; ++r) t = cadd(t, cmul(rx[1 + ci * p + r], x[(int64_t)(col0 + c) * n + row0 + r]));
          acc = cadd(acc, cmul(t, ry[1 + cj * p + c]));
        }
      }
    for (int c = 0; c < E; ++c) acc = cadd(acc, cmul(cmul(rx[1 + c], Dy), uy[((int64_t)b * E + c) * M + m]));
    for (int c = 0; c < E; ++c) acc = cadd(acc, cmul(cmul(ry[1 + c], Dx), ux[((int64_t)b * E + c) * M + m]));
  }
  y[gi] = acc;
}

// adjoint inputs (freq2wave.cpp:334-337, 364-383): v2 = conj(Dx Dy) y,
// vy_c = conj(Ax_c Dy) y, vx_c = conj(By_c Dx) y
__global__ void k_g2_adj_prep(int64_t M, int p, int Rr, const cplx* __restrict__ recx, const cplx* __restrict__ recy,
                              const cplx* __restrict__ y, cplx* __restrict__ v2, cplx* __restrict__ vy,
                              cplx* __restrict__ vx) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int b = blockIdx.y;
  const int64_t gi = (int64_t)b * M + m;
  const cplx* rx = recx + gi * Rr;
  const cplx* ry = recy + gi * Rr;
  const cplx Dx = rx[0], Dy = ry[0], u = y[gi];
  v2[gi] = cmul(conj_(cmul(Dx, Dy)), u);
  const int E = p >= 2 ? 2 * p : 0;
  for (int c = 0; c < E; ++c) {
    vy[((int64_t)b * E + c) * M + m] = cmul(conj_(cmul(rx[1 + c], Dy)), u);
    vx[((int64_t)b * E + c) * M + m] = cmul(conj_(cmul(ry[1 + c], Dx)), u);
  }
}

// Z = interior block of W (freq2wave.cpp:338-345) + side lines on the edge
// rows / columns (361-385); corners are written by k_g2_adj_corners
__global__ void k_g2_adj_assemble(int n, int p, const cplx* __restrict__ W, const cplx* __restrict__ wy,
                                  const cplx* __restrict__ wx, cplx* __restrict__ z) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * n) return;
  const int b = blockIdx.y;
  const int j = (int)(t / n), i = (int)(t % n);  // z[j n + i] = Z(i, j)
  const int64_t zi = (int64_t)b * n * n + t;
  if (p < 2) {
    z[zi] = W[zi];
    return;
  }
  const int E = 2 * p;
  const bool ii = i >= p && i < n - p, ji = j >= p && j < n - p;
  cplx v = mk(0, 0);
  if (ii && ji) v = W[zi];
  else if (!ii && ji) v = wy[((int64_t)b * E + (i < p ? i : i - (n - 2 * p))) * n + j];
  else if (ii && !ji) v = wx[((int64_t)b * E + (j < p ? j : j - (n - 2 * p))) * n + i];
  else return;  // corner: k_g2_adj_corners
  z[zi] = v;
}

// corners: Z(row_ri, col_cj) = sum_m conj(Ax(m, ri)) (y_m conj(By(m, cj)))
// (freq2wave.cpp:347-355); one CTA per entry, fixed-order block reduction
__global__ void k_g2_adj_corners(int64_t M, int n, int p, int Rr, const cplx* __restrict__ recx,
                                 const cplx* __restrict__ recy, const cplx* __restrict__ y, cplx* __restrict__ z) {
  __shared__ double red[32];
  const int E = 2 * p, b = blockIdx.y;
  const int ri = blockIdx.x / E, cj = blockIdx.x % E;
  const cplx* rx = recx + (int64_t)b * M * Rr;
  const cplx* ry = recy + (int64_t)b * M * Rr;
  y += (int64_t)b * M;
  cplx acc = mk(0, 0);
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x)
    acc = cadd(acc, cmul(conj_(rx[m * Rr + 1 + ri]), cmul(y[m], conj_(ry[m * Rr + 1 + cj]))));
  const double re = block_sum(acc.x, red);
  __syncthreads();
  const double im = block_sum(acc.y, red);
  const int i = ri < p ? ri : n - 2 * p + ri, j = cj < p ? cj : n - 2 * p + cj;
  if (threadIdx.x == 0) z[(int64_t)b * n * n + (int64_t)j * n + i] = mk(re, im);
}

namespace {

// device state of a general route (held by gs_op)
struct GeneralRoute {
  std::unique_ptr<NfftPlanDev> px, py, p2;  // 1D: px only; 2D: 2D plan + the two axis plans (vps = 2p)
  std::unique_ptr<UniformDev> uni;          // 1D uniform route at any DFT length
  DBuf<cplx> u, v, ly, lx, uy, ux;          // per-apply scratch
};

}  // namespace
