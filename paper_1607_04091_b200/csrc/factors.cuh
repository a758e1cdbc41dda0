// factors.cuh -- operator construction on the device ("init"):
// per sample point and axis, the diagonal factor D, the p left- and p right-
// edge factors L / R (boundary-corrected Daubechies), and the Kaiser-Bessel
// gridding window.  One thread per (problem, point, axis).
#pragma once
#include "gs_common.cuh"

#define GS_MAXP 8

// Family constants passed by value (kernel parameter bank).
struct FamDev {
  int p;
  int has_edges;
  double taps[2 * GS_MAXP];                          // k = -p+1..p
  double U[2][GS_MAXP * GS_MAXP];                    // [side][i*p+j], side 0 = left
  double V[2][GS_MAXP * (2 * GS_MAXP - 1)];          // [side][i*(2p-1)+j]
  double vz[2][GS_MAXP];                             // fixed point v_zero (real)
};

// m0(xi) = sum_k h_k e^{-2 pi i k xi}   (fourier.cpp:16-24)
__device__ cplx d_transfer(const FamDev& f, double xi) {
  cplx acc = mk(0.0, 0.0);
  int k = -f.p + 1;
  for (int i = 0; i < 2 * f.p; ++i, ++k) {
    cplx e = polar1((-GS_TWO_PI * (double)k) * xi);
    acc = cadd(acc, cscale(e, f.taps[i]));
  }
  return acc;
}

// (1 - e^{-2 pi i xi}) / (2 pi i xi), 1 at 0   (fourier.cpp:26-30)
__device__ cplx d_haar(double xi) {
  if (xi == 0.0) return mk(1.0, 0.0);
  cplx e = polar1(-GS_TWO_PI * xi);
  double a = 1.0 - e.x, b = -e.y, d = GS_TWO_PI * xi;
  double den = d * d;
  return mk((b * d) / den, (-a * d) / den);
}

// phihat(xi) = prod_{j=1..terms} m0(xi / 2^j), early exit |m0 - 1| < 1e-16
// (fourier.cpp:34-49)
__device__ cplx d_fourier_scaling(const FamDev& f, double xi, int terms) {
  if (f.p == 1) return d_haar(xi);
  cplx prod = mk(1.0, 0.0);
  double arg = xi;
  for (int j = 1; j <= terms; ++j) {
    arg *= 0.5;
    cplx fac = d_transfer(f, arg);
    prod = cmul(prod, fac);
    if (hypot(fac.x - 1.0, fac.y) < 1e-16) break;
  }
  return prod;
}

// Edge transforms by the depth-level two-scale recursion (fourier.cpp:85-120).
// phihat(xi / 2^(l+1)) is carried down the Horner loop instead of stored per
// level (same products in the same order as fourier.cpp:92-98), so any
// depth >= 1 is accepted.
__device__ void d_fourier_boundary(const FamDev& f, int side, double xi, int depth, int terms,
                                   cplx* out /* p */) {
  const int p = f.p;
  cplx amp = d_fourier_scaling(f, ldexp(xi, -depth), terms);  // phihat[depth]
  cplx acc[GS_MAXP], v2[2 * GS_MAXP - 1], nxt[GS_MAXP];
  for (int i = 0; i < p; ++i) acc[i] = mk(f.vz[side][i], 0.0);
  const double* U = f.U[side];
  const double* V = f.V[side];
  for (int l = depth - 1; l >= 0; --l) {
    double arg = ldexp(xi, -(l + 1));
    cplx step = side == 0 ? polar1(-GS_TWO_PI * arg) : polar1(GS_TWO_PI * arg);
    cplx phase = side == 0 ? polar1((-GS_TWO_PI * arg) * (double)p) : polar1((GS_TWO_PI * arg) * (double)(p + 1));
    for (int m = 0; m < 2 * p - 1; ++m) {
      v2[m] = cmul(amp, phase);
      phase = cmul(phase, step);
    }
    for (int i = 0; i < p; ++i) {
      cplx s = mk(0, 0), t = mk(0, 0);
      for (int j = 0; j < p; ++j) s = cadd(s, cscale(acc[j], U[i * p + j]));
      for (int j = 0; j < 2 * p - 1; ++j) t = cadd(t, cscale(v2[j], V[i * (2 * p - 1) + j]));
      nxt[i] = cadd(s, t);
    }
    for (int i = 0; i < p; ++i) acc[i] = nxt[i];
    if (l >= 1) amp = cmul(d_transfer(f, arg), amp);  // phihat[l] = m0(xi/2^(l+1)) phihat[l+1]
  }
  for (int i = 0; i < p; ++i) out[i] = acc[i];
}

// Per point record [D, L_0..L_{p-1}, R_0..R_{p-1}] (build_axis, freq2wave.cpp:45-76),
// optionally scaled by sqrt(mu) (x axis only, freq2wave.cpp:159-168).
// xi: [count] natural frequencies; rec: [count][1+2p].
__global__ void k_build_factors(FamDev f, const double* __restrict__ xi, const double* __restrict__ sqrtw,
                                int64_t count, int J, int depth, int terms, cplx* __restrict__ rec) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int p = f.p;
  const int R = 1 + (f.has_edges ? 2 * p : 0);
  double x = xi[i];
  double amp = exp2(-0.5 * (double)J);
  double scaled = ldexp(x, -J);
  cplx D = cscale(d_fourier_scaling(f, scaled, terms), amp);
  cplx* out = rec + i * R;
  double sw = sqrtw ? sqrtw[i] : 1.0;
  out[0] = sqrtw ? cscale(D, sw) : D;
  if (f.has_edges) {
    cplx vl[GS_MAXP], vr[GS_MAXP];
    d_fourier_boundary(f, 0, scaled, depth, terms, vl);
    d_fourier_boundary(f, 1, scaled, depth, terms, vr);
    cplx pl = cscale(polar1(GS_PI * x), amp);
    cplx pr = cscale(polar1(-GS_PI * x), amp);
    for (int c = 0; c < p; ++c) {
      cplx l = cmul(pl, vl[c]);
      cplx r = cmul(pr, vr[p - 1 - c]);
      if (sqrtw) {
        l = cscale(l, sw);
        r = cscale(r, sw);
      }
      out[1 + c] = l;
      out[1 + p + c] = r;
    }
  }
}

// wrap_half_open (freq2wave.cpp:15-19)
__device__ __forceinline__ double d_wrap(double z) {
  double w = z - floor(z + 0.5);
  if (w >= 0.5) w -= 1.0;
  return w;
}

// Kaiser-Bessel window of one axis (NfftPlan ctor, nufft.cpp:208-223, kb_kernel 173-177):
// base = (llround(pos) - w) mod n_ov, weights[t] = I0(beta sqrt(1 - (u/w)^2)), 0 if |u| > w.
__global__ void k_kb_window(const double* __restrict__ xi, int64_t count, int J, int n_ov, int w, double beta,
                            int* __restrict__ base, double* __restrict__ wts) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int S = 2 * w + 1;
  double z = d_wrap(ldexp(xi[i], -J));
  double pos = z * (double)n_ov;
  long long j0 = llround(pos);
  long long b = j0 - w;
  base[i] = (int)(((b % n_ov) + n_ov) % n_ov);
  if (!wts) return;  // base only (bin keys)
  for (int t = 0; t < S; ++t) {
    double u = pos - (double)(j0 - w + t);
    double q = 1.0 - (u / w) * (u / w);
    wts[i * S + t] = q < 0 ? 0.0 : cyl_bessel_i0(beta * sqrt(q));
  }
}
