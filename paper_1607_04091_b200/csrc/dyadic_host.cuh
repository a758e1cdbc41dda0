// dyadic_host.cuh -- host side of the dyadic-grid evaluation,
// included into gs_capi.cu's internal namespace (shares fail / CK / DBuf /
// pmark).  The tiny integer-value eigenproblem is solved on the host; every
// table refinement level, the basis rows and the contractions run on the GPU
// (kernels_dyadic.cuh).
#pragma once
#include "kernels_dyadic.cuh"

// phi at the integers -p+2..p-1: the eigenvector of T(n, m) = 2 h(2n - m) for
// eigenvalue 1 with sum 1 (dyadic.cpp:14-35).  The (n+1) x n system is
// consistent; solved by Householder QR with column pivoting.
std::vector<double> dy_integer_values(int p) {
  const double* taps = gsdata::kFamilies[p - 1].taps;
  auto tap = [&](int k) { return (k < -p + 1 || k > p) ? 0.0 : taps[k + p - 1]; };
  const int n = 2 * p - 2, rows = n + 1;
  std::vector<double> A((size_t)rows * n, 0.0), b(rows, 0.0);
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) A[(size_t)r * n + c] = 2.0 * tap(2 * (r - p + 2) - (c - p + 2)) - (r == c ? 1.0 : 0.0);
  for (int c = 0; c < n; ++c) A[(size_t)n * n + c] = 1.0;
  b[n] = 1.0;
  const std::vector<double> A0 = A, b0 = b;
  std::vector<int> perm(n);
  for (int c = 0; c < n; ++c) perm[c] = c;
  for (int k = 0; k < n; ++k) {
    int best = k;  // pivot: the remaining column of largest norm
    double bn = -1.0;
    for (int c = k; c < n; ++c) {
      double s = 0.0;
      for (int r = k; r < rows; ++r) s += A[(size_t)r * n + c] * A[(size_t)r * n + c];
      if (s > bn) {
        bn = s;
        best = c;
      }
    }
    if (best != k) {
      for (int r = 0; r < rows; ++r) std::swap(A[(size_t)r * n + k], A[(size_t)r * n + best]);
      std::swap(perm[k], perm[best]);
    }
    const double nrm = std::sqrt(bn);
    if (nrm == 0.0) fail(GS_ERR_NUMERICAL, "integer value eigenproblem did not solve");
    const double alpha = A[(size_t)k * n + k] > 0 ? -nrm : nrm;
    std::vector<double> v(rows, 0.0);
    for (int r = k; r < rows; ++r) v[r] = A[(size_t)r * n + k];
    v[k] -= alpha;
    double vv = 0.0;
    for (int r = k; r < rows; ++r) vv += v[r] * v[r];
    for (int c = k; c < n; ++c) {
      double d = 0.0;
      for (int r = k; r < rows; ++r) d += v[r] * A[(size_t)r * n + c];
      d = 2.0 * d / vv;
      for (int r = k; r < rows; ++r) A[(size_t)r * n + c] -= d * v[r];
    }
    double d = 0.0;
    for (int r = k; r < rows; ++r) d += v[r] * b[r];
    d = 2.0 * d / vv;
    for (int r = k; r < rows; ++r) b[r] -= d * v[r];
  }
  std::vector<double> y(n), x(n);
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A[(size_t)i * n + j] * y[j];
    y[i] = s / A[(size_t)i * n + i];
  }
  for (int c = 0; c < n; ++c) x[perm[c]] = y[c];
  double res = 0.0;  // dyadic.cpp:30-32
  for (int r = 0; r < rows; ++r) {
    double s = -b0[r];
    for (int c = 0; c < n; ++c) s += A0[(size_t)r * n + c] * x[c];
    res += s * s;
  }
  if (std::sqrt(res) > 1e-10) fail(GS_ERR_NUMERICAL, "integer value eigenproblem did not solve");
  return x;
}

// All dyadic tables of family p at resolution R, resident on the device:
// table 0 = interior (support [-p+1, p]), 1..p = left edge functions k
// (support [0, p+k]), p+1..2p = right edge functions k (support [-(p+k), 0]).
struct DyTables {
  DyP P{};
  DBuf<double> buf, coef;  // tables; taps | left H | left h | right H | right h
  int64_t total = 0;
};

void dy_build(DyTables& T, int p, int R, bool edges, cudaStream_t st) {
  if (R < 0) fail(GS_ERR_DOMAIN, "resolution must be >= 0");
  if (R > 24) fail(GS_ERR_DOMAIN, "resolution out of range");
  DyP& P = T.P;
  P.p = p;
  P.R = R;
  P.ntab = (edges && p >= 2) ? 1 + 2 * p : 1;
  int64_t off = 0;
  for (int t = 0; t < P.ntab; ++t) {
    if (t == 0) {
      P.side[t] = 0;
      P.kidx[t] = 0;
      P.sb[t] = -p + 1;
      P.len[t] = ((int64_t)(2 * p - 1) << R) + 1;
    } else {
      const bool left = t <= p;
      const int k = left ? t - 1 : t - 1 - p;
      P.side[t] = left ? 1 : 2;
      P.kidx[t] = k;
      P.sb[t] = left ? 0 : -(p + k);
      P.len[t] = ((int64_t)(p + k) << R) + 1;
    }
    P.off[t] = off;
    off += P.len[t];
  }
  T.total = off;
  // level 0: integer seeds (dyadic.cpp:47-56, 84-94)
  std::vector<double> h0((size_t)off, 0.0);
  if (p == 1) {
    for (int64_t i = 0; i + 1 < P.len[0]; ++i) h0[(size_t)i] = 1.0;  // indicator of [0, 1) (dyadic.cpp:47-51)
  } else {
    std::vector<double> iv = dy_integer_values(p);
    for (size_t k = 0; k < iv.size(); ++k) h0[(size_t)((int64_t)(k + 1) << R)] = iv[k];
    const gsdata::FamilyData& f = gsdata::kFamilies[p - 1];
    for (int t = 1; t < P.ntab; ++t) {
      const bool left = P.side[t] == 1;
      const int k = P.kidx[t];
      const double* seed = left ? f.left_seed : f.right_seed;
      for (int d = 0; d <= p + k; ++d) {
        const int64_t num = left ? d : -d;
        h0[(size_t)(P.off[t] + ((num - P.sb[t]) << R))] = seed[k * 2 * p + d];
      }
    }
  }
  T.buf.upload(h0.data(), h0.size(), st);
  const gsdata::FamilyData& f = gsdata::kFamilies[p - 1];
  std::vector<double> c(2 * p);
  std::copy(f.taps, f.taps + 2 * p, c.begin());
  if (p >= 2) {
    c.insert(c.end(), f.left_H, f.left_H + p * p);
    c.insert(c.end(), f.left_h, f.left_h + p * (2 * p - 1));
    c.insert(c.end(), f.right_H, f.right_H + p * p);
    c.insert(c.end(), f.right_h, f.right_h + p * (2 * p - 1));
  }
  T.coef.upload(c.data(), c.size(), st);
  P.taps = T.coef.p;
  if (p >= 2) {
    P.H[0] = T.coef.p + 2 * p;
    P.h[0] = P.H[0] + p * p;
    P.H[1] = P.h[0] + p * (2 * p - 1);
    P.h[1] = P.H[1] + p * p;
  }
  if (p == 1) return;  // haar: the indicator needs no refinement
  int64_t maxlen = 0;
  for (int t = 0; t < P.ntab; ++t) maxlen = std::max(maxlen, P.len[t]);
  for (int r = 1; r <= R; ++r) {
    const int64_t step = 1LL << (R - r);
    const int64_t odd = (maxlen - step + 2 * step - 1) / (2 * step);
    k_dy_level<<<dim3(nblk(odd, 256), P.ntab), 256, 0, st>>>(P, T.buf.p, r);
    pmark("k_dy_level", st);
  }
  CKL();
}

void dy_copy_table(const DyTables& T, int t, double* out, cudaStream_t st) {
  CK(cudaMemcpyAsync(out, T.buf.p + T.P.off[t], T.P.len[t] * sizeof(double), cudaMemcpyDefault, st));
  CK(cudaStreamSynchronize(st));
}

// weval_1d / weval_2d (dyadic.cpp:172-230); coeffs / out host or device
void dy_weval(int dim, int p, int J, int R, const double* coeffs, int64_t ncoeffs, double* out, cudaStream_t st) {
  if (dim != 1 && dim != 2) fail(GS_ERR_DOMAIN, "dim must be 1 or 2");
  if (p < 1 || p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
  if (J < 0 || J > 24) fail(GS_ERR_DOMAIN, "scale J out of range");
  if ((1LL << J) < 2 * p) fail(GS_ERR_DOMAIN, "scale too small: 2^J must be >= 2p");
  if (R < J) fail(GS_ERR_DOMAIN, "resolution too coarse: R must be >= J");
  if (R > (dim == 1 ? 28 : 15)) fail(GS_ERR_DOMAIN, "resolution out of range");
  const int64_t n = 1LL << J, g = (1LL << R) + 1;
  if (ncoeffs != (dim == 1 ? n : n * n)) fail(GS_ERR_SHAPE, "coefficient vector has wrong length");
  if (!coeffs || !out) fail(GS_ERR_USAGE, "null buffer");
  DyTables T;
  dy_build(T, p, R - J, true, st);
  const int km = 4 * p + 2;
  DBuf<int> cnt, col;
  DBuf<double> val, din, dout, Z;
  cnt.alloc(g);
  col.alloc((size_t)g * km);
  val.alloc((size_t)g * km);
  k_dy_ell<<<nblk(g, 256), 256, 0, st>>>(T.P, T.buf.p, J, R, km, cnt.p, col.p, val.p);
  pmark("k_dy_ell", st);
  const double amp = std::exp2(0.5 * J);  // dyadic.cpp:135
  const double* c = coeffs;
  if (!is_device_ptr(coeffs)) {
    din.upload(coeffs, (size_t)ncoeffs, st);
    c = din.p;
  }
  const int64_t nout = dim == 1 ? g : g * g;
  const bool dev_out = is_device_ptr(out);
  double* o = out;
  if (!dev_out) {
    dout.alloc((size_t)nout);
    o = dout.p;
  }
  if (dim == 1) {
    k_dy_weval1<<<nblk(g, 256), 256, 0, st>>>(g, km, cnt.p, col.p, val.p, c, amp, o);
    pmark("k_dy_weval1", st);
  } else {
    Z.alloc((size_t)g * n);
    k_dy_rows<<<dim3(nblk(n, 128), (unsigned)g), 128, 0, st>>>(g, (int)n, km, cnt.p, col.p, val.p, c, amp, Z.p);
    pmark("k_dy_rows", st);
    k_dy_cols<<<dim3(nblk(g, 128), (unsigned)g), 128, 0, st>>>(g, (int)n, km, cnt.p, col.p, val.p, Z.p, amp, o);
    pmark("k_dy_cols", st);
  }
  CKL();
  if (!dev_out) CK(cudaMemcpyAsync(out, o, (size_t)nout * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}
