// gs_capi.cu -- host side of the B200 operator: validation (mirrors
// freq2wave.cpp:86-193), device-side construction, route dispatch for
// apply_forward / apply_adjoint, the device-resident CGLS loop and the C-ABI
// declared in include/gs_b200.h.  No torch types anywhere: plain CUDA runtime.
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gs_b200.h"
#include "factors.cuh"
#include "family_data.h"
#include "gs_common.cuh"
#include "host_common.cuh"
#include "kernels_nfft.cuh"
#include "kernels_nfft2d_fast.cuh"
#include "kernels_uniform.cuh"
#include "kernels_vec.cuh"
#include "kernels_cgls_fused.cuh"
#include "ndft.h"
#include "host_math.h"
#include "plan.h"

using namespace gsb;

namespace {

// v_zero = (I - U)^{-1} V 1 by partial-pivot LU (fourier.cpp:60-72)
bool fixed_point(const double* U, const double* V, int p, double* v) {
  std::vector<double> A(p * p), b(p, 0.0);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) A[i * p + j] = (i == j ? 1.0 : 0.0) - U[i * p + j];
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < 2 * p - 1; ++j) b[i] += V[i * (2 * p - 1) + j];
  std::vector<double> A0 = A, b0 = b;
  for (int k = 0; k < p; ++k) {
    int best = k;
    for (int i = k + 1; i < p; ++i)
      if (std::abs(A[i * p + k]) > std::abs(A[best * p + k])) best = i;
    if (best != k) {
      for (int j = 0; j < p; ++j) std::swap(A[k * p + j], A[best * p + j]);
      std::swap(b[k], b[best]);
    }
    double d = A[k * p + k];
    if (d == 0.0) return false;
    for (int i = k + 1; i < p; ++i) {
      double f = A[i * p + k] / d;
      for (int j = k + 1; j < p; ++j) A[i * p + j] -= f * A[k * p + j];
      b[i] -= f * b[k];
    }
  }
  for (int i = p - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < p; ++j) s -= A[i * p + j] * v[j];
    v[i] = s / A[i * p + i];
  }
  double res = 0, rn = 0;
  for (int i = 0; i < p; ++i) {
    double s = -b0[i];
    for (int j = 0; j < p; ++j) s += A0[i * p + j] * v[j];
    res += s * s;
    rn += b0[i] * b0[i];
  }
  return std::sqrt(res) <= 1e-10 * (1.0 + std::sqrt(rn));
}

FamDev make_family(int p) {
  FamDev f;
  std::memset(&f, 0, sizeof(f));
  f.p = p;
  f.has_edges = p >= 2;
  const gsdata::FamilyData& src = gsdata::kFamilies[p - 1];
  for (int i = 0; i < 2 * p; ++i) f.taps[i] = src.taps[i];
  if (p >= 2) {
    for (int side = 0; side < 2; ++side) {
      const double* H = side == 0 ? src.left_H : src.right_H;
      const double* h = side == 0 ? src.left_h : src.right_h;
      for (int i = 0; i < p * p; ++i) f.U[side][i] = H[i] / std::sqrt(2.0);  // scaling.cpp:63-70
      for (int i = 0; i < p * (2 * p - 1); ++i) f.V[side][i] = h[i] / std::sqrt(2.0);
      if (!fixed_point(f.U[side], f.V[side], p, f.vz[side]))
        fail(GS_ERR_NUMERICAL, "boundary_fourier_at_zero: singular fixed-point system");
    }
  }
  return f;
}

}  // namespace

#include "general_route.cuh"

// ====================================================================== op
struct gs_op {
  gs_op_desc d{};
  int dim = 1, p = 1, edges = 0, J = 0, B = 1, route = 0, device = 0;
  long long n = 0;
  int64_t M = 0, Nc = 0;
  bool weighted = false;
  int Rr = 1;  // record length 1 + 2p
  int depth = 30, terms = 48;
  FamDev fam;
  double uniform_eps = 0.0;
  // FFT twiddles
  DBuf<cplx> tw;
  int logLmax = 0;
  // uniform / tensor
  UniP up{}, upx{}, upy{};
  int64_t Ma = 0, Mb = 0;
  DBuf<cplx> rec_u, rec_ax, rec_ay, ph_u, ph_x, ph_y;
  // NFFT
  NfP np{};
  double beta = 0;
  DBuf<double> deconv;
  DBuf<int> perm, base_x, base_y, bins;
  bool fast2d = false;  // kernels_nfft2d_fast.cuh path (w = 6, p <= 4)
  int cap = 1;          // chunk capacity per problem (2D work list)
  DBuf<int> ch_tile, ch_s0, ch_s1, ch_count, tcs;
  DBuf<uint4> ch_rows;  // per chunk: row starts + warps per band (k2f_chunk_rows)
  bool balanced = false;  // uneven static bands: the DMMA kernels run the balanced band schedule
  DBuf<int> fs_start;  // per (problem, tile): range of fold sources (k2_fold_src)
  DBuf<int4> fsrc;
  DBuf<int2> cov;        // per grid coordinate: (tile, offset) of the regions covering it
  DBuf<int> covn;
  DBuf<unsigned> units;  // fast 2D interpolation work units (k2f_build_units)
  DBuf<int> ucount;
  DBuf<double> wts_x, wts_y;
  DBuf<cplx> rec_x, rec_y;
  DBuf<double> sqrtw;  // internal order ([B][M]) or empty
  // workspace
  DBuf<cplx> G, lines, TB, TL, TLF, TC, TCF, W;
  DBuf<cplx> EP;  // 1D route: per-CTA edge-sum partials of k_n1_spread
  bool general = false;  // general route (general_route.cuh): caller-order samples, plan-based T / T*
  GeneralRoute gen;
  DBuf<double> nd_pts;  // NDFT_1D route: wrapped scaled points (caller order)
  DBuf<cplx> nd_part;   // NDFT_1D route: split partial sums
  DBuf<cplx> stage_a, stage_b;
  gs_cgls_session* solve_cache = nullptr;  // workspace of the last gs_solve_least_squares
  std::mutex mu;

  size_t device_bytes() const {
    return tw.bytes() + rec_u.bytes() + rec_ax.bytes() + rec_ay.bytes() + deconv.bytes() + perm.bytes() +
           base_x.bytes() + base_y.bytes() + bins.bytes() + wts_x.bytes() + wts_y.bytes() + rec_x.bytes() +
           rec_y.bytes() + sqrtw.bytes() + G.bytes() + lines.bytes() + TB.bytes() + TL.bytes() + TLF.bytes() + TC.bytes() + TCF.bytes() +
           W.bytes() + stage_a.bytes() + stage_b.bytes() + nd_pts.bytes() + nd_part.bytes();
  }
};

namespace {

const int kSmemMax = 227 * 1024;

template <class K>
void allow_big_smem(K kernel) {
  cudaFuncAttributes a;
  CK(cudaFuncGetAttributes(&a, kernel));
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax - (int)a.sharedSizeBytes));
}

// cudaFuncSetAttribute applies to the current device only: once per device
// ordinal, serialised across threads (call after cudaSetDevice)
void set_smem_attrs() {
  static std::mutex m;
  static std::vector<char> done_dev;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(m);
  if (dev < (int)done_dev.size() && done_dev[dev]) return;
  allow_big_smem(k_uni_fwd);
  allow_big_smem(k_uni_adj);
  allow_big_smem(k_uni_cgls_iter);
  allow_big_smem(k_n1_embed_fft);
  allow_big_smem(k_n1_ifft_crop);
  allow_big_smem(k2_rows_embed_fft);
  allow_big_smem(k2_cols_fft);
  allow_big_smem(k2_lines_fft);
  allow_big_smem(k2_spread);
  allow_big_smem(k2_cols_ifft);
  allow_big_smem(k2_cols_fft8<true>);
  allow_big_smem(k2_rows_fft8<true>);
  allow_big_smem(k2_rows_fft8<false>);
  allow_big_smem(k2_cols_fft8<false>);
  allow_big_smem(k2_rows_ifft_crop);
  allow_big_smem(k2_edges);
  allow_big_smem(k2f_interp<1>);
  allow_big_smem(k2f_interp<2>);
  allow_big_smem(k2f_interp<3>);
  allow_big_smem(k2f_interp<4>);
  allow_big_smem(k2f_spread<1>);
  allow_big_smem(k2f_spread<2>);
  allow_big_smem(k2f_spread<3>);
  allow_big_smem(k2f_spread<4>);
  allow_big_smem(k2f_interp_mma<1, false>);
  allow_big_smem(k2f_interp_mma<1, true>);
  allow_big_smem(k2f_interp_mma<2, false>);
  allow_big_smem(k2f_interp_mma<2, true>);
  allow_big_smem(k2f_interp_mma<3, false>);
  allow_big_smem(k2f_interp_mma<3, true>);
  allow_big_smem(k2f_interp_mma<4, false>);
  allow_big_smem(k2f_interp_mma<4, true>);
  allow_big_smem(k2f_spread_mma<1, false>);
  allow_big_smem(k2f_spread_mma<1, true>);
  allow_big_smem(k2f_spread_mma<2, false>);
  allow_big_smem(k2f_spread_mma<2, true>);
  allow_big_smem(k2f_spread_mma<3, false>);
  allow_big_smem(k2f_spread_mma<3, true>);
  allow_big_smem(k2f_spread_mma<4, false>);
  allow_big_smem(k2f_spread_mma<4, true>);
  if ((int)done_dev.size() <= dev) done_dev.resize(dev + 1, 0);
  done_dev[dev] = 1;
}

void make_twiddles(gs_op* op, long long Lmax, cudaStream_t st) {
  op->logLmax = ilog2(std::max<long long>(Lmax, 2));
  long long L = 1LL << op->logLmax;
  std::vector<cplx> h(L / 2);
  for (long long k = 0; k < L / 2; ++k) {
    double a = -GS_TWO_PI * (double)k / (double)L;
    h[k] = mk(std::cos(a), std::sin(a));
  }
  op->tw.upload(h.data(), h.size(), st);
}

// __global__ helpers used only at construction
__global__ void k_gather_d(const double* __restrict__ src, const int* __restrict__ perm, int64_t M, int64_t total,
                           double* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  dst[i] = src[(i / M) * M + perm[i]];
}
__global__ void k_keys(const int* __restrict__ by, const int* __restrict__ bx, int64_t M, int64_t total, int T, int nt,
                       int band, unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  unsigned long long prob = (unsigned long long)(i / M);
  // 2D: tile-major, then inside the tile either the cell row-major (band = 0) or
  // band-major with bands of `band` rows, column-major inside a band (the DMMA
  // kernels: a warp's 4- / 8-sample K steps then span ~band columns instead of
  // a row stretch, so fewer column tiles are reached); 1D: cell
  unsigned long long bin = (unsigned long long)bx[i];
  if (by) {
    const int r = by[i] % T, c = bx[i] % T;
    const int in_tile = band > 0 ? (r / band) * (band * T) + c * band + r % band : r * T + c;
    bin = (unsigned long long)(((by[i] / T) * nt + bx[i] / T) * T * T + in_tile);
  }
  keys[i] = (prob << 32) | bin;
  vals[i] = (int)(i - (int64_t)prob * M);
}
__global__ void k_bin_starts(const unsigned long long* __restrict__ keys, int64_t total, int64_t M, int B, int nbins,
                             int scale, int* __restrict__ starts) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t per = nbins + 1;
  if (i >= (int64_t)B * per) return;
  unsigned long long prob = (unsigned long long)(i / per), bin = (unsigned long long)(i % per) * scale;
  unsigned long long key = (prob << 32) | bin;
  int64_t lo = 0, hi = total;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  starts[i] = (int)(lo - (int64_t)prob * M);
}

// sort the samples of every problem by bin; perm[s] = original index
void sort_bins(gs_op* op, const int* by, const int* bx, int nbins, int T, int nt, int band, cudaStream_t st) {
  const int64_t total = op->M * op->B;
  DBuf<unsigned long long> k_in, k_out;
  DBuf<int> v_in;
  k_in.alloc(total);
  k_out.alloc(total);
  v_in.alloc(total);
  op->perm.alloc(total);
  k_keys<<<nblk(total, 256), 256, 0, st>>>(by, bx, op->M, total, T, nt, band, k_in.p, v_in.p);
  CKL();
  size_t tmp = 0;
  int end_bit = 32 + std::max(1, ilog2(op->B + 1));
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k_in.p, k_out.p, v_in.p, op->perm.p, (int)total, 0, end_bit, st));
  DBuf<char> scratch;
  scratch.alloc(tmp);
  CK(cub::DeviceRadixSort::SortPairs(scratch.p, tmp, k_in.p, k_out.p, v_in.p, op->perm.p, (int)total, 0, end_bit, st));
  op->bins.alloc((size_t)op->B * (nbins + 1));
  k_bin_starts<<<nblk((int64_t)op->B * (nbins + 1), 256), 256, 0, st>>>(k_out.p, total, op->M, op->B, nbins,
                                                                        by ? T * T : 1, op->bins.p);
  CKL();
  CK(cudaStreamSynchronize(st));
}

void build_factors(gs_op* op, const double* d_xi, const double* d_sw, int64_t count, cplx* rec, cudaStream_t st) {
  k_build_factors<<<nblk(count, 128), 128, 0, st>>>(op->fam, d_xi, d_sw, count, op->J, op->depth, op->terms, rec);
  CKL();
}

UniP make_uni(gs_op* op, int64_t M, double eps) {
  UniSetup s = uniform_setup(M, eps, op->n);
  if (s.n2 > 8192) fail(GS_ERR_DOMAIN, "uniform route: DFT length " + std::to_string(s.n2) + " exceeds 8192 on this build");
  UniP P{};
  P.n = (int)op->n;
  P.M = (int)M;
  P.q = (int)s.q;
  P.N2 = (int)s.n2;
  P.logN2 = is_pow2(s.n2) ? ilog2(s.n2) : -1;
  if (P.logN2 < 0 && s.n2 > 4096) fail(GS_ERR_DOMAIN, "uniform route: non power-of-two DFT length > 4096");
  P.p = op->p;
  P.edges = op->edges;
  P.eps = eps;
  P.phase_step = GS_PI * eps * (double)M / (double)op->n;  // nufft.cpp:412
  return P;
}
// phase tables of a uniform setup (see UniP), computed with the reference's formulas
void attach_phases(UniP& P, DBuf<cplx>& buf, cudaStream_t st) {
  std::vector<cplx> h((size_t)P.n + P.M);
  for (int l = 0; l < P.n; ++l) {
    const double a = P.phase_step * (double)l;
    h[l] = mk(std::cos(a), std::sin(a));
  }
  for (int m = 0; m < P.M; ++m) {
    const double xi = P.eps / (double)P.n * ((double)m - (double)P.M / 2.0);
    const double a = GS_PI * (double)P.n * xi;
    h[(size_t)P.n + m] = mk(std::cos(a), std::sin(a));
  }
  buf.upload(h.data(), h.size(), st);
  P.ph_in = buf.p;
  P.ph_out = buf.p + P.n;
}
// tensor-route passes: many CTAs of one short vector each -> small CTAs, one wave
constexpr int UNI_TENSOR_THREADS = 128;
// k_uni_cgls_iter with the problem resident in shared memory: FFT buffer +
// twiddles + p, x, s (n) + r, q (M) + factor records (M x Rr); 0 when it does not fit
size_t uni_cg_resident_smem(const UniP& P, int Rr) {
  const size_t buf = P.logN2 >= 0 ? (size_t)fpad_len(P.N2) + P.N2 / 2 : 2 * (size_t)P.N2;
  const size_t bytes = (buf + 3 * (size_t)P.n + 2 * (size_t)P.M + (size_t)P.M * Rr) * sizeof(cplx);
  return bytes + UNI_MAX_WARPS * 32 * sizeof(double) <= (size_t)kSmemMax ? bytes : 0;
}
// single-CTA 1D FFT kernels: padded line + staged twiddles
size_t n1_fft_smem(const NfP& P) { return (size_t)(fpad_len(P.n_ov) + P.n_ov / 2) * sizeof(cplx); }
size_t uni_smem(const UniP& P) { return (size_t)(P.logN2 >= 0 ? fpad_len(P.N2) : 2 * P.N2) * sizeof(cplx); }
// k_uni_* and the fused CGLS iteration: FFT buffer + the staged twiddle table
size_t uni_smem_tw(const UniP& P) { return uni_smem(P) + (P.logN2 >= 0 ? (size_t)(P.N2 / 2) * sizeof(cplx) : 0); }

bool interp_mma();  // kernel variant selectors (defined with the launch code)
bool cols_fft8();
bool rows_fft8();
bool spread_mma();
static_assert(F_T / F_WARPS == F_T / F_IWARPS, "the DMMA kernels share the in-tile band order");
bool fold_src();


// ------------------------------------------------------------------ family / transform evaluation
// (fourier.cpp:34-130 at caller frequencies; densify, freq2wave.cpp:389-450)
__global__ void k_eval_scaling(FamDev f, const double* __restrict__ xi, int64_t n, int terms, cplx* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = d_fourier_scaling(f, xi[i], terms);
}
__global__ void k_eval_boundary(FamDev f, int side, const double* __restrict__ xi, int64_t n, int depth, int terms,
                                cplx* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) d_fourier_boundary(f, side, xi[i], depth, terms, out + i * f.p);
}
// dense_axis_row (freq2wave.cpp:392-418) for every point: rows[m][c], unweighted,
// default depth / terms as the reference's densify uses
__global__ void k_densify_axis(FamDev f, const double* __restrict__ coords, int dim, int axis, int64_t M, int J,
                               int n, cplx* __restrict__ rows) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= M) return;
  const double xi = coords[m * dim + axis];
  const double scaled = ldexp(xi, -J);
  const double amp = exp2(-0.5 * (double)J);
  const cplx interior = cscale(d_fourier_scaling(f, scaled, 48), amp);
  cplx* row = rows + m * n;
  for (int c = 0; c < n; ++c) {
    const long long k = (long long)c - n / 2;
    row[c] = cmul(interior, polar1((-GS_TWO_PI * (double)k) * scaled));
  }
  if (f.p >= 2) {
    cplx vl[GS_MAXP], vr[GS_MAXP];
    d_fourier_boundary(f, 0, scaled, 30, 48, vl);
    d_fourier_boundary(f, 1, scaled, 30, 48, vr);
    const cplx pl = cscale(polar1(GS_PI * xi), amp), pr = cscale(polar1(-GS_PI * xi), amp);
    for (int c = 0; c < f.p; ++c) {
      row[c] = cmul(pl, vl[c]);
      row[n - f.p + c] = cmul(pr, vr[f.p - 1 - c]);
    }
  }
}
// out (M x cols, column-major): 1D weight * rx(c); 2D weight * (rx(i) ry(j)) at column j n + i.
// (freq2wave.cpp:443 writes weight * rx(i) * ry(j); scaling the finished
// product instead keeps the weighted section exactly sqrt(mu) times the
// unweighted one, the property the reference's test_freq2wave.cpp:198-219 pins)
__global__ void k_densify_out(int dim, int64_t M, int n, const cplx* __restrict__ rx, const cplx* __restrict__ ry,
                              const double* __restrict__ sw, cplx* __restrict__ out) {
  const int64_t cols = dim == 1 ? n : (int64_t)n * n;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= M * cols) return;
  const int64_t m = e % M, col = e / M;
  const double w = sw ? sw[m] : 1.0;
  if (dim == 1) {
    out[e] = cscale(rx[m * n + col], w);
    return;
  }
  const int64_t i = col % n, j = col / n;
  out[e] = cscale(cmul(rx[m * n + i], ry[m * n + j]), w);
}

// ------------------------------------------------------------------ construction
gs_op* create(const gs_op_desc* dsc) {
  if (!dsc) fail(GS_ERR_USAGE, "null descriptor");
  std::unique_ptr<gs_op> op(new gs_op);
  gs_op_desc d = *dsc;
  op->d = d;
  op->dim = d.dim;
  op->J = d.J;
  op->B = d.batch <= 0 ? 1 : d.batch;
  op->M = d.M;
  op->depth = d.boundary_depth;
  op->terms = d.product_terms;
  if (d.family_p < 1 || d.family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
  op->p = d.family_p;
  if (op->p >= 2) {  // checked per point by the reference (fourier.cpp:36, 87); haar evaluates neither
    if (d.product_terms < 1) fail(GS_ERR_DOMAIN, "fourier_scaling: terms must be >= 1");
    if (d.boundary_depth < 1) fail(GS_ERR_DOMAIN, "fourier_boundary: depth must be >= 1");
  }
  op->edges = op->p >= 2;
  op->Rr = 1 + (op->edges ? 2 * op->p : 0);
  // freq2wave.cpp:93-102
  if (d.dim != 1 && d.dim != 2) fail(GS_ERR_DOMAIN, "sampling set must be 1D or 2D");
  if (d.M <= 0 || !d.coords) fail(GS_ERR_SHAPE, "empty sampling set");
  if (d.J < 0 || d.J > 24) fail(GS_ERR_DOMAIN, "scale J out of range");
  op->n = 1LL << d.J;
  if (op->n < 2 * op->p) fail(GS_ERR_DOMAIN, "scale too small: 2^J must be >= 2p");
  if (d.M > (int64_t)INT32_MAX / 2) fail(GS_ERR_DOMAIN, "too many samples per problem");
  const int64_t M = d.M, B = op->B, total = M * B;
  const double* coords = d.coords;
  for (int64_t i = 0; i < total * d.dim; ++i)
    if (!std::isfinite(coords[i])) fail(GS_ERR_DOMAIN, "non-finite frequency");
  std::vector<double> sw;
  if (d.weights) {  // freq2wave.cpp:105-114
    op->weighted = true;
    sw.resize(total);
    for (int64_t i = 0; i < total; ++i) {
      if (!(d.weights[i] > 0.0)) fail(GS_ERR_DOMAIN, "weights must be positive");
      sw[i] = std::sqrt(d.weights[i]);
    }
  }
  const bool has_bw = !std::isnan(d.bandwidth);
  std::vector<double> xi_x(total), xi_y(d.dim == 2 ? total : 0);
  for (int64_t i = 0; i < total; ++i) {
    xi_x[i] = coords[i * d.dim];
    if (d.dim == 2) xi_y[i] = coords[i * 2 + 1];
  }
  auto check_axis = [&](const std::vector<double>& xi) {  // freq2wave.cpp:123-140
    for (double v : xi) {
      if (has_bw) {
        if (std::abs(v) > d.bandwidth) fail(GS_ERR_DOMAIN, "bandwidth exceeded: |xi| > bandwidth");
      } else {
        double z = std::ldexp(v, -d.J);
        if (!(z >= -0.5 && z < 0.5))
          fail(GS_ERR_DOMAIN,
               "bandwidth exceeded: scaled point outside [-1/2, 1/2) (pass a bandwidth to allow periodized rows)");
      }
    }
  };
  check_axis(xi_x);
  if (d.dim == 2) check_axis(xi_y);

  op->device = d.device;
  CK(cudaSetDevice(d.device));
  set_smem_attrs();
  op->fam = make_family(op->p);
  op->Nc = d.dim == 1 ? op->n : op->n * op->n;
  cudaStream_t st = 0;

  // ---- route selection (freq2wave.cpp:170-191, plus the exact tensor route)
  const bool allow_u = d.allow_uniform_fast_path != 0;
  std::vector<double> zeta(M);
  if (d.dim == 1) {
    bool uni = allow_u;
    double eps0 = 0;
    for (int64_t b = 0; uni && b < B; ++b) {
      for (int64_t m = 0; m < M; ++m) zeta[m] = std::ldexp(xi_x[b * M + m], -d.J);
      double e = 0;
      if (!detect_uniform(zeta.data(), M, op->n, &e)) uni = false;
      else if (b == 0) eps0 = e;
      else if (e != eps0) uni = false;
    }
    if (uni) {
      try {  // DFT lengths the fused single-CTA kernels cannot hold take the general uniform route
        op->up = make_uni(op.get(), M, eps0);
      } catch (const GsError&) {
        op->general = true;
      }
    }
    op->route = uni ? GS_ROUTE_UNIFORM_1D : (d.exact_ndft ? GS_ROUTE_NDFT_1D : GS_ROUTE_NFFT_1D);
    op->uniform_eps = uni ? eps0 : 0.0;
  } else {
    bool ten = allow_u && d.allow_tensor_route != 0;
    int64_t Mb = 1;
    if (ten) {
      while (Mb < M && coords[2 * Mb] == coords[0]) ++Mb;
      if (M % Mb != 0) ten = false;
    }
    int64_t Ma = ten ? M / Mb : 0;
    double ex = 0, ey = 0;
    std::vector<double> ax, ay;
    for (int64_t b = 0; ten && b < B; ++b) {
      const double* c = coords + b * M * 2;
      for (int64_t a = 0; ten && a < Ma; ++a)
        for (int64_t k = 0; k < Mb; ++k)
          if (c[2 * (a * Mb + k)] != c[2 * a * Mb] || c[2 * (a * Mb + k) + 1] != c[2 * k + 1]) {
            ten = false;
            break;
          }
      if (!ten) break;
      std::vector<double> za(Ma), zb(Mb);
      for (int64_t a = 0; a < Ma; ++a) za[a] = std::ldexp(c[2 * a * Mb], -d.J);
      for (int64_t k = 0; k < Mb; ++k) zb[k] = std::ldexp(c[2 * k + 1], -d.J);
      double e1 = 0, e2 = 0;
      if (!detect_uniform(za.data(), Ma, op->n, &e1) || !detect_uniform(zb.data(), Mb, op->n, &e2)) ten = false;
      else if (b == 0) {
        ex = e1;
        ey = e2;
      } else if (e1 != ex || e2 != ey) ten = false;
    }
    if (ten) {
      try {
        op->upx = make_uni(op.get(), Ma, ex);
        op->upy = make_uni(op.get(), Mb, ey);
      } catch (const GsError&) {
        ten = false;
      }
    }
    op->route = ten ? GS_ROUTE_TENSOR_2D : GS_ROUTE_NFFT_2D;
    op->Ma = Ma;
    op->Mb = Mb;
  }

  // ---- per-route construction, all per-point work on the device
  DBuf<double> d_xi_x, d_xi_y, d_sw;
  if (op->route == GS_ROUTE_UNIFORM_1D && op->general) {
    op->gen.uni = uniform_build(M, op->uniform_eps, op->n, (int)B);  // uniform_ndft_fft at any length
    d_xi_x.upload(xi_x.data(), total, st);
    if (op->weighted) op->sqrtw.upload(sw.data(), total, st);
    op->rec_u.alloc(total * op->Rr);
    build_factors(op.get(), d_xi_x.p, op->weighted ? op->sqrtw.p : nullptr, total, op->rec_u.p, st);
    CK(cudaStreamSynchronize(st));
  } else if (op->route == GS_ROUTE_UNIFORM_1D) {
    attach_phases(op->up, op->ph_u, st);
    make_twiddles(op.get(), op->up.N2, st);
    d_xi_x.upload(xi_x.data(), total, st);
    if (op->weighted) op->sqrtw.upload(sw.data(), total, st);
    op->rec_u.alloc(total * op->Rr);
    build_factors(op.get(), d_xi_x.p, op->weighted ? op->sqrtw.p : nullptr, total, op->rec_u.p, st);
  } else if (op->route == GS_ROUTE_NDFT_1D) {
    // the reference builds plan_x here (freq2wave.cpp:175-176): same option checks
    if ((d.sigma > 0 ? d.sigma : 2.0) < 1.25) fail(GS_ERR_DOMAIN, "oversampling factor must be >= 1.25");
    if ((d.w > 0 ? d.w : 6) < 2) fail(GS_ERR_DOMAIN, "kernel half-width must be >= 2");
    // direct NDFT on the wrapped scaled points the plan would get (freq2wave.cpp:79-84, 176)
    std::vector<double> zw(total);
    for (int64_t i = 0; i < total; ++i) zw[i] = wrap_half_open(std::ldexp(xi_x[i], -d.J));
    op->nd_pts.upload(zw.data(), total, st);
    d_xi_x.upload(xi_x.data(), total, st);
    if (op->weighted) op->sqrtw.upload(sw.data(), total, st);
    op->rec_x.alloc(total * op->Rr);
    build_factors(op.get(), d_xi_x.p, op->weighted ? op->sqrtw.p : nullptr, total, op->rec_x.p, st);
    CK(cudaStreamSynchronize(st));
  } else if (op->route == GS_ROUTE_TENSOR_2D) {
    const int64_t Ma = op->Ma, Mb = op->Mb;
    std::vector<double> ax(B * Ma), ay(B * Mb);
    for (int64_t b = 0; b < B; ++b) {
      for (int64_t a = 0; a < Ma; ++a) ax[b * Ma + a] = coords[(b * M + a * Mb) * 2];
      for (int64_t k = 0; k < Mb; ++k) ay[b * Mb + k] = coords[(b * M + k) * 2 + 1];
    }
    make_twiddles(op.get(), std::max(op->upx.N2, op->upy.N2), st);
    attach_phases(op->upx, op->ph_x, st);
    attach_phases(op->upy, op->ph_y, st);
    DBuf<double> dax, day;
    dax.upload(ax.data(), ax.size(), st);
    day.upload(ay.data(), ay.size(), st);
    op->rec_ax.alloc(B * Ma * op->Rr);
    op->rec_ay.alloc(B * Mb * op->Rr);
    build_factors(op.get(), dax.p, nullptr, B * Ma, op->rec_ax.p, st);
    build_factors(op.get(), day.p, nullptr, B * Mb, op->rec_ay.p, st);
    if (op->weighted) op->sqrtw.upload(sw.data(), total, st);
    op->W.alloc(B * Ma * op->n);
    CK(cudaStreamSynchronize(st));
  } else {
    // NfftPlan constants (nufft.cpp:190-230)
    const double sigma = d.sigma > 0 ? d.sigma : 2.0;
    const int w = d.w > 0 ? d.w : 6;
    if (sigma < 1.25) fail(GS_ERR_DOMAIN, "oversampling factor must be >= 1.25");
    if (w < 2) fail(GS_ERR_DOMAIN, "kernel half-width must be >= 2");
    const int n_ov = (int)std::ceil(sigma * (double)op->n / 2.0) * 2;
    if (!is_pow2(n_ov) || n_ov > 4096 || 2 * w + 1 > 16) {
      // option values the fused gridding kernels do not take: the general route
      op->general = true;
      op->np.n = (int)op->n;
      op->np.n_ov = n_ov;
      op->np.p = op->p;
      op->np.edges = op->edges;
      op->np.S = 2 * w + 1;
      op->np.M = M;
      std::vector<double> zx(total), zy(d.dim == 2 ? total : 0);
      for (int64_t i = 0; i < total; ++i) zx[i] = wrap_half_open(std::ldexp(xi_x[i], -d.J));
      for (int64_t i = 0; i < (int64_t)zy.size(); ++i) zy[i] = wrap_half_open(std::ldexp(xi_y[i], -d.J));
      const int e = op->edges ? op->p : 0;
      const int Nn[2] = {(int)op->n, (int)op->n};
      if (d.dim == 1) {
        op->gen.px = nfft_plan_build(1, Nn, M, (int)B, zx.data(), sigma, w, st);
      } else {
        std::vector<double> pts(2 * total);  // 2D plan axes: 0 = y, 1 = x (freq2wave.cpp:183-190)
        for (int64_t i = 0; i < total; ++i) {
          pts[2 * i] = zy[i];
          pts[2 * i + 1] = zx[i];
        }
        op->gen.p2 = nfft_plan_build(2, Nn, M, (int)B, pts.data(), sigma, w, st);
        if (op->edges) {
          op->gen.px = nfft_plan_build(1, Nn, M, (int)B, zx.data(), sigma, w, st, 2 * op->p);
          op->gen.py = nfft_plan_build(1, Nn, M, (int)B, zy.data(), sigma, w, st, 2 * op->p);
        }
      }
      NfftPlanDev* core = d.dim == 1 ? op->gen.px.get() : op->gen.p2.get();
      if (op->edges) {
        core->lo = e;
        core->hi = (int)op->n - e;
      }
      d_xi_x.upload(xi_x.data(), total, st);
      if (op->weighted) op->sqrtw.upload(sw.data(), total, st);
      op->rec_x.alloc(total * op->Rr);
      build_factors(op.get(), d_xi_x.p, op->weighted ? op->sqrtw.p : nullptr, total, op->rec_x.p, st);
      if (d.dim == 2) {
        d_xi_y.upload(xi_y.data(), total, st);
        op->rec_y.alloc(total * op->Rr);
        build_factors(op.get(), d_xi_y.p, nullptr, total, op->rec_y.p, st);
      }
      CK(cudaStreamSynchronize(st));
      CKL();
      return op.release();
    }
    {
      double width = 2.0 * w;
      double t = (width / sigma) * (width / sigma) * (sigma - 0.5) * (sigma - 0.5) - 0.8;
      op->beta = GS_PI * std::sqrt(std::max(t, 1.0));
    }
    std::vector<double> dec(op->n);
    for (long long k = -op->n / 2; k < op->n / 2; ++k)
      dec[k + op->n / 2] = 1.0 / kb_transform((double)k / (double)n_ov, w, op->beta);
    op->deconv.upload(dec.data(), dec.size(), st);
    make_twiddles(op.get(), n_ov, st);
    NfP& P = op->np;
    P.n = (int)op->n;
    P.n_ov = n_ov;
    P.log_nov = ilog2(n_ov);
    P.p = op->p;
    P.edges = op->edges;
    P.S = 2 * w + 1;
    P.M = M;
    op->fast2d = d.dim == 2 && P.S == F_S && op->p <= 4 && n_ov >= 2 * F_R;
    P.T = op->fast2d ? F_T : std::min(16, n_ov);
    P.R = P.T + P.S - 1;
    P.nt = (n_ov + P.T - 1) / P.T;
#ifndef F_CWMAX
#define F_CWMAX 8
#endif
#ifndef F_CWBUDGET  // shared-memory budget of the column-FFT CTAs (bytes of column lines)
#define F_CWBUDGET (120 * 1024)
#endif
    P.CW = std::max(1, std::min(F_CWMAX, (int)((F_CWBUDGET) / ((fpad_len(n_ov) + 1) * (int)sizeof(cplx)))));
    while (n_ov % P.CW) --P.CW;
#ifndef F_RWPTS  // grid points per row-FFT CTA (256 threads, one 8-point group each at 2048)
#define F_RWPTS 2048
#endif
    P.RW = std::max(1, std::min(8, F_RWPTS / n_ov));
    d_xi_x.upload(xi_x.data(), total, st);
    if (d.dim == 2) d_xi_y.upload(xi_y.data(), total, st);
    // 1. windows in the caller's order -> bin keys -> sort
    DBuf<int> bx0, by0;
    bx0.alloc(total);
    k_kb_window<<<nblk(total, 256), 256, 0, st>>>(d_xi_x.p, total, d.J, n_ov, w, op->beta, bx0.p, nullptr);
    CKL();
    if (d.dim == 2) {
      by0.alloc(total);
      k_kb_window<<<nblk(total, 256), 256, 0, st>>>(d_xi_y.p, total, d.J, n_ov, w, op->beta, by0.p, nullptr);
      CKL();
      // band-major order inside tiles for the DMMA kernels (their bands are F_T / F_WARPS rows);
      // the DFMA A/B variants walk rows and keep the row-major order
      const int band = (op->fast2d && interp_mma() && spread_mma()) ? F_T / F_WARPS : 0;
      sort_bins(op.get(), by0.p, bx0.p, P.nt * P.nt, P.T, P.nt, band, st);
    } else {
      sort_bins(op.get(), nullptr, bx0.p, n_ov, 1, 1, 0, st);
    }
    // 2. sorted coordinates -> windows and factors in sorted order
    DBuf<double> sx, sy, ssw;
    sx.alloc(total);
    k_gather_d<<<nblk(total, 256), 256, 0, st>>>(d_xi_x.p, op->perm.p, M, total, sx.p);
    op->base_x.alloc(total);
    op->wts_x.alloc(total * P.S + 2);  // +2: 16-B staging reads may round past the end
    k_kb_window<<<nblk(total, 256), 256, 0, st>>>(sx.p, total, d.J, n_ov, w, op->beta, op->base_x.p, op->wts_x.p);
    if (op->weighted) {
      d_sw.upload(sw.data(), total, st);
      op->sqrtw.alloc(total);
      k_gather_d<<<nblk(total, 256), 256, 0, st>>>(d_sw.p, op->perm.p, M, total, op->sqrtw.p);
    }
    op->rec_x.alloc(total * op->Rr);
    build_factors(op.get(), sx.p, op->weighted ? op->sqrtw.p : nullptr, total, op->rec_x.p, st);
    if (d.dim == 2) {
      sy.alloc(total);
      k_gather_d<<<nblk(total, 256), 256, 0, st>>>(d_xi_y.p, op->perm.p, M, total, sy.p);
      op->base_y.alloc(total);
      op->wts_y.alloc(total * P.S + 2);
      k_kb_window<<<nblk(total, 256), 256, 0, st>>>(sy.p, total, d.J, n_ov, w, op->beta, op->base_y.p, op->wts_y.p);
      op->rec_y.alloc(total * op->Rr);
      build_factors(op.get(), sy.p, nullptr, total, op->rec_y.p, st);
      const int64_t ntiles = (int64_t)P.nt * P.nt;
      // work list: (tile, sample range) chunks; the generic kernels use one
      // chunk per tile (empty ones included), the fast ones skip empty tiles
      // and split dense tiles into chunks of <= kChunk samples
      std::vector<int> starts((size_t)B * (ntiles + 1));
      CK(cudaMemcpy(starts.data(), op->bins.p, starts.size() * sizeof(int), cudaMemcpyDeviceToHost));
      const int kChunk = F_CHUNK;
      const char* ec_env = getenv("GS_B200_EVEN_CHUNKS");
      const bool even_chunks = !(ec_env && atoi(ec_env) == 0);
      std::vector<std::vector<int>> ct(B), c0(B), c1(B);
      std::vector<int> tcs((size_t)B * (ntiles + 1));
      int cap = 1;
      for (int64_t b = 0; b < B; ++b) {
        const int* sb = starts.data() + b * (ntiles + 1);
        int* tb = tcs.data() + b * (ntiles + 1);
        for (int64_t t = 0; t < ntiles; ++t) {
          tb[t] = (int)ct[b].size();
          const int a = sb[t], e = sb[t + 1];
          if (!op->fast2d) {
            ct[b].push_back((int)t);
            c0[b].push_back(a);
            c1[b].push_back(e);
            continue;
          }
          // dense tiles: equal chunks (a tile of 150 samples is 75 + 75, not 144 + 6), rounded
          // up to whole K steps of 4 samples; GS_B200_EVEN_CHUNKS=0 restores the greedy split
          int step = kChunk;
          if (even_chunks && e - a > kChunk) {
            const int k = (e - a + kChunk - 1) / kChunk;
            step = std::min(kChunk, ((e - a + k - 1) / k + 3) / 4 * 4);
          }
          for (int s = a; s < e; s += step) {
            ct[b].push_back((int)t);
            c0[b].push_back(s);
            c1[b].push_back(std::min(e, s + step));
          }
        }
        tb[ntiles] = (int)ct[b].size();
        cap = std::max(cap, (int)ct[b].size());
      }
      std::vector<int> h_t((size_t)B * cap, 0), h_0((size_t)B * cap, 0), h_1((size_t)B * cap, 0), h_n(B);
      for (int64_t b = 0; b < B; ++b) {
        h_n[b] = (int)ct[b].size();
        for (size_t k = 0; k < ct[b].size(); ++k) {
          h_t[b * cap + k] = ct[b][k];
          h_0[b * cap + k] = c0[b][k];
          h_1[b * cap + k] = c1[b][k];
        }
      }
      op->cap = cap;
      op->ch_tile.upload(h_t.data(), h_t.size(), st);
      op->ch_s0.upload(h_0.data(), h_0.size(), st);
      op->ch_s1.upload(h_1.data(), h_1.size(), st);
      op->ch_count.upload(h_n.data(), h_n.size(), st);
      op->tcs.upload(tcs.data(), tcs.size(), st);
      if (op->fast2d) {
        op->ch_rows.alloc((size_t)B * cap);
        // row starts + the balanced schedule's warps per band; the balanced DMMA kernels are used
        // when the longest static band of a chunk exceeds the balanced run by > 5 % over the operator
        DBuf<unsigned long long> bal;
        bal.alloc(2);
        CK(cudaMemsetAsync(bal.p, 0, 2 * sizeof(unsigned long long), st));
        k2f_chunk_rows<<<nblk((int64_t)B * cap, 128), 128, 0, st>>>(op->ch_tile.p, op->ch_s0.p, op->ch_s1.p,
                                                                   op->ch_count.p, (int64_t)B * cap, cap, M, P.nt,
                                                                   op->base_y.p, op->ch_rows.p, bal.p);
        CKL();
        unsigned long long hb[2] = {0, 0};
        CK(cudaMemcpyAsync(hb, bal.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const char* benv = getenv("GS_B200_BALANCE");  // 0 / 1 force the static / balanced kernels (A/B, tests)
        op->balanced = benv ? atoi(benv) != 0 : (double)hb[0] > 1.05 * (double)hb[1];
      }
      if (op->fast2d) {  // fold sources per tile (k2_fold_src): same order as k2_fold_tiles' coverage loops
        std::vector<int> fst((size_t)B * (ntiles + 1));
        std::vector<int4> fs;
        const int dmax = (P.R + P.T - 1) / P.T;
        std::vector<int> ct_t, ct_o;  // covering tiles / offsets of a tile's rows (same for columns)
        for (int64_t b = 0; b < B; ++b) {
          const int* tb = tcs.data() + b * (ntiles + 1);
          for (int tyy = 0; tyy < P.nt; ++tyy)
            for (int txx = 0; txx < P.nt; ++txx) {
              fst[b * (ntiles + 1) + tyy * P.nt + txx] = (int)fs.size();
              auto covers = [&](int t0, std::vector<int>& tt, std::vector<int>& oo) {
                tt.clear();
                oo.clear();
                for (int d = 0; d <= dmax && d < P.nt; ++d) {
                  const int t = ((t0 - d) % P.nt + P.nt) % P.nt;
                  const int o = ((t0 * P.T - t * P.T) % n_ov + n_ov) % n_ov;
                  bool any = false;
                  for (int a = 0; a < P.T && t0 * P.T + a < n_ov; ++a) any |= (o + a) % n_ov < P.R;
                  if (any) {
                    tt.push_back(t);
                    oo.push_back(o);
                  }
                }
              };
              std::vector<int> ry_t, ry_o, rx_t, rx_o;
              covers(tyy, ry_t, ry_o);
              covers(txx, rx_t, rx_o);
              for (size_t i = 0; i < ry_t.size(); ++i)
                for (size_t j = 0; j < rx_t.size(); ++j) {
                  const int tl = ry_t[i] * P.nt + rx_t[j];
                  for (int ch = tb[tl]; ch < tb[tl + 1]; ++ch) fs.push_back(int4{ch, ry_o[i], rx_o[j], 0});
                }
            }
          fst[b * (ntiles + 1) + ntiles] = (int)fs.size();
        }
        op->fs_start.upload(fst.data(), fst.size(), st);
        op->fsrc.upload(fs.data(), fs.size(), st);
        CK(cudaStreamSynchronize(st));
      }
      {  // coverage of each grid coordinate by tile regions (k2_fold_tiles)
        std::vector<int2> hc((size_t)n_ov * MAX_COVER, int2{0, 0});
        std::vector<int> hn(n_ov);
        int tl[MAX_COVER], ll[MAX_COVER];
        for (int r = 0; r < n_ov; ++r) {
          hn[r] = cover(r, P.T, P.R, P.nt, n_ov, tl, ll);
          for (int k = 0; k < hn[r]; ++k) hc[(size_t)r * MAX_COVER + k] = int2{tl[k], ll[k]};
        }
        op->cov.upload(hc.data(), hc.size(), st);
        op->covn.upload(hn.data(), hn.size(), st);
      }
      if (op->fast2d && !interp_mma()) {  // work units of the DFMA interpolation variant only
        op->units.alloc(total);
        op->ucount.alloc((size_t)B * cap);
        k2f_build_units<<<nblk((int64_t)B * cap, 128), 128, 0, st>>>(op->ch_tile.p, op->ch_s0.p, op->ch_s1.p,
                                                                     op->ch_count.p, cap, (int)B, (int)M, P.nt,
                                                                     op->base_x.p, op->base_y.p,
                                                                     op->units.p, op->ucount.p);
        CKL();
      }
      op->G.alloc((size_t)B * n_ov * n_ov);
      op->TB.alloc((size_t)B * cap * P.R * P.R);
      if (op->edges) {
        op->lines.alloc((size_t)B * 4 * op->p * n_ov);
        op->TL.alloc((size_t)B * cap * 2 * 2 * op->p * P.R);
        op->TC.alloc((size_t)B * cap * 4 * op->p * op->p);
        op->TLF.alloc((size_t)B * 2 * P.nt * 2 * op->p * P.R);
        op->TCF.alloc((size_t)B * ((cap + K2_CGROUP - 1) / K2_CGROUP) * 4 * op->p * op->p);
      }
    } else {
      op->G.alloc((size_t)B * n_ov);
      if (op->edges) op->EP.alloc((size_t)B * ((n_ov + N1_SPREAD_CELLS - 1) / N1_SPREAD_CELLS) * 2 * op->p);
    }
    CKL();
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaStreamSynchronize(st));
  CKL();
  return op.release();
}

// ------------------------------------------------------------------ per-kernel timing
// When armed by gs_profile_pair, every launch in forward_dev / adjoint_dev is
// followed by an event on the launching stream; consecutive events bracket
// exactly one kernel.
// 2D spreading variant: FP64 tensor cores (default) or the lane-per-column
// DFMA kernel (GS_B200_SPREAD=dfma, for A/B measurements)
bool interp_mma() {
  static const bool on = [] {
    const char* e = std::getenv("GS_B200_INTERP");
    return !(e && std::string(e) == "dfma");
  }();
  return on;
}
bool fold_src() {
  static const bool on = [] {
    const char* e = std::getenv("GS_B200_FOLD");
    return !(e && std::string(e) == "cover");
  }();
  return on;
}
bool cols_fft8() {  // radix-8 column FFTs with global I/O in the first / last pass (default for n_ov = 8^k)
  static const bool on = [] {
    const char* e = std::getenv("GS_B200_COLFFT");
    return !(e && std::string(e) == "smem");
  }();
  return on;
}
bool rows_fft8() {  // row FFTs with global I/O in the first / last pass (default)
  static const bool on = [] {
    const char* e = std::getenv("GS_B200_ROWFFT");
    return !(e && std::string(e) == "smem");
  }();
  return on;
}
// seeded pseudo-random complex fill in [-1, 1)^2 (splitmix64 of the index): profiling inputs
__global__ void k_fill_hash(cplx* __restrict__ v, int64_t n, unsigned long long seed) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto mix = [](unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  const unsigned long long a = mix(seed + 2 * (unsigned long long)i), b = mix(seed + 2 * (unsigned long long)i + 1);
  v[i] = mk((double)(a >> 11) * (2.0 / 9007199254740992.0) - 1.0, (double)(b >> 11) * (2.0 / 9007199254740992.0) - 1.0);
}
bool spread_mma() {
  static const bool on = [] {
    const char* e = std::getenv("GS_B200_SPREAD");
    return !(e && std::string(e) == "dfma");
  }();
  return on;
}



// ------------------------------------------------------------------ general routes (general_route.cuh)
void general_forward(gs_op* op, const cplx* x, cplx* y, cudaStream_t st) {
  GeneralRoute& G = op->gen;
  const int B = op->B, n = (int)op->n, p = op->p, e = op->edges ? p : 0;
  const int64_t M = op->M;
  if (op->dim == 1) {
    G.u.alloc((size_t)B * M);
    if (G.uni) uniform_forward(*G.uni, x, e, n - e, G.u.p, st);
    else nfft_plan_forward(*G.px, x, G.u.p, st);
    op1d_epilogue_launch(M, B, G.u.p, op->route == GS_ROUTE_UNIFORM_1D ? op->rec_u.p : op->rec_x.p, p, op->edges, x,
                         n, y, st);
    return;
  }
  const int E = op->edges ? 2 * p : 0;
  G.u.alloc((size_t)B * M);
  nfft_plan_forward(*G.p2, x, G.u.p, st);
  if (E) {
    G.ly.alloc((size_t)B * E * n);
    G.lx.alloc((size_t)B * E * n);
    G.uy.alloc((size_t)B * E * M);
    G.ux.alloc((size_t)B * E * M);
    k_g2_lines_in<<<dim3(nblk((int64_t)E * n, 256), B), 256, 0, st>>>(n, p, x, G.ly.p, G.lx.p);
    pmark("k_g2_lines_in", st);
    nfft_plan_forward(*G.py, G.ly.p, G.uy.p, st);
    nfft_plan_forward(*G.px, G.lx.p, G.ux.p, st);
  }
  k_g2_fwd_combine<<<dim3(nblk(M, 128), B), 128, 0, st>>>(M, n, op->edges ? p : 1, op->Rr, op->rec_x.p, op->rec_y.p,
                                                           G.u.p, G.uy.p, G.ux.p, x, y);
  pmark("k_g2_fwd_combine", st);
  CKL();
}

void general_adjoint(gs_op* op, const cplx* y, cplx* z, cudaStream_t st) {
  GeneralRoute& G = op->gen;
  const int B = op->B, n = (int)op->n, p = op->p;
  const int64_t M = op->M;
  if (op->dim == 1) {
    const cplx* rec = op->route == GS_ROUTE_UNIFORM_1D ? op->rec_u.p : op->rec_x.p;
    G.v.alloc((size_t)B * M);
    k_g_conjd<<<dim3(nblk(M, 256), B), 256, 0, st>>>(M, op->Rr, rec, y, G.v.p);
    pmark("k_g_conjd", st);
    if (G.uni) uniform_adjoint(*G.uni, G.v.p, z, st);
    else nfft_plan_adjoint(*G.px, G.v.p, z, st);
    if (op->edges) op1d_edges_launch(M, B, rec, p, y, n, z, st);
    CKL();
    return;
  }
  const int E = op->edges ? 2 * p : 0;
  G.v.alloc((size_t)B * M);
  G.u.alloc(std::max((size_t)B * M, (size_t)B * n * n));
  if (E) {
    G.uy.alloc((size_t)B * E * M);
    G.ux.alloc((size_t)B * E * M);
    G.ly.alloc((size_t)B * E * n);
    G.lx.alloc((size_t)B * E * n);
  }
  k_g2_adj_prep<<<dim3(nblk(M, 128), B), 128, 0, st>>>(M, op->edges ? p : 0, op->Rr, op->rec_x.p, op->rec_y.p, y,
                                                        G.v.p, G.uy.p, G.ux.p);
  pmark("k_g2_adj_prep", st);
  nfft_plan_adjoint(*G.p2, G.v.p, G.u.p, st);  // W
  if (E) {
    nfft_plan_adjoint(*G.py, G.uy.p, G.ly.p, st);  // side lines along y (x-edge rows)
    nfft_plan_adjoint(*G.px, G.ux.p, G.lx.p, st);  // side lines along x (y-edge columns)
  }
  k_g2_adj_assemble<<<dim3(nblk((int64_t)n * n, 256), B), 256, 0, st>>>(n, op->edges ? p : 1, G.u.p, G.ly.p, G.lx.p, z);
  pmark("k_g2_adj_assemble", st);
  if (E) {
    k_g2_adj_corners<<<dim3(E * E, B), 256, 0, st>>>(M, n, p, op->Rr, op->rec_x.p, op->rec_y.p, y, z);
    pmark("k_g2_adj_corners", st);
  }
  CKL();
}

// ------------------------------------------------------------------ applies
// x, y are device pointers; perm_io: samples in the caller's order (true) or
// the internal bin-sorted order (false, used inside CGLS).
// npart (tensor route only): per-vector partials of ||y||^2 from the last pass, [B][Ma]
// n1q (1D NFFT route inside CGLS): the interpolation applies the deferred r
// update and writes ||q||^2 partials; the spreading runs the q-step
// pre_a (tensor route): a CGLS vector update the x-pass CTAs apply first
void forward_dev(gs_op* op, const cplx* x, cplx* y, bool perm_io, cudaStream_t st, double* npart = nullptr,
                 const N1QStep* n1q = nullptr, const UniPre* pre_a = nullptr) {
  const int B = op->B;
  if (op->general) {
    general_forward(op, x, y, st);
    return;
  }
  switch (op->route) {
    case GS_ROUTE_UNIFORM_1D: {
      const UniP& P = op->up;
      k_uni_fwd<<<dim3(1, B), 256, uni_smem_tw(P), st>>>(P, x, Strided{op->n, 0, 1}, op->rec_u.p, op->M * op->Rr, y,
                                                     Strided{op->M, 0, 1}, nullptr, 0, op->tw.p, op->logLmax, nullptr,
                                                     UniPre{});
      pmark("k_uni_fwd", st);
      break;
    }
    case GS_ROUTE_TENSOR_2D: {
      const int64_t n = op->n, Ma = op->Ma, Mb = op->Mb;
      // W(a, j) = sum_i ax_a(i) X(i, j): one vector per column j
      k_uni_fwd<<<dim3((unsigned)n, B), UNI_TENSOR_THREADS, uni_smem_tw(op->upx), st>>>(
          op->upx, x, Strided{n * n, n, 1}, op->rec_ax.p, Ma * op->Rr, op->W.p, Strided{Ma * n, 1, n}, nullptr, 0,
          op->tw.p, op->logLmax, nullptr, pre_a ? *pre_a : UniPre{});
      pmark("k_uni_fwd[x-pass]", st);
      // Y(a, b) = sum_j ay_b(j) W(a, j): one vector per row a
      k_uni_fwd<<<dim3((unsigned)Ma, B), UNI_TENSOR_THREADS, uni_smem_tw(op->upy), st>>>(
          op->upy, op->W.p, Strided{Ma * n, n, 1}, op->rec_ay.p, Mb * op->Rr, y, Strided{op->M, Mb, 1},
          op->weighted ? op->sqrtw.p : nullptr, op->M, op->tw.p, op->logLmax, npart, UniPre{});
      pmark("k_uni_fwd[y-pass]", st);
      break;
    }
    case GS_ROUTE_NDFT_1D: {
      const NdftShape s{1, 1, (int)op->n, op->M, B};
      const int e = op->edges ? op->p : 0;
      ndft_forward_launch(s, op->nd_pts.p, x, y, e, (int)op->n - e, op->rec_x.p, op->p, op->edges, op->nd_part, st);
      break;
    }
    case GS_ROUTE_NFFT_1D: {
      const NfP& P = op->np;
      k_n1_embed_fft<<<B, 256, n1_fft_smem(P), st>>>(P, x, op->deconv.p, op->G.p, op->tw.p, op->logLmax);
      pmark("k_n1_embed_fft", st);
      k_n1_interp<<<dim3(nblk(op->M, 128), B), 128, 0, st>>>(P, op->base_x.p, op->wts_x.p, op->rec_x.p, op->G.p, x,
                                                              perm_io ? op->perm.p : nullptr, y,
                                                              n1q ? *n1q : N1QStep{});
      pmark("k_n1_interp", st);
      break;
    }
    case GS_ROUTE_NFFT_2D: {
      const NfP& P = op->np;
      if (op->logLmax == P.log_nov && rows_fft8())
        k2_rows_fft8<true><<<dim3((P.n + P.RW - 1) / P.RW, B), 256,
                              ((size_t)P.RW * (rpad_len(P.n_ov) + 1) + P.n_ov / 2) * sizeof(cplx), st>>>(
            P, x, op->deconv.p, op->G.p, op->tw.p);
      else
        k2_rows_embed_fft<<<dim3((P.n + P.RW - 1) / P.RW, B), 256, (size_t)P.RW * (fpad_len(P.n_ov) + 1) * sizeof(cplx), st>>>(P, x, op->deconv.p, op->G.p, op->tw.p,
                                                                          op->logLmax);
      pmark("k2_rows_embed_fft", st);
      if (op->logLmax == P.log_nov && cols_fft8())
        k2_cols_fft8<true><<<dim3(P.n_ov / P.CW, B), F_COLS_THREADS,
                              ((size_t)P.CW * (fpad_len(P.n_ov) + 1) + P.n_ov / (F_COLS_QW ? 4 : 2)) * sizeof(cplx), st>>>(P, op->G.p,
                                                                                                        op->tw.p);
      else
        k2_cols_fft<<<dim3(P.n_ov / P.CW, B), 256, (size_t)P.CW * (fpad_len(P.n_ov) + 1) * sizeof(cplx), st>>>(
            P, op->G.p, op->tw.p, op->logLmax);
      pmark("k2_cols_fft", st);
      if (P.edges) {
        k2_lines_fft<<<dim3(4 * P.p, B), 256, n1_fft_smem(P), st>>>(P, x, op->deconv.p, op->lines.p, op->tw.p,
                                                                           op->logLmax);
        pmark("k2_lines_fft", st);
      }
      if (op->fast2d) {
        const dim3 grid(op->cap, B);
        const int* pp = perm_io ? op->perm.p : nullptr;
#define GS_F_INTERP(PP)                                                                                            \
  if (interp_mma() && op->balanced)                                                                                \
    k2f_interp_mma<PP, true><<<grid, 32 * F_IWARPS * F_IMSPLIT, FInterpM<PP>::bytes(), st>>>(                      \
        P, op->ch_tile.p, op->ch_s0.p, op->ch_s1.p, op->ch_count.p, op->ch_rows.p, op->cap, op->base_x.p, op->base_y.p,            \
        op->wts_x.p, op->wts_y.p, op->rec_x.p, op->rec_y.p, op->G.p, op->lines.p, x, pp, y);                        \
  else if (interp_mma())                                                                                           \
    k2f_interp_mma<PP, false><<<grid, 32 * F_IWARPS * F_IMSPLIT, FInterpM<PP>::bytes(), st>>>(                     \
        P, op->ch_tile.p, op->ch_s0.p, op->ch_s1.p, op->ch_count.p, op->ch_rows.p, op->cap, op->base_x.p, op->base_y.p,            \
        op->wts_x.p, op->wts_y.p, op->rec_x.p, op->rec_y.p, op->G.p, op->lines.p, x, pp, y);                        \
  else                                                                                                             \
    k2f_interp<PP><<<grid, F_ITHREADS, FInterp<PP>::bytes(), st>>>(                                              \
        P, op->ch_tile.p, op->ch_s0.p, op->ch_s1.p, op->ch_count.p, op->cap, op->units.p, op->ucount.p,             \
        op->base_x.p, op->base_y.p, op->wts_x.p, op->wts_y.p, op->rec_x.p, op->rec_y.p, op->G.p, op->lines.p, x,   \
        pp, y)
        switch (op->p) {
          case 1: GS_F_INTERP(1); break;
          case 2: GS_F_INTERP(2); break;
          case 3: GS_F_INTERP(3); break;
          default: GS_F_INTERP(4); break;
        }
#undef GS_F_INTERP
        pmark("k2f_interp", st);
      } else {
        k2_interp<<<dim3(nblk(op->M, 128), B), 128, 0, st>>>(P, op->base_x.p, op->base_y.p, op->wts_x.p, op->wts_y.p,
                                                              op->rec_x.p, op->rec_y.p, op->G.p, op->lines.p, x,
                                                              perm_io ? op->perm.p : nullptr, y);
        pmark("k2_interp", st);
      }
      break;
    }
  }
  CKL();
}

// CGLS s-step (k_cg_sstep's arguments) a route may fuse into its last adjoint kernel
struct SStep {
  CgState* st;
  cplx* p;
  double tol;
  double* hist;
  int hist_stride;
};

// returns true when the route ran the s-step `ss` itself (NFFT_1D: in k_n1_ifft_crop)
// npart (tensor route only): per-vector partials of ||z||^2 from the last pass, [B][n]
// pre_a / pre_b (tensor route): CGLS vector updates the y-pass / x-pass CTAs apply first
bool adjoint_dev(gs_op* op, const cplx* y, cplx* z, bool perm_io, cudaStream_t st, const SStep* ss = nullptr,
                 double* npart = nullptr, const N1QStep* n1q = nullptr, const UniPre* pre_a = nullptr,
                 const UniPre* pre_b = nullptr) {
  bool fused_sstep = false;
  const int B = op->B;
  if (op->general) {
    general_adjoint(op, y, z, st);
    return false;
  }
  switch (op->route) {
    case GS_ROUTE_UNIFORM_1D: {
      const UniP& P = op->up;
      k_uni_adj<<<dim3(1, B), 256, uni_smem_tw(P), st>>>(P, y, Strided{op->M, 0, 1}, nullptr, 0, op->rec_u.p,
                                                     op->M * op->Rr, z, Strided{op->n, 0, 1}, op->tw.p, op->logLmax, nullptr,
                                                     UniPre{});
      pmark("k_uni_adj", st);
      break;
    }
    case GS_ROUTE_TENSOR_2D: {
      const int64_t n = op->n, Ma = op->Ma, Mb = op->Mb;
      // V(a, j) = sum_b conj(ay_b(j)) (sqrt(mu) y)(a, b): one vector per row a
      k_uni_adj<<<dim3((unsigned)Ma, B), UNI_TENSOR_THREADS, uni_smem_tw(op->upy), st>>>(
          op->upy, y, Strided{op->M, Mb, 1}, op->weighted ? op->sqrtw.p : nullptr, op->M, op->rec_ay.p, Mb * op->Rr,
          op->W.p, Strided{Ma * n, n, 1}, op->tw.p, op->logLmax, nullptr, pre_a ? *pre_a : UniPre{});
      pmark("k_uni_adj[y-pass]", st);
      // X(i, j) = sum_a conj(ax_a(i)) V(a, j): one vector per column j
      k_uni_adj<<<dim3((unsigned)n, B), UNI_TENSOR_THREADS, uni_smem_tw(op->upx), st>>>(
          op->upx, op->W.p, Strided{Ma * n, 1, n}, nullptr, 0, op->rec_ax.p, Ma * op->Rr, z, Strided{n * n, n, 1},
          op->tw.p, op->logLmax, npart, pre_b ? *pre_b : UniPre{});
      pmark("k_uni_adj[x-pass]", st);
      break;
    }
    case GS_ROUTE_NDFT_1D: {
      const NdftShape s{1, 1, (int)op->n, op->M, B};
      const int e = op->edges ? op->p : 0;
      ndft_adjoint_launch(s, op->nd_pts.p, y, z, e, (int)op->n - e, op->rec_x.p, op->p, op->edges, op->nd_part, st);
      break;
    }
    case GS_ROUTE_NFFT_1D: {
      const NfP& P = op->np;
      const int nparts = (P.n_ov + N1_SPREAD_CELLS - 1) / N1_SPREAD_CELLS;
      k_n1_spread<<<dim3(nparts, B), N1_SPREAD_THREADS, 0, st>>>(P, op->bins.p, op->wts_x.p, op->rec_x.p, y,
                                                                perm_io ? op->perm.p : nullptr, op->G.p, op->EP.p,
                                                                n1q ? *n1q : N1QStep{});
      pmark("k_n1_spread", st);
      k_n1_ifft_crop<<<B, 256, n1_fft_smem(P), st>>>(P, op->G.p, op->deconv.p, op->EP.p, nparts, z, op->tw.p,
                                                      op->logLmax, ss ? ss->st : nullptr, ss ? ss->p : nullptr,
                                                      ss ? ss->tol : 0.0, ss ? ss->hist : nullptr,
                                                      ss ? ss->hist_stride : 0);
      fused_sstep = ss != nullptr;
      pmark("k_n1_ifft_crop", st);
      break;
    }
    case GS_ROUTE_NFFT_2D: {
      const NfP& P = op->np;
      const int ntiles = P.nt * P.nt;
      if (op->fast2d) {
        const dim3 grid(op->cap, B);
        const int* pp = perm_io ? op->perm.p : nullptr;
#define GS_F_SPREAD(PP)                                                                                          \
  if (spread_mma() && op->balanced)                                                                              \
    k2f_spread_mma<PP, true><<<grid, 32 * F_MWARPS, FSpreadM<PP>::bytes(), st>>>(                               \
        P, op->ch_tile.p, op->ch_s0.p, op->ch_s1.p, op->ch_count.p, op->ch_rows.p, op->cap, op->base_x.p, op->base_y.p,          \
        op->wts_x.p, op->wts_y.p, op->rec_x.p, op->rec_y.p, y, pp, op->TB.p, op->TL.p, op->TC.p);                 \
  else if (spread_mma())                                                                                         \
    k2f_spread_mma<PP, false><<<grid, 32 * F_MWARPS, FSpreadM<PP>::bytes(), st>>>(                              \
        P, op->ch_tile.p, op->ch_s0.p, op->ch_s1.p, op->ch_count.p, op->ch_rows.p, op->cap, op->base_x.p, op->base_y.p,          \
        op->wts_x.p, op->wts_y.p, op->rec_x.p, op->rec_y.p, y, pp, op->TB.p, op->TL.p, op->TC.p);                 \
  else                                                                                                           \
    k2f_spread<PP><<<grid, 32 * F_WARPS, FSpread<PP>::bytes(), st>>>(                                          \
        P, op->ch_tile.p, op->ch_s0.p, op->ch_s1.p, op->ch_count.p, op->cap, op->base_x.p, op->base_y.p,          \
        op->wts_x.p, op->wts_y.p, op->rec_x.p, op->rec_y.p, y, pp, op->TB.p, op->TL.p, op->TC.p)
        switch (op->p) {
          case 1: GS_F_SPREAD(1); break;
          case 2: GS_F_SPREAD(2); break;
          case 3: GS_F_SPREAD(3); break;
          default: GS_F_SPREAD(4); break;
        }
#undef GS_F_SPREAD
        pmark("k2f_spread", st);
      } else {
        const size_t per_warp = (size_t)P.R * P.R + (P.edges ? 2 * 2 * P.p * P.R : 0);
        k2_spread<<<dim3(ntiles, B), 32 * K2_WARPS, per_warp * K2_WARPS * sizeof(cplx), st>>>(
            P, op->bins.p, op->base_x.p, op->base_y.p, op->wts_x.p, op->wts_y.p, op->rec_x.p, op->rec_y.p, y,
            perm_io ? op->perm.p : nullptr, op->TB.p, op->TL.p, op->TC.p);
        pmark("k2_spread", st);
      }
      if (op->fast2d && fold_src())
        k2_fold_src<<<dim3(P.nt * P.nt, B), (P.T * P.T + 31) / 32 * 32, 0, st>>>(P, op->TB.p, op->fs_start.p,
                                                                               op->fsrc.p, op->cap, op->G.p);
      else
        k2_fold_tiles<<<dim3(P.nt * P.nt, B), (P.T * P.T + 31) / 32 * 32, 0, st>>>(P, op->TB.p, op->tcs.p, op->cap,
                                                                                  op->cov.p, op->covn.p, op->G.p);
      pmark("k2_fold_tiles", st);
      if (op->logLmax == P.log_nov && cols_fft8())
        k2_cols_fft8<false><<<dim3(P.n_ov / P.CW, B), F_COLS_THREADS,
                               ((size_t)P.CW * (fpad_len(P.n_ov) + 1) + P.n_ov / (F_COLS_QW ? 4 : 2)) * sizeof(cplx), st>>>(P, op->G.p,
                                                                                                         op->tw.p);
      else
        k2_cols_ifft<<<dim3(P.n_ov / P.CW, B), 256, (size_t)P.CW * (fpad_len(P.n_ov) + 1) * sizeof(cplx), st>>>(
          P, op->G.p, op->tw.p, op->logLmax);
      pmark("k2_cols_ifft", st);
      if (op->logLmax == P.log_nov && rows_fft8())
        k2_rows_fft8<false><<<dim3((P.n + P.RW - 1) / P.RW, B), 256,
                               ((size_t)P.RW * (rpad_len(P.n_ov) + 1) + P.n_ov / 2) * sizeof(cplx), st>>>(
            P, op->G.p, op->deconv.p, z, op->tw.p);
      else
        k2_rows_ifft_crop<<<dim3((P.n + P.RW - 1) / P.RW, B), 256, (size_t)P.RW * (fpad_len(P.n_ov) + 1) * sizeof(cplx), st>>>(P, op->G.p, op->deconv.p, z, op->tw.p,
                                                                          op->logLmax);
      pmark("k2_rows_ifft_crop", st);
      if (P.edges) {
        const int per = P.nt * 2 * P.p * P.R;
        k2_fold_lines<<<dim3(nblk(per, 32), 2, B), 32 * K2_FL_SPLIT, 0, st>>>(P, op->TL.p, op->tcs.p, op->cap, op->TLF.p);
        pmark("k2_fold_lines", st);
        const int ngroups = (op->cap + K2_CGROUP - 1) / K2_CGROUP;
        k2_fold_corners<<<dim3(nblk(ngroups * 4 * P.p * P.p, 128), B), 128, 0, st>>>(
            P, op->TC.p, op->ch_count.p, op->cap, ngroups, op->TCF.p);
        pmark("k2_fold_corners", st);
        k2_edges<<<dim3(4 * P.p + 1, B), 256, std::max(n1_fft_smem(P), (size_t)256 * sizeof(cplx)), st>>>(
            P, op->TLF.p, op->TCF.p, op->tcs.p, op->ch_count.p, op->cap, op->deconv.p, z, op->tw.p, op->logLmax);
        pmark("k2_edges", st);
      }
      break;
    }
  }
  CKL();
  return fused_sstep;
}

// ------------------------------------------------------------------ dyadic evaluation
#include "dyadic_host.cuh"

// ------------------------------------------------------------------ NCCL (sample-sharded CGLS)
// libnccl.so.2 is opened on first use (the copy torch already loaded when there
// is one), so the library itself loads on hosts without NCCL.
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
    a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
    a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
    a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
    a.errorString = (decltype(a.errorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.commDestroy && a.errorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks the expected symbols";
    return a;
  }();
  if (!api.ok) fail(GS_ERR_CUDA, api.err);
  return api;
}
#define NCK(call)                                                                                        \
  do {                                                                                                   \
    ncclResult_t r_ = (call);                                                                            \
    if (r_ != ncclSuccess) fail(GS_ERR_CUDA, std::string(#call) + ": " + nccl().errorString(r_));        \
  } while (0)

}  // namespace

struct gs_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  ~gs_comm() {
    if (comm) nccl().commDestroy(comm);
  }
};

namespace {

// in-place sum over the ranks of a sharded session (doubles; complex = 2 doubles)
void comm_sum(gs_comm* c, double* v, size_t n, cudaStream_t st) {
  if (!c || c->nranks == 1) return;  // one rank: the sum is the vector itself
  NCK(nccl().allReduce(v, v, n, ncclFloat64, ncclSum, c->comm, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// ------------------------------------------------------------------ CGLS
struct Session {
  gs_op* op = nullptr;
  gs_comm* comm = nullptr;  // sample-sharded solve: T* r and ||q||^2 summed over the ranks
  int B = 1;
  int64_t M = 0, Nc = 0;
  double tol = 1e-10;
  int hist_cap = 0;
  int it = 0;
  DBuf<cplx> b, r, q, x, p, s;
  DBuf<CgState> st;
  DBuf<double> n2, part, hist;
  DBuf<double> vpart;  // tensor route: per-vector norm partials of T / T* outputs
  DBuf<int> flag;
  int chunks_M = 1, chunks_N = 1;
  // one CGLS iteration captured as a CUDA graph (replayed on a private stream
  // that is event-chained to the caller's stream); rebuilt if a buffer moved
  cudaStream_t gst = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  long long graph_kernels = 0;
  std::vector<const void*> graph_sig;
  Session() = default;
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
  ~Session() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (gst) cudaStreamDestroy(gst);
  }
};

void norm2(Session& S, const cplx* v, int64_t len, int chunks, cudaStream_t st) {
  if (chunks <= 1) {
    k_norm2<<<S.B, 1024, 0, st>>>(v, len, S.n2.p); pmark("k_norm2", st);
  } else {
    k_norm2_part<<<dim3(chunks, S.B), 512, 0, st>>>(v, len, chunks, S.part.p); pmark("k_norm2_part", st);
    k_norm2_fold<<<nblk(S.B, 128), 128, 0, st>>>(S.part.p, chunks, S.B, S.n2.p); pmark("k_norm2_fold", st);
  }
  CKL();
}

// ||v||^2 per problem followed by the alpha (q) or beta (s) step of the iteration
void norm2_step(Session& S, const cplx* v, int64_t len, int chunks, cudaStream_t st, bool alpha) {
  if (chunks <= 1) {
    norm2(S, v, len, chunks, st);
    if (alpha) k_cg_alpha<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, S.B);
    else k_cg_beta<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, S.tol, S.hist.p, S.hist_cap, S.B);
    pmark(alpha ? "k_cg_alpha" : "k_cg_beta", st);
  } else {
    k_norm2_part<<<dim3(chunks, S.B), 512, 0, st>>>(v, len, chunks, S.part.p);
    pmark("k_norm2_part", st);
    if (alpha) k_norm2_fold_alpha<<<nblk(S.B, 128), 128, 0, st>>>(S.part.p, chunks, S.B, S.st.p);
    else
      k_norm2_fold_beta<<<nblk(S.B, 128), 128, 0, st>>>(S.part.p, chunks, S.B, S.st.p, S.tol, S.hist.p, S.hist_cap);
    pmark(alpha ? "k_norm2_fold_alpha" : "k_norm2_fold_beta", st);
  }
  CKL();
}

int pick_chunks(int B, int64_t len) {
  int c = (int)std::max<int64_t>(1, std::min<int64_t>(64, (296 + B - 1) / B));
  c = (int)std::min<int64_t>(c, std::max<int64_t>(1, len / 4096));
  return c;
}

void session_begin(Session& S, gs_op* op, const cplx* b_raw, bool b_perm, const cplx* x0, double tol, int hist_cap,
                   cudaStream_t st) {
  S.op = op;
  S.B = op->B;
  S.M = op->M;
  S.Nc = op->Nc;
  S.tol = tol;
  S.hist_cap = hist_cap;
  S.it = 0;
  const int64_t TM = S.M * S.B, TN = S.Nc * S.B;
  S.b.alloc(TM);
  S.r.alloc(TM);
  S.q.alloc(TM);
  S.x.alloc(TN);
  S.p.alloc(TN);
  S.s.alloc(TN);
  S.st.alloc(S.B);
  S.n2.alloc(S.B);
  S.chunks_M = pick_chunks(S.B, S.M);
  S.chunks_N = pick_chunks(S.B, S.Nc);
  S.part.alloc((size_t)S.B * std::max(S.chunks_M, S.chunks_N));
  if (op->route == GS_ROUTE_TENSOR_2D) S.vpart.alloc((size_t)S.B * std::max<int64_t>(op->Ma, op->n));
  if (op->route == GS_ROUTE_NFFT_1D) S.vpart.alloc((size_t)S.B * ((S.M + 127) / 128));  // interpolation CTAs
  S.hist.alloc((size_t)S.B * hist_cap);
  S.flag.alloc(1);
  const bool sorted = !op->general && (op->route == GS_ROUTE_NFFT_1D || op->route == GS_ROUTE_NFFT_2D);
  // b = sqrt(mu) o b_raw in internal order (solver.cpp:30-33); the tensor route
  // applies sqrt(mu) inside T, so it takes the raw data scaled here as well.
  k_gather_scale<<<nblk(TM, 256), 256, 0, st>>>(b_raw, (sorted && b_perm) ? op->perm.p : nullptr,
                                                op->weighted ? op->sqrtw.p : nullptr, S.M, S.B, S.b.p);
  CKL();
  // ref = ||T* b||   (solver.cpp:42); sharded: T* b = sum over ranks of T_g* b_g
  adjoint_dev(op, S.b.p, S.s.p, false, st);
  comm_sum(S.comm, reinterpret_cast<double*>(S.s.p), 2 * (size_t)TN, st);
  norm2(S, S.s.p, S.Nc, S.chunks_N, st);
  k_cg_ref<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, S.B);
  // x = x0 or 0; r = b - T x; s = T* r; gamma; p = s   (solver.cpp:35-68)
  if (x0) CK(cudaMemcpyAsync(S.x.p, x0, TN * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
  else CK(cudaMemsetAsync(S.x.p, 0, TN * sizeof(cplx), st));
  forward_dev(op, S.x.p, S.q.p, false, st);
  k_sub<<<nblk(TM, 256), 256, 0, st>>>(S.b.p, S.q.p, TM, S.r.p);
  adjoint_dev(op, S.r.p, S.s.p, false, st);
  comm_sum(S.comm, reinterpret_cast<double*>(S.s.p), 2 * (size_t)TN, st);
  norm2(S, S.s.p, S.Nc, S.chunks_N, st);
  k_cg_gamma0<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, tol, S.hist.p, hist_cap, S.B);
  CK(cudaMemcpyAsync(S.p.p, S.s.p, TN * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
  CKL();
}

// one CGLS iteration for every still-active problem (solver.cpp:70-88)
bool cg_fused_enabled() {  // GS_B200_CG_FUSED=0: the generic multi-kernel iteration (A/B)
  static const bool on = [] {
    const char* e = std::getenv("GS_B200_CG_FUSED");
    return !(e && *e == '0');
  }();
  return on;
}

void session_iterate_body(Session& S, cudaStream_t st) {
  gs_op* op = S.op;
  const int64_t TM = S.M * S.B, TN = S.Nc * S.B;
  if (S.comm) {
    // sample-sharded iteration: rows local, x / p / s replicated;
    // two exchanges per iteration, both on the device stream (no host sync)
    forward_dev(op, S.p.p, S.q.p, false, st);                            // q_g = T_g p
    norm2(S, S.q.p, S.M, S.chunks_M, st);                                // ||q_g||^2
    comm_sum(S.comm, S.n2.p, (size_t)S.B, st);                           // qq = sum_g ||q_g||^2
    k_cg_alpha<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, S.B);    // alpha (or stop)
    pmark("k_cg_alpha", st);
    k_axpy_alpha<<<nblk(TN, 256), 256, 0, st>>>(S.x.p, S.p.p, S.Nc, S.B, S.st.p, 1.0);   // x += alpha p
    pmark("k_axpy_x", st);
    k_axpy_alpha<<<nblk(TM, 256), 256, 0, st>>>(S.r.p, S.q.p, S.M, S.B, S.st.p, -1.0);   // r_g -= alpha q_g
    pmark("k_axpy_r", st);
    adjoint_dev(op, S.r.p, S.s.p, false, st);                            // T_g* r_g
    comm_sum(S.comm, reinterpret_cast<double*>(S.s.p), 2 * (size_t)TN, st);  // s = sum_g T_g* r_g
    norm2(S, S.s.p, S.Nc, S.chunks_N, st);
    k_cg_beta<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, S.tol, S.hist.p, S.hist_cap, S.B);
    pmark("k_cg_beta", st);
    k_pupdate<<<nblk(TN, 256), 256, 0, st>>>(S.p.p, S.s.p, S.Nc, S.B, S.st.p);  // p = s + beta p
    pmark("k_pupdate", st);
    CKL();
    return;
  }
  if (op->route == GS_ROUTE_UNIFORM_1D && !op->general && cg_fused_enabled()) {  // whole iteration in one launch
    const UniP& P = op->up;
    const size_t rs = uni_cg_resident_smem(P, op->Rr);
    k_uni_cgls_iter<<<S.B, UNI_CG_THREADS, rs ? rs : uni_smem_tw(P), st>>>(
        P, op->rec_u.p, op->M * op->Rr, S.x.p, S.p.p, S.s.p, S.r.p, S.q.p, S.st.p, S.tol, S.hist.p, S.hist_cap,
        op->tw.p, op->logLmax, 1, rs != 0);
    pmark("k_uni_cgls_iter", st);
    CKL();
    return;
  }
  if (op->route == GS_ROUTE_NFFT_1D && !op->general && cg_fused_enabled()) {
    // 4 launches: embed+FFT, interpolation (+ deferred r update, ||q||^2 partials),
    // spreading (+ q-step), inverse FFT (+ s-step)
    const N1QStep q1{S.vpart.p, (int)((S.M + 127) / 128), S.q.p, S.r.p, S.st.p, S.x.p, S.p.p};
    forward_dev(op, S.p.p, S.q.p, false, st, nullptr, &q1);
    const SStep ss{S.st.p, S.p.p, S.tol, S.hist.p, S.hist_cap};
    adjoint_dev(op, S.r.p, S.s.p, false, st, &ss, nullptr, &q1);
    CKL();
    return;
  }
  if (S.chunks_M == 1 && S.chunks_N == 1 && cg_fused_enabled()) {
    // one CTA reduces each problem's vectors: the scalar / vector phases in 2 launches
    forward_dev(op, S.p.p, S.q.p, false, st);                                                  // q = T p
    k_cg_qstep<<<S.B, CG_STEP_THREADS, 0, st>>>(S.st.p, S.q.p, S.r.p, S.x.p, S.p.p, S.M, S.Nc);  // qq, alpha, x, r
    pmark("k_cg_qstep", st);
    const SStep ss{S.st.p, S.p.p, S.tol, S.hist.p, S.hist_cap};
    if (!adjoint_dev(op, S.r.p, S.s.p, false, st, &ss)) {                                      // s = T* r
      k_cg_sstep<<<S.B, CG_STEP_THREADS, 0, st>>>(S.st.p, S.s.p, S.p.p, S.Nc, S.tol, S.hist.p, S.hist_cap);
      pmark("k_cg_sstep", st);                                                                 // gamma', beta, p
    }
    CKL();
    return;
  }
  if (op->route == GS_ROUTE_TENSOR_2D && cg_fused_enabled()) {
    // the last pass of T / T* writes per-vector norm partials: 4 launches around the 4 passes
    // and the axpys ride on the passes that own the vectors: the x-pass of T
    // forms p = s + beta p (deferred from the previous iteration), the y-pass of
    // T* forms r -= alpha q, the x-pass of T* x += alpha p: 6 launches
    const int Ma = (int)op->Ma, n = (int)op->n, Mb = (int)op->Mb;
    const UniPre pre_p{S.st.p, 1, S.p.p, S.s.p, (int64_t)n * n, n, 1, n};
    const UniPre pre_r{S.st.p, 2, S.r.p, S.q.p, S.M, Mb, 1, Mb};
    const UniPre pre_x{S.st.p, 3, S.x.p, S.p.p, (int64_t)n * n, n, 1, n};
    forward_dev(op, S.p.p, S.q.p, false, st, S.vpart.p, nullptr, &pre_p);  // q = T p (+ ||q||^2 partials)
    k_fold_alpha_w<<<S.B, 32, 0, st>>>(S.vpart.p, Ma, S.st.p);
    pmark("k_fold_alpha_w", st);
    adjoint_dev(op, S.r.p, S.s.p, false, st, nullptr, S.vpart.p, nullptr, &pre_r, &pre_x);  // s = T* r
    k_fold_beta_w<<<S.B, 32, 0, st>>>(S.vpart.p, n, S.st.p, S.tol, S.hist.p, S.hist_cap);
    pmark("k_fold_beta_w", st);
    CKL();
    return;
  }
  if (cg_fused_enabled()) {  // 6 launches around T / T*: folds fused with alpha / beta, one axpy launch
    forward_dev(op, S.p.p, S.q.p, false, st);  // q = T p
    norm2_step(S, S.q.p, S.M, S.chunks_M, st, true);  // qq, alpha (or stop)
    k_axpy_xr<<<nblk(TN + TM, 256), 256, 0, st>>>(S.x.p, S.p.p, S.Nc, S.r.p, S.q.p, S.M, S.B, S.st.p);
    pmark("k_axpy_xr", st);  // x += alpha p, r -= alpha q
    adjoint_dev(op, S.r.p, S.s.p, false, st);  // s = T* r
    norm2_step(S, S.s.p, S.Nc, S.chunks_N, st, false);  // gamma', beta
    k_pupdate<<<nblk(TN, 256), 256, 0, st>>>(S.p.p, S.s.p, S.Nc, S.B, S.st.p);  // p = s + beta p
    pmark("k_pupdate", st);
    CKL();
    return;
  }
  forward_dev(op, S.p.p, S.q.p, false, st);                          // q = T p
  norm2(S, S.q.p, S.M, S.chunks_M, st);                              // qq
  k_cg_alpha<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, S.B);  // alpha (or stop)
  pmark("k_cg_alpha", st);
  k_axpy_alpha<<<nblk(TN, 256), 256, 0, st>>>(S.x.p, S.p.p, S.Nc, S.B, S.st.p, 1.0);  // x += alpha p
  pmark("k_axpy_x", st);
  k_axpy_alpha<<<nblk(TM, 256), 256, 0, st>>>(S.r.p, S.q.p, S.M, S.B, S.st.p, -1.0);  // r -= alpha q
  pmark("k_axpy_r", st);
  adjoint_dev(op, S.r.p, S.s.p, false, st);                          // s = T* r
  norm2(S, S.s.p, S.Nc, S.chunks_N, st);                             // gamma'
  k_cg_beta<<<nblk(S.B, 128), 128, 0, st>>>(S.st.p, S.n2.p, S.tol, S.hist.p, S.hist_cap, S.B);
  pmark("k_cg_beta", st);
  k_pupdate<<<nblk(TN, 256), 256, 0, st>>>(S.p.p, S.s.p, S.Nc, S.B, S.st.p);  // p = s + beta p
  pmark("k_pupdate", st);
  CKL();
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GS_B200_NO_GRAPHS");
    return !(e && *e && *e != '0');
  }();
  return on;
}

// k iterations of solver.cpp:70-88 for every active problem, no host sync
void session_iterate(Session& S, cudaStream_t st, int k) {
  if (k <= 0) return;
  S.it += k;
  if (S.op->route == GS_ROUTE_UNIFORM_1D && !S.op->general && !S.comm && cg_fused_enabled() && !g_prof.on) {
    // all k iterations in one launch (k_uni_cgls_iter loops on the device)
    const UniP& P = S.op->up;
    const size_t rs = uni_cg_resident_smem(P, S.op->Rr);
    k_uni_cgls_iter<<<S.B, UNI_CG_THREADS, rs ? rs : uni_smem_tw(P), st>>>(
        P, S.op->rec_u.p, S.op->M * S.op->Rr, S.x.p, S.p.p, S.s.p, S.r.p, S.q.p, S.st.p, S.tol, S.hist.p,
        S.hist_cap, S.op->tw.p, S.op->logLmax, k, rs != 0);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    return;
  }
  if (!graphs_enabled() || g_prof.on || S.comm) {
    for (int i = 0; i < k; ++i) session_iterate_body(S, st);
    return;
  }
  uint64_t tol_bits = 0;
  std::memcpy(&tol_bits, &S.tol, sizeof(tol_bits));
  const std::vector<const void*> sig = {S.p.p, S.q.p, S.r.p, S.s.p, S.x.p, S.st.p, S.n2.p, S.hist.p, S.part.p, S.vpart.p,
                                        reinterpret_cast<const void*>((intptr_t)S.hist_cap),
                                        reinterpret_cast<const void*>((uintptr_t)tol_bits)};
  if (S.gexec && (sig != S.graph_sig)) {
    cudaGraphExecDestroy(S.gexec);
    S.gexec = nullptr;
  }
  if (!S.gst) {
    CK(cudaStreamCreateWithFlags(&S.gst, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&S.ev_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.ev_out, cudaEventDisableTiming));
  }
  if (!S.gexec) {
    cudaGraph_t g = nullptr;
    const long long n0 = g_launches.load();
    CK(cudaStreamBeginCapture(S.gst, cudaStreamCaptureModeThreadLocal));
    session_iterate_body(S, S.gst);
    CK(cudaStreamEndCapture(S.gst, &g));
    S.graph_kernels = g_launches.load() - n0;
    g_launches.fetch_sub(S.graph_kernels);  // counted when replayed
    CK(cudaGraphInstantiate(&S.gexec, g, 0));
    CK(cudaGraphDestroy(g));
    S.graph_sig = sig;
  }
  CK(cudaEventRecord(S.ev_in, st));
  CK(cudaStreamWaitEvent(S.gst, S.ev_in, 0));
  for (int i = 0; i < k; ++i) CK(cudaGraphLaunch(S.gexec, S.gst));
  g_launches.fetch_add(S.graph_kernels * k);
  CK(cudaEventRecord(S.ev_out, S.gst));
  CK(cudaStreamWaitEvent(st, S.ev_out, 0));
}

bool session_any_active(Session& S, cudaStream_t st) {
  k_any_active<<<1, 256, 0, st>>>(S.st.p, S.B, S.flag.p);
  int h = 0;
  CK(cudaMemcpyAsync(&h, S.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h != 0;
}

}  // namespace

// ====================================================================== C-ABI
struct gs_cgls_session {
  Session s;
};

extern "C" {

const char* gs_last_error(void) { return g_err.c_str(); }
long long gs_launch_count(void) { return g_launches.load(); }
int gs_build_arch(void) { return 100; }

int gs_op_create(const gs_op_desc* desc, gs_op** out) {
  return guard_call([&] {
    if (!out) fail(GS_ERR_USAGE, "null output handle");
    *out = create(desc);
  });
}

int gs_op_destroy(gs_op* op) {
  if (!op) return GS_OK;
  cudaSetDevice(op->device);
  cudaDeviceSynchronize();
  gs_cgls_destroy(op->solve_cache);
  delete op;
  return GS_OK;
}

int gs_op_info(const gs_op* op, gs_op_info_t* info) {
  if (!op || !info) {
    g_err = "null argument";
    return GS_ERR_USAGE;
  }
  info->dim = op->dim;
  info->family_p = op->p;
  info->J = op->J;
  info->batch = op->B;
  info->route = op->route;
  info->rows = op->M;
  info->cols = op->Nc;
  info->uniform_fast = op->route == GS_ROUTE_UNIFORM_1D;
  info->uniform_epsilon = op->uniform_eps;
  info->weighted = op->weighted;
  info->n_over = (op->route == GS_ROUTE_NFFT_1D || op->route == GS_ROUTE_NFFT_2D) ? op->np.n_ov : 0;
  info->device_bytes = (int64_t)op->device_bytes();
  return GS_OK;
}

static void apply_common(gs_op* op, const double* in, int64_t in_len, int64_t want_in, double* out, int64_t out_len,
                         void* stream, bool fwd) {
  if (!op || !in || !out) fail(GS_ERR_USAGE, "null argument");
  if (in_len != want_in)
    fail(GS_ERR_SHAPE, fwd ? "coefficient vector length mismatch" : "sample vector length mismatch");
  std::lock_guard<std::mutex> lk(op->mu);
  CK(cudaSetDevice(op->device));
  cudaStream_t st = (cudaStream_t)stream;
  const bool din = is_device_ptr(in), dout = is_device_ptr(out);
  const cplx* src = (const cplx*)in;
  cplx* dst = (cplx*)out;
  if (!din) {
    op->stage_a.alloc(in_len);
    CK(cudaMemcpyAsync(op->stage_a.p, in, in_len * sizeof(cplx), cudaMemcpyHostToDevice, st));
    src = op->stage_a.p;
  }
  if (!dout) {
    op->stage_b.alloc(out_len);
    dst = op->stage_b.p;
  }
  if (fwd) forward_dev(op, src, dst, true, st);
  else adjoint_dev(op, src, dst, true, st);
  if (!dout) {
    CK(cudaMemcpyAsync(out, dst, out_len * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } else if (!din) {
    CK(cudaStreamSynchronize(st));  // staging buffer reuse
  }
}

int gs_apply_forward(gs_op* op, const double* coeffs, int64_t coeffs_len, double* samples, void* stream) {
  return guard_call([&] {
    if (!op) fail(GS_ERR_USAGE, "null handle");
    apply_common(op, coeffs, coeffs_len, op->Nc * op->B, samples, op->M * op->B, stream, true);
  });
}

int gs_apply_adjoint(gs_op* op, const double* samples, int64_t samples_len, double* coeffs, void* stream) {
  return guard_call([&] {
    if (!op) fail(GS_ERR_USAGE, "null handle");
    apply_common(op, samples, samples_len, op->M * op->B, coeffs, op->Nc * op->B, stream, false);
  });
}

// ---- CGLS sessions: begin (preamble), step (n iterations, no host sync), finish
namespace {
// preamble of a solve into a new session, or into `reuse` (a session of this
// op whose device buffers are recycled; consumed either way)
int cgls_begin_into(gs_op* op, gs_cgls_session* reuse, const double* raw_samples, int64_t samples_len,
                    const double* x0, double tolerance, int history_capacity, void* stream, gs_cgls_session** out,
                    gs_comm* comm = nullptr) {
  std::unique_ptr<gs_cgls_session> R(reuse);
  return guard_call([&] {
    if (!op || !raw_samples || !out) fail(GS_ERR_USAGE, "null argument");
    *out = nullptr;
    if (samples_len != op->M * op->B) fail(GS_ERR_SHAPE, "sample vector length mismatch");
    if (!(tolerance > 0)) fail(GS_ERR_DOMAIN, "tolerance must be positive");
    std::lock_guard<std::mutex> lk(op->mu);
    CK(cudaSetDevice(op->device));
    cudaStream_t st = (cudaStream_t)stream;
    std::unique_ptr<gs_cgls_session> S((R && R->s.op == op) ? R.release() : new gs_cgls_session);
    const int64_t TM = op->M * op->B, TN = op->Nc * op->B;
    const cplx* b = (const cplx*)raw_samples;
    if (!is_device_ptr(raw_samples)) {
      op->stage_a.upload((const cplx*)raw_samples, TM, st);
      b = op->stage_a.p;
    }
    const cplx* xx = (const cplx*)x0;
    if (x0 && !is_device_ptr(x0)) {
      op->stage_b.upload((const cplx*)x0, TN, st);
      xx = op->stage_b.p;
    }
    S->s.comm = comm;
    if (comm && comm->device != op->device) fail(GS_ERR_USAGE, "communicator and operator are on different devices");
    session_begin(S->s, op, b, true, xx, tolerance, std::max(1, history_capacity), st);
    *out = S.release();
  });
}
}  // namespace

int gs_cgls_begin(gs_op* op, const double* raw_samples, int64_t samples_len, const double* x0, double tolerance,
                  int history_capacity, void* stream, gs_cgls_session** out) {
  return cgls_begin_into(op, nullptr, raw_samples, samples_len, x0, tolerance, history_capacity, stream, out);
}

int gs_cgls_step(gs_cgls_session* s, int iterations, void* stream) {
  return guard_call([&] {
    if (!s) fail(GS_ERR_USAGE, "null session");
    std::lock_guard<std::mutex> lk(s->s.op->mu);
    CK(cudaSetDevice(s->s.op->device));
    session_iterate(s->s, (cudaStream_t)stream, iterations);
  });
}

int gs_cgls_active(gs_cgls_session* s, void* stream, int* any_active) {
  return guard_call([&] {
    if (!s || !any_active) fail(GS_ERR_USAGE, "null argument");
    std::lock_guard<std::mutex> lk(s->s.op->mu);
    *any_active = session_any_active(s->s, (cudaStream_t)stream) ? 1 : 0;
  });
}

int gs_cgls_finish(gs_cgls_session* s, double* x_out, gs_solve_stats* stats, double* history, void* stream) {
  return guard_call([&] {
    if (!s) fail(GS_ERR_USAGE, "null session");
    Session& S = s->s;
    std::lock_guard<std::mutex> lk(S.op->mu);
    CK(cudaSetDevice(S.op->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t TN = S.Nc * S.B;
    k_zero_if_ref0<<<nblk(TN, 256), 256, 0, st>>>(S.x.p, S.Nc, S.B, S.st.p);
    CKL();
    if (x_out) CK(cudaMemcpyAsync(x_out, S.x.p, TN * sizeof(cplx), cudaMemcpyDefault, st));
    std::vector<CgState> hs(S.B);
    CK(cudaMemcpyAsync(hs.data(), S.st.p, S.B * sizeof(CgState), cudaMemcpyDeviceToHost, st));
    std::vector<double> hh((size_t)S.B * S.hist_cap);
    CK(cudaMemcpyAsync(hh.data(), S.hist.p, hh.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < S.B; ++b) {
      const CgState& c = hs[b];
      int hl = std::max(1, std::min(c.hist_len, S.hist_cap));
      if (stats) {
        stats[b].iterations = c.iterations;
        stats[b].converged = c.converged;
        stats[b].residual = c.ref == 0.0 ? 0.0 : hh[(size_t)b * S.hist_cap + hl - 1];
      }
      if (history)
        for (int i = 0; i < hl; ++i) history[(size_t)b * S.hist_cap + i] = hh[(size_t)b * S.hist_cap + i];
    }
  });
}

int gs_cgls_destroy(gs_cgls_session* s) {
  delete s;
  return GS_OK;
}

int gs_solve_least_squares(gs_op* op, const double* raw_samples, int64_t samples_len, const double* x0,
                           int max_iterations, double tolerance, double* x_out, gs_solve_stats* stats,
                           double* history, void* stream) {
  if (!op) {
    g_err = "null handle";
    return GS_ERR_USAGE;
  }
  // the op keeps its last solve workspace, so repeated solves allocate nothing
  gs_cgls_session* cached = nullptr;
  {
    std::lock_guard<std::mutex> lk(op->mu);
    cached = std::exchange(op->solve_cache, nullptr);
  }
  const int max_iter = max_iterations > 0 ? max_iterations : (int)std::min<int64_t>(INT32_MAX / 2, 2 * op->Nc);
  gs_cgls_session* s = nullptr;
  int rc = cgls_begin_into(op, cached, raw_samples, samples_len, x0, tolerance, max_iter + 1, stream, &s);
  if (rc) return rc;
  int done = 0;
  int active = 1;
  rc = gs_cgls_active(s, stream, &active);
  int chunk = 4;
  while (rc == 0 && active && done < max_iter) {
    int k = std::min(chunk, max_iter - done);
    rc = gs_cgls_step(s, k, stream);
    done += k;
    if (rc == 0) rc = gs_cgls_active(s, stream, &active);
    chunk = std::min(chunk * 2, 64);
  }
  if (rc == 0) rc = gs_cgls_finish(s, x_out, stats, history, stream);
  {
    std::lock_guard<std::mutex> lk(op->mu);
    std::swap(op->solve_cache, s);
  }
  gs_cgls_destroy(s);  // another thread's session parked meanwhile, if any
  return rc;
}

// ---------------------------------------------------------------- sample-sharded CGLS
int gs_comm_unique_id(unsigned char* id) {
  return guard_call([&] {
    if (!id) fail(GS_ERR_USAGE, "null argument");
    ncclUniqueId u;
    NCK(nccl().getUniqueId(&u));
    static_assert(sizeof(u.internal) == GS_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, u.internal, sizeof(u.internal));
  });
}

int gs_comm_init(int nranks, int rank, const unsigned char* id, int device, gs_comm** out) {
  return guard_call([&] {
    if (!id || !out) fail(GS_ERR_USAGE, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(GS_ERR_USAGE, "bad rank / size");
    *out = nullptr;
    CK(cudaSetDevice(device));
    std::unique_ptr<gs_comm> c(new gs_comm);
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    NCK(nccl().commInitRank(&c->comm, nranks, u, rank));
    *out = c.release();
  });
}

int gs_comm_destroy(gs_comm* c) {
  delete c;
  return GS_OK;
}

int gs_cgls_begin_sharded(gs_op* op, gs_comm* comm, const double* raw_samples, int64_t samples_len, const double* x0,
                          double tolerance, int history_capacity, void* stream, gs_cgls_session** out) {
  if (!comm) {
    g_err = "null communicator";
    return GS_ERR_USAGE;
  }
  return cgls_begin_into(op, nullptr, raw_samples, samples_len, x0, tolerance, history_capacity, stream, out, comm);
}

int gs_solve_least_squares_sharded(gs_op* op, gs_comm* comm, const double* raw_samples, int64_t samples_len,
                                   const double* x0, int max_iterations, double tolerance, double* x_out,
                                   gs_solve_stats* stats, double* history, void* stream) {
  if (!op || !comm) {
    g_err = "null handle";
    return GS_ERR_USAGE;
  }
  const int max_iter = max_iterations > 0 ? max_iterations : (int)std::min<int64_t>(INT32_MAX / 2, 2 * op->Nc);
  gs_cgls_session* s = nullptr;
  int rc = gs_cgls_begin_sharded(op, comm, raw_samples, samples_len, x0, tolerance, max_iter + 1, stream, &s);
  if (rc) return rc;
  // every rank holds the same (all-reduced) scalars, so the ranks step in lockstep
  int done = 0, active = 1, chunk = 4;
  rc = gs_cgls_active(s, stream, &active);
  while (rc == 0 && active && done < max_iter) {
    const int k = std::min(chunk, max_iter - done);
    rc = gs_cgls_step(s, k, stream);
    done += k;
    if (rc == 0) rc = gs_cgls_active(s, stream, &active);
    chunk = std::min(chunk * 2, 64);
  }
  if (rc == 0) rc = gs_cgls_finish(s, x_out, stats, history, stream);
  gs_cgls_destroy(s);
  return rc;
}

int gs_profile_pair(gs_op* op, int reps, void* stream, int max_kernels, double* ms_out, char* names_out,
                    int* count) {
  return guard_call([&] {
    if (!op || !ms_out || !count || reps <= 0) fail(GS_ERR_USAGE, "bad argument");
    std::lock_guard<std::mutex> lk(op->mu);
    CK(cudaSetDevice(op->device));
    cudaStream_t st = (cudaStream_t)stream;
    DBuf<cplx> x, y, z;
    x.alloc(op->Nc * op->B);
    y.alloc(op->M * op->B);
    z.alloc(op->Nc * op->B);
    // live data, not zeros: x = seeded pseudo-random coefficients, y = T x from the warm-up apply
    k_fill_hash<<<nblk(op->Nc * op->B, 256), 256, 0, st>>>(x.p, op->Nc * op->B, 0x9E3779B97F4A7C15ull);
    CKL();
    forward_dev(op, x.p, y.p, false, st);  // warm
    adjoint_dev(op, y.p, z.p, false, st);
    CK(cudaStreamSynchronize(st));
    std::vector<double> acc;
    std::vector<std::string> names;
    for (int r = 0; r < reps; ++r) {
      g_prof = Prof();
      g_prof.on = true;
      pmark("start", st);
      forward_dev(op, x.p, y.p, false, st);
      adjoint_dev(op, y.p, z.p, false, st);
      CK(cudaStreamSynchronize(st));
      g_prof.on = false;
      const size_t k = g_prof.ev.size() - 1;
      if (acc.empty()) {
        acc.assign(k, 0.0);
        names.assign(g_prof.names.begin() + 1, g_prof.names.end());
      }
      for (size_t i = 0; i < k; ++i) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, g_prof.ev[i], g_prof.ev[i + 1]));
        acc[i] += ms;
      }
      for (auto e : g_prof.ev) cudaEventDestroy(e);
    }
    g_prof = Prof();
    const int k = (int)std::min<size_t>(acc.size(), (size_t)max_kernels);
    for (int i = 0; i < k; ++i) {
      ms_out[i] = acc[i] / reps;
      if (names_out) {
        std::strncpy(names_out + 32 * i, names[i].c_str(), 31);
        names_out[32 * i + 31] = 0;
      }
    }
    *count = k;
  });
}

int gs_op_export_factors(gs_op* op, int b, int axis, double* D, double* L, double* R) {
  return guard_call([&] {
    if (!op || !D) fail(GS_ERR_USAGE, "null argument");
    if (b < 0 || b >= op->B) fail(GS_ERR_USAGE, "problem index out of range");
    if (axis < 0 || axis >= op->dim) fail(GS_ERR_USAGE, "axis out of range");
    std::lock_guard<std::mutex> lk(op->mu);
    CK(cudaSetDevice(op->device));
    const int64_t M = op->M;
    const int Rr = op->Rr, p = op->p;
    std::vector<cplx> recs(M * Rr);  // per point in the caller's order
    if (op->route == GS_ROUTE_UNIFORM_1D || op->route == GS_ROUTE_NDFT_1D || op->general) {  // caller order already
      const cplx* src = op->route == GS_ROUTE_UNIFORM_1D ? op->rec_u.p : (axis == 0 ? op->rec_x.p : op->rec_y.p);
      CK(cudaMemcpy(recs.data(), src + b * M * Rr, M * Rr * sizeof(cplx), cudaMemcpyDeviceToHost));
    } else if (op->route == GS_ROUTE_TENSOR_2D) {
      const int64_t Ma = op->Ma, Mb = op->Mb;
      const int64_t Ml = axis == 0 ? Ma : Mb;
      std::vector<cplx> ax(Ml * Rr);
      CK(cudaMemcpy(ax.data(), (axis == 0 ? op->rec_ax.p + b * Ma * Rr : op->rec_ay.p + b * Mb * Rr),
                    Ml * Rr * sizeof(cplx), cudaMemcpyDeviceToHost));
      std::vector<double> sw;
      if (op->weighted && axis == 0) {
        sw.resize(M);
        CK(cudaMemcpy(sw.data(), op->sqrtw.p + b * M, M * sizeof(double), cudaMemcpyDeviceToHost));
      }
      for (int64_t m = 0; m < M; ++m) {
        const int64_t k = axis == 0 ? m / Mb : m % Mb;
        for (int c = 0; c < Rr; ++c) recs[m * Rr + c] = sw.empty() ? ax[k * Rr + c] : cscale(ax[k * Rr + c], sw[m]);
      }
    } else {
      std::vector<cplx> srt(M * Rr);
      std::vector<int> pm(M);
      CK(cudaMemcpy(srt.data(), (axis == 0 ? op->rec_x.p : op->rec_y.p) + b * M * Rr, M * Rr * sizeof(cplx),
                    cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(pm.data(), op->perm.p + b * M, M * sizeof(int), cudaMemcpyDeviceToHost));
      for (int64_t s = 0; s < M; ++s)
        for (int c = 0; c < Rr; ++c) recs[(int64_t)pm[s] * Rr + c] = srt[s * Rr + c];
    }
    for (int64_t m = 0; m < M; ++m) {
      D[2 * m] = recs[m * Rr].x;
      D[2 * m + 1] = recs[m * Rr].y;
      if (op->edges) {
        for (int c = 0; c < p; ++c) {  // Eigen col-major M x p: (m, c) at c*M + m
          if (L) {
            L[2 * (c * M + m)] = recs[m * Rr + 1 + c].x;
            L[2 * (c * M + m) + 1] = recs[m * Rr + 1 + c].y;
          }
          if (R) {
            R[2 * (c * M + m)] = recs[m * Rr + 1 + p + c].x;
            R[2 * (c * M + m) + 1] = recs[m * Rr + 1 + p + c].y;
          }
        }
      }
    }
  });
}


// ---------------------------------------------------------------- dyadic evaluation (dyadic.hpp)
static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int gs_scaling_dyadic(int family_p, int R, double* values, int64_t* len, int64_t* support_begin, void* stream) {
  return guard_call([&] {
    if (family_p < 1 || family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
    if (!len || !support_begin) fail(GS_ERR_USAGE, "null output");
    if (!values) {  // sizes only
      if (R < 0) fail(GS_ERR_DOMAIN, "resolution must be >= 0");
      *len = ((int64_t)(2 * family_p - 1) << R) + 1;
      *support_begin = -family_p + 1;
      return;
    }
    DyTables T;
    dy_build(T, family_p, R, false, as_stream(stream));
    *len = T.P.len[0];
    *support_begin = T.P.sb[0];
    dy_copy_table(T, 0, values, as_stream(stream));
  });
}

int gs_boundary_dyadic(int family_p, int left, int R, int k, double* values, int64_t* len, int64_t* support_begin,
                       void* stream) {
  return guard_call([&] {
    if (family_p < 1 || family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
    if (family_p < 2) fail(GS_ERR_DOMAIN, "boundary functions require p >= 2");
    if (R < 0) fail(GS_ERR_DOMAIN, "resolution must be >= 0");
    if (k < 0 || k >= family_p) fail(GS_ERR_DOMAIN, "edge function index out of range");
    if (!len || !support_begin) fail(GS_ERR_USAGE, "null output");
    *len = ((int64_t)(family_p + k) << R) + 1;
    *support_begin = left ? 0 : -(family_p + k);
    if (!values) return;
    DyTables T;
    dy_build(T, family_p, R, true, as_stream(stream));
    dy_copy_table(T, left ? 1 + k : 1 + family_p + k, values, as_stream(stream));
  });
}

int gs_weval(int dim, int family_p, int J, int R, const double* coeffs, int64_t coeffs_len, double* out,
             void* stream) {
  return guard_call([&] { dy_weval(dim, family_p, J, R, coeffs, coeffs_len, out, as_stream(stream)); });
}


// ---------------------------------------------------------------- family data / transforms (scaling.hpp, fourier.hpp)
int gs_family_filter(int family_p, double* taps) {
  return guard_call([&] {
    if (family_p < 1 || family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
    if (!taps) fail(GS_ERR_USAGE, "null output");
    const gsdata::FamilyData& src = gsdata::kFamilies[family_p - 1];
    for (int i = 0; i < 2 * family_p; ++i) taps[i] = src.taps[i];
  });
}

int gs_boundary_filter_set(int family_p, int left, double* H, double* h, double* integer_values) {
  return guard_call([&] {
    if (family_p < 1 || family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
    if (family_p < 2) fail(GS_ERR_DOMAIN, "haar has no boundary corrections (p = 1)");
    const gsdata::FamilyData& src = gsdata::kFamilies[family_p - 1];
    const int p = family_p;
    if (H) std::memcpy(H, left ? src.left_H : src.right_H, sizeof(double) * p * p);
    if (h) std::memcpy(h, left ? src.left_h : src.right_h, sizeof(double) * p * (2 * p - 1));
    if (integer_values) std::memcpy(integer_values, left ? src.left_seed : src.right_seed, sizeof(double) * p * 2 * p);
  });
}

int gs_boundary_at_zero(int family_p, int left, double* v) {
  return guard_call([&] {
    if (family_p < 1 || family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
    if (family_p < 2) fail(GS_ERR_DOMAIN, "haar has no boundary corrections (p = 1)");
    if (!v) fail(GS_ERR_USAGE, "null output");
    const FamDev f = make_family(family_p);  // NumericalError if the fixed point is singular
    for (int i = 0; i < family_p; ++i) v[i] = f.vz[left ? 0 : 1][i];
  });
}

namespace {
int eval_call(int family_p, int side, int64_t n, const double* xi, int depth, int terms, double* out, void* stream) {
  return guard_call([&] {
    if (family_p < 1 || family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
    if (side >= 0 && family_p < 2) fail(GS_ERR_DOMAIN, "haar has no boundary corrections (p = 1)");
    if (family_p >= 2 && terms < 1) fail(GS_ERR_DOMAIN, "fourier_scaling: terms must be >= 1");
    if (side >= 0 && depth < 1) fail(GS_ERR_DOMAIN, "fourier_boundary: depth must be >= 1");
    if (n < 0 || (n > 0 && (!xi || !out))) fail(GS_ERR_USAGE, "null argument");
    if (n == 0) return;
    cudaStream_t st = (cudaStream_t)stream;
    const FamDev f = make_family(family_p);
    const int per = side >= 0 ? family_p : 1;
    DBuf<double> dx;
    DBuf<cplx> dout;
    const double* px = xi;
    if (!is_device_ptr(xi)) {
      dx.upload(xi, n, st);
      px = dx.p;
    }
    const bool dev_out = is_device_ptr(out);
    cplx* po = (cplx*)out;
    if (!dev_out) {
      dout.alloc(n * per);
      po = dout.p;
    }
    if (side >= 0) k_eval_boundary<<<nblk(n, 128), 128, 0, st>>>(f, side, px, n, depth, terms, po);
    else k_eval_scaling<<<nblk(n, 128), 128, 0, st>>>(f, px, n, terms, po);
    pmark(side >= 0 ? "k_eval_boundary" : "k_eval_scaling", st);
    CKL();
    if (!dev_out) CK(cudaMemcpyAsync(out, po, n * per * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}
}  // namespace

int gs_fourier_scaling_eval(int family_p, int64_t n, const double* xi, int terms, double* out, void* stream) {
  return eval_call(family_p, -1, n, xi, 1, terms, out, stream);
}

int gs_fourier_boundary_eval(int family_p, int left, int64_t n, const double* xi, int depth, int terms, double* out,
                             void* stream) {
  return eval_call(family_p, left ? 0 : 1, n, xi, depth, terms, out, stream);
}

int gs_densify(int dim, int family_p, int J, int64_t M, const double* coords, const double* sqrt_weights,
               int64_t entry_cap, double* out, void* stream) {
  return guard_call([&] {
    if (dim != 1 && dim != 2) fail(GS_ERR_DOMAIN, "sampling set must be 1D or 2D");
    if (family_p < 1 || family_p > 8) fail(GS_ERR_DOMAIN, "unsupported family");
    if (J < 0 || J > 24) fail(GS_ERR_DOMAIN, "scale J out of range");
    if (M <= 0 || !coords || !out) fail(GS_ERR_USAGE, "null argument");
    const int64_t n = 1LL << J;
    const int64_t cols = dim == 1 ? n : n * n;
    if ((double)M * (double)cols > (double)entry_cap) fail(GS_ERR_DOMAIN, "densify: matrix exceeds the entry cap");
    cudaStream_t st = (cudaStream_t)stream;
    const FamDev f = make_family(family_p);
    DBuf<double> dc, dw;
    dc.upload(coords, M * dim, st);
    if (sqrt_weights) dw.upload(sqrt_weights, M, st);
    DBuf<cplx> rx, ry, dout;
    rx.alloc(M * n);
    k_densify_axis<<<nblk(M, 128), 128, 0, st>>>(f, dc.p, dim, 0, M, J, (int)n, rx.p);
    pmark("k_densify_axis", st);
    if (dim == 2) {
      ry.alloc(M * n);
      k_densify_axis<<<nblk(M, 128), 128, 0, st>>>(f, dc.p, dim, 1, M, J, (int)n, ry.p);
      pmark("k_densify_axis", st);
    }
    dout.alloc(M * cols);
    k_densify_out<<<nblk(M * cols, 256), 256, 0, st>>>(dim, M, (int)n, rx.p, ry.p, sqrt_weights ? dw.p : nullptr,
                                                        dout.p);
    pmark("k_densify_out", st);
    CKL();
    CK(cudaMemcpyAsync(out, dout.p, M * cols * sizeof(cplx), cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
  });
}

int gs_op_balanced_schedule(const gs_op* op) { return op && op->balanced ? 1 : 0; }

#ifdef F_TIMELINE
// debug builds only: copy the CTA timeline of the last fast-path launch (kernels_nfft2d_fast.cuh)
int gs_debug_timeline(unsigned long long* host, int64_t rows) {
  const int64_t n = rows < F_TL_MAX ? rows : F_TL_MAX;
  return cudaMemcpyFromSymbol(host, g_tl, sizeof(unsigned long long) * 5 * n) == cudaSuccess ? 0 : 7;
}
int gs_debug_timeline_clear() {
  static unsigned long long zero[F_TL_MAX][5];
  return cudaMemcpyToSymbol(g_tl, zero, sizeof(zero)) == cudaSuccess ? 0 : 7;
}
#endif
}  // extern "C"
