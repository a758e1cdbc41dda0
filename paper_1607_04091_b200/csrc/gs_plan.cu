// gs_plan.cu -- general-length FFT engine, the device NfftPlan and the
// uniform-grid reduction at any length: the lower-level API of nufft.hpp:41-77
// (NfftPlan / plan_nfft / nfft_forward / nfft_adjoint, uniform_ndft_fft /
// uniform_ndft_adjoint_fft) behind the C-ABI of include/gs_b200.h, and the
// building blocks of the operator's general routes.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "host_math.h"
#include "kernels_fftg.cuh"
#include "kernels_plan.cuh"
#include "plan.h"

namespace gsb {

namespace {
constexpr int FG_CAP = 6144;  // points per CTA (two ping-pong buffers: 192 KB)
constexpr int kSmemMaxFg = 227 * 1024;

void fg_smem_attr() {
  static std::mutex m;
  static std::vector<char> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(m);
  if (dev < (int)done.size() && done[dev]) return;
  CK(cudaFuncSetAttribute(k_fftg_lines, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxFg));
  if ((int)done.size() <= dev) done.resize(dev + 1, 0);
  done[dev] = 1;
}

int sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// e^{-2 pi i k / L}, k < L, in extended precision, symmetric reduction
std::vector<cplx> twiddles(int L) {
  std::vector<cplx> t(L);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int k = 0; k < L; ++k) {
    const long double a = -2.0L * pi * (long double)k / (long double)L;
    t[k] = mk((double)cosl(a), (double)sinl(a));
  }
  return t;
}
}  // namespace

FftG::FftG(int L) : L_(L) {
  if (L < 1) fail(GS_ERR_DOMAIN, "FFT length must be positive");
  fg_smem_attr();
  if (L > FG_CAP) {
    // four-step: the divisor L1 <= FG_CAP closest to sqrt(L) with L / L1 <= FG_CAP
    int best = 0;
    for (int d = 2; d <= FG_CAP && d < L; ++d)
      if (L % d == 0 && L / d <= FG_CAP) {
        if (!best || std::abs(std::log((double)d) - 0.5 * std::log((double)L)) <
                         std::abs(std::log((double)best) - 0.5 * std::log((double)L)))
          best = d;
      }
    if (!best) fail(GS_ERR_DOMAIN, "FFT length " + std::to_string(L) + " has a prime factor beyond this build's engine");
    L1_ = best;
    L2_ = L / best;
    sub1_ = std::make_unique<FftG>(L1_);
    sub2_ = std::make_unique<FftG>(L2_);
  } else {
    int r = L;
    while (r % 2 == 0) {
      f_.push_back(2);
      r /= 2;
    }
    for (int p = 3; (long long)p * p <= r; p += 2)
      while (r % p == 0) {
        f_.push_back(p);
        r /= p;
      }
    if (r > 1) f_.push_back(r);
    if ((int)f_.size() > FG_MAXF) fail(GS_ERR_DOMAIN, "FFT length has too many factors");
  }
  std::vector<cplx> h = twiddles(L);
  tw_.upload(h.data(), h.size(), 0);
  CK(cudaStreamSynchronize(0));
}

void FftG::run(const cplx* in, cplx* out, int64_t count, int64_t batch, int64_t lstride, int64_t estride,
               int64_t bstride, int64_t olstride, int64_t oestride, int64_t obstride, int sign, cudaStream_t st) {
  if (L_ == 1) {
    if (in != out)
      for (int64_t b = 0; b < batch; ++b)
        for (int64_t l = 0; l < count; ++l)
          CK(cudaMemcpyAsync(out + b * obstride + l * olstride, in + b * bstride + l * lstride, sizeof(cplx),
                             cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (sub1_) {
    // X[k1 + L1 k2] = sum_n2 W_L^{n2 k1} W_L2^{n2 k2} sum_n1 x[L2 n1 + n2] W_L1^{n1 k1}
    const int64_t lines = count * batch;
    tmp_.alloc((size_t)lines * L_);
    // step 1: FFT_L1 over n1 for each n2 (input element stride L2 * estride) -> tmp[line][L2 k1 + n2]
    for (int64_t l = 0; l < count; ++l)
      sub1_->run(in + l * lstride, tmp_.p + l * L_, L2_, batch, estride, (int64_t)L2_ * estride, bstride, 1, L2_,
                 count * L_, sign, st);
    // step 2: pre-twiddle W_L^{n2 k1} + FFT_L2 over n2 for each k1 -> out[k1 + L1 k2]
    for (int64_t l = 0; l < count; ++l) {
      FgLines P{};
      P.L = L2_;
      P.nf = (int)sub2_->f_.size();
      for (int i = 0; i < P.nf; ++i) P.f[i] = sub2_->f_[i];
      P.tw = sub2_->tw_.p;
      P.sign = sign;
      P.G = std::max(1, std::min(8, FG_CAP / L2_));
      P.nlines = (int64_t)L1_ * batch;
      P.per = L1_;
      P.bstride = count * L_;
      P.lstride = L2_;
      P.estride = 1;
      P.obstride = obstride;
      P.olstride = oestride;
      P.oestride = (int64_t)L1_ * oestride;
      P.pretw = tw_.p;
      P.Lpre = L_;
      const size_t smem = 2 * (size_t)P.G * P.L * sizeof(cplx);
      k_fftg_lines<<<nblk(P.nlines, P.G), FG_THREADS, smem, st>>>(P, tmp_.p + l * L_, out + l * olstride);
      pmark("k_fftg_lines", st);
    }
    CKL();
    return;
  }
  FgLines P{};
  P.L = L_;
  P.nf = (int)f_.size();
  for (int i = 0; i < P.nf; ++i) P.f[i] = f_[i];
  P.tw = tw_.p;
  P.sign = sign;
  const int64_t lines = count * batch;
  int G = std::max(1, std::min(8, FG_CAP / L_));
  while (G > 1 && (lines + G - 1) / G < 2 * sms()) G /= 2;
  P.G = G;
  P.nlines = lines;
  P.per = count;
  P.bstride = bstride;
  P.lstride = lstride;
  P.estride = estride;
  P.obstride = obstride;
  P.olstride = olstride;
  P.oestride = oestride;
  P.pretw = nullptr;
  P.Lpre = 1;
  const size_t smem = 2 * (size_t)G * L_ * sizeof(cplx);
  k_fftg_lines<<<nblk(lines, G), FG_THREADS, smem, st>>>(P, in, out);
  pmark("k_fftg_lines", st);
  CKL();
}

// ------------------------------------------------------------------ device NfftPlan
void nfft_plan_validate(int dim, const int* N, int64_t M, int batch, const double* h_points, double sigma, int w) {
  // NfftPlan ctor checks in order (nufft.cpp:181-188, check_points 57-66)
  if (dim != 1 && dim != 2) fail(GS_ERR_DOMAIN, "dim must be 1 or 2");
  for (int d = 0; d < dim; ++d)
    if (N[d] <= 0 || N[d] % 2 != 0) fail(GS_ERR_DOMAIN, "transform length must be even");
  if (sigma < 1.25) fail(GS_ERR_DOMAIN, "oversampling factor must be >= 1.25");
  if (w < 2) fail(GS_ERR_DOMAIN, "kernel half-width must be >= 2");
  const int64_t cnt = M * dim * batch;
  for (int64_t i = 0; i < cnt; ++i)
    if (!(h_points[i] >= -0.5 && h_points[i] < 0.5)) fail(GS_ERR_DOMAIN, "scaled point outside [-1/2, 1/2)");
  if (M <= 0) fail(GS_ERR_SHAPE, "point array size is not a multiple of dim");
}

std::unique_ptr<NfftPlanDev> nfft_plan_build(int dim, const int* N, int64_t M, int batch, const double* h_points,
                                             double sigma, int w, cudaStream_t st, int vps) {
  nfft_plan_validate(dim, N, M, batch, h_points, sigma, w);
  const int64_t cnt = M * dim * batch;
  auto P = std::make_unique<NfftPlanDev>();
  P->dim = dim;
  P->batch = batch;
  P->vps = vps;
  P->M = M;
  P->w = w;
  P->S = 2 * w + 1;
  for (int d = 0; d < dim; ++d) {
    P->N[d] = N[d];
    P->nov[d] = (int)std::ceil(sigma * N[d] / 2.0) * 2;  // nufft.cpp:197-200
  }
  if (dim == 2 && ((int64_t)P->nov[0] > FG_CAP || (int64_t)P->nov[1] > FG_CAP))
    fail(GS_ERR_DOMAIN, "2D oversampled axis longer than " + std::to_string(FG_CAP) + " unsupported on this build");
  P->beta = kb_beta(sigma, w);
  DBuf<double> dp;
  dp.upload(h_points, cnt, st);
  P->base.alloc(cnt);
  P->wts.alloc(cnt * P->S);
  k_plan_window<<<nblk(cnt, 256), 256, 0, st>>>(dp.p, cnt, dim, P->nov[0], dim == 2 ? P->nov[1] : 1, w, P->beta,
                                               P->base.p, P->wts.p);
  pmark("k_plan_window", st);
  CKL();
  for (int d = 0; d < dim; ++d) {
    std::vector<double> dec(N[d]);
    for (int k = -N[d] / 2; k < N[d] / 2; ++k)
      dec[k + N[d] / 2] = 1.0 / kb_transform((double)k / (double)P->nov[d], w, P->beta);
    (d == 0 ? P->dec0 : P->dec1).upload(dec.data(), dec.size(), st);
  }
  if (dim == 1) {
    double one = 1.0;
    P->dec1.upload(&one, 1, st);
  }
  P->G.alloc((size_t)batch * vps * P->over_size());
  P->f0 = std::make_unique<FftG>(P->nov[0]);
  if (dim == 2) P->f1 = std::make_unique<FftG>(P->nov[1]);
  CK(cudaStreamSynchronize(st));
  return P;
}

namespace {
PlanDev pdev(const NfftPlanDev& P) {
  PlanDev d;
  d.dim = P.dim;
  d.N0 = P.N[0];
  d.N1 = P.dim == 2 ? P.N[1] : 1;
  d.n0 = P.nov[0];
  d.n1 = P.dim == 2 ? P.nov[1] : 1;
  d.S = P.S;
  d.M = P.M;
  d.vps = P.vps;
  d.lo = P.hi >= 0 ? P.lo : 0;
  d.hi = P.hi >= 0 ? P.hi : (P.dim == 2 ? std::max(P.N[0], P.N[1]) : P.N[0]);
  return d;
}
void grid_fft(NfftPlanDev& P, int sign, cudaStream_t st) {
  const int64_t over = P.over_size();
  const int64_t nv = (int64_t)P.batch * P.vps;
  if (P.dim == 1) {
    P.f0->run1d(P.G.p, P.G.p, nv, sign, st);
    return;
  }
  const int n0 = P.nov[0], n1 = P.nov[1];
  // rows (last axis, contiguous) then columns (stride n1): FFTW's 2D c2c
  P.f1->run(P.G.p, P.G.p, n0, nv, n1, 1, over, n1, 1, over, sign, st);
  P.f0->run(P.G.p, P.G.p, n1, nv, 1, n1, over, 1, n1, over, sign, st);
}
}  // namespace

void nfft_plan_forward(NfftPlanDev& P, const cplx* x, cplx* y, cudaStream_t st) {
  const PlanDev d = pdev(P);
  CK(cudaMemsetAsync(P.G.p, 0, P.G.bytes(), st));
  k_plan_embed<<<dim3(nblk(P.grid_size(), 256), P.batch * P.vps), 256, 0, st>>>(d, x, P.dec0.p, P.dec1.p, P.G.p);
  pmark("k_plan_embed", st);
  grid_fft(P, -1, st);
  k_plan_interp<<<dim3(nblk(P.M, 128), P.batch * P.vps), 128, 0, st>>>(d, P.base.p, P.wts.p, P.G.p, y);
  pmark("k_plan_interp", st);
  CKL();
}

void nfft_plan_adjoint(NfftPlanDev& P, const cplx* y, cplx* z, cudaStream_t st) {
  const PlanDev d = pdev(P);
  CK(cudaMemsetAsync(P.G.p, 0, P.G.bytes(), st));
  k_plan_spread<<<dim3(nblk(P.M, 128), P.batch * P.vps), 128, 0, st>>>(d, P.base.p, P.wts.p, y, P.G.p);
  pmark("k_plan_spread", st);
  grid_fft(P, +1, st);
  k_plan_crop<<<dim3(nblk(P.grid_size(), 256), P.batch * P.vps), 256, 0, st>>>(d, P.G.p, P.dec0.p, P.dec1.p, z);
  pmark("k_plan_crop", st);
  CKL();
}


// ------------------------------------------------------------------ uniform reduction, any length
__global__ void k_uni_embed(const cplx* __restrict__ x, int64_t n1, int64_t q, double phase_step, int64_t n2,
                            cplx* __restrict__ z, int lo, int hi) {
  // z[q l] = x_l e^{i phase_step l} (nufft.cpp:410-415), zeros elsewhere; batch = blockIdx.y
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n2) return;
  x += (int64_t)blockIdx.y * n1;
  z += (int64_t)blockIdx.y * n2;
  cplx v = mk(0, 0);
  if (i % q == 0 && i / q < n1 && i / q >= lo && i / q < hi) {
    const int64_t l = i / q;
    double s, c;
    sincos(phase_step * (double)l, &s, &c);
    v = cmul(x[l], mk(c, s));
  }
  z[i] = v;
}
__global__ void k_uni_out(const cplx* __restrict__ t, int64_t M, double eps, int64_t N, int64_t n1, cplx* __restrict__ y,
                          int64_t n2) {
  // y_m = e^{i pi n1 xi_m} FFT(z)_m, xi_m = eps / N (m - M/2) (nufft.cpp:421-427)
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= M) return;
  t += (int64_t)blockIdx.y * n2;
  y += (int64_t)blockIdx.y * M;
  const double xi = eps / (double)N * ((double)m - (double)M / 2.0);
  double s, c;
  sincos(GS_PI * (double)n1 * xi, &s, &c);
  y[m] = cmul(mk(c, s), t[m]);
}
__global__ void k_uni_adj_in(const cplx* __restrict__ y, int64_t M, double eps, int64_t N, int64_t n2,
                             cplx* __restrict__ z) {
  // padded[m] = y_m e^{-i pi N xi_m} (nufft.cpp:438-444), zeros past M
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n2) return;
  y += (int64_t)blockIdx.y * M;
  z += (int64_t)blockIdx.y * n2;
  cplx v = mk(0, 0);
  if (m < M) {
    const double xi = eps / (double)N * ((double)m - (double)M / 2.0);
    double s, c;
    sincos(-GS_PI * (double)N * xi, &s, &c);
    v = cmul(y[m], mk(c, s));
  }
  z[m] = v;
}
__global__ void k_uni_adj_out(const cplx* __restrict__ t, int64_t q, double phase_step, int64_t N, cplx* __restrict__ out,
                              int64_t n2) {
  // out_l = FFT+(padded)[q l] e^{-i phase_step l} (nufft.cpp:452-456)
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= N) return;
  t += (int64_t)blockIdx.y * n2;
  out += (int64_t)blockIdx.y * N;
  double s, c;
  sincos(-phase_step * (double)l, &s, &c);
  out[l] = cmul(t[q * l], mk(c, s));
}


std::unique_ptr<UniformDev> uniform_build(int64_t M, double eps, int64_t N, int batch) {
  const UniSetup s = uniform_setup(M, eps, N);
  if (s.n2 > (int64_t)INT32_MAX) fail(GS_ERR_DOMAIN, "DFT length too large");
  auto U = std::make_unique<UniformDev>();
  U->M = M;
  U->N = N;
  U->eps = eps;
  U->q = s.q;
  U->n2 = s.n2;
  U->batch = batch;
  U->fft = std::make_unique<FftG>((int)s.n2);
  U->z.alloc((size_t)batch * s.n2);
  return U;
}

void uniform_forward(UniformDev& U, const cplx* x, int lo, int hi, cplx* y, cudaStream_t st) {
  const double phase_step = GS_PI * U.eps * (double)U.M / (double)U.N;  // nufft.cpp:412
  k_uni_embed<<<dim3(nblk(U.n2, 256), U.batch), 256, 0, st>>>(x, U.N, U.q, phase_step, U.n2, U.z.p, lo, hi);
  pmark("k_uni_embed", st);
  U.fft->run1d(U.z.p, U.z.p, U.batch, -1, st);
  k_uni_out<<<dim3(nblk(U.M, 256), U.batch), 256, 0, st>>>(U.z.p, U.M, U.eps, U.N, U.N, y, U.n2);
  pmark("k_uni_out", st);
  CKL();
}

void uniform_adjoint(UniformDev& U, const cplx* y, cplx* z, cudaStream_t st) {
  const double phase_step = GS_PI * U.eps * (double)U.M / (double)U.N;
  k_uni_adj_in<<<dim3(nblk(U.n2, 256), U.batch), 256, 0, st>>>(y, U.M, U.eps, U.N, U.n2, U.z.p);
  pmark("k_uni_adj_in", st);
  U.fft->run1d(U.z.p, U.z.p, U.batch, +1, st);
  k_uni_adj_out<<<dim3(nblk(U.N, 256), U.batch), 256, 0, st>>>(U.z.p, U.q, phase_step, U.N, z, U.n2);
  pmark("k_uni_adj_out", st);
  CKL();
}

}  // namespace gsb

// ====================================================================== C-ABI
using namespace gsb;

struct gs_nfft_plan {
  std::unique_ptr<NfftPlanDev> P;
  int device = 0;
  std::mutex mu;
  DBuf<cplx> in, out;
};

namespace plan_capi {

// host or device vector -> device pointer (staged copy in `buf` when host)
const cplx* dev_in(const double* p, int64_t n, DBuf<cplx>& buf, cudaStream_t st) {
  if (is_device_ptr(p)) return (const cplx*)p;
  buf.upload((const cplx*)p, n, st);
  return buf.p;
}

int uniform_call(bool adjoint, const double* in, int64_t in_len, int64_t M, double eps, int64_t N, double* out,
                 void* stream) {
  return guard_call([&] {
    if (!in || !out) fail(GS_ERR_USAGE, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (!adjoint && in_len > N) fail(GS_ERR_DOMAIN, "signal length must not exceed N");
    auto U = uniform_build(adjoint ? in_len : M, eps, N, 1);
    thread_local DBuf<cplx> t_in, t_x, t_out;
    const cplx* din = dev_in(in, in_len, t_in, st);
    const int64_t out_len = adjoint ? N : M;
    const bool dev_out = is_device_ptr(out);
    if (!dev_out) t_out.alloc(out_len);
    cplx* dout = dev_out ? (cplx*)out : t_out.p;
    if (!adjoint) {
      // x shorter than N: zero-extend (nufft.cpp:408-415 embeds only l < n1, and the
      // output phase uses n1, not N)
      t_x.alloc(N);
      CK(cudaMemsetAsync(t_x.p, 0, N * sizeof(cplx), st));
      CK(cudaMemcpyAsync(t_x.p, din, in_len * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      const double phase_step = GS_PI * eps * (double)M / (double)N;
      k_uni_embed<<<dim3(nblk(U->n2, 256), 1), 256, 0, st>>>(t_x.p, N, U->q, phase_step, U->n2, U->z.p, 0, (int)in_len);
      pmark("k_uni_embed", st);
      U->fft->run1d(U->z.p, U->z.p, 1, -1, st);
      k_uni_out<<<dim3(nblk(M, 256), 1), 256, 0, st>>>(U->z.p, M, eps, N, in_len, dout, U->n2);
      pmark("k_uni_out", st);
      CKL();
    } else {
      uniform_adjoint(*U, din, dout, st);
    }
    if (!dev_out) CK(cudaMemcpyAsync(out, dout, out_len * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

}  // namespace plan_capi

extern "C" {

int gs_nfft_plan_create(int dim, const int* N, const double* points, int64_t M, double sigma, int w, int device,
                        gs_nfft_plan** out) {
  return guard_call([&] {
    if (!N || !out || (!points && M > 0)) fail(GS_ERR_USAGE, "null argument");
    *out = nullptr;
    std::vector<double> h;
    const double* hp = points;
    if (M > 0 && is_device_ptr(points)) {
      h.resize((size_t)M * (dim == 2 ? 2 : 1));
      CK(cudaMemcpy(h.data(), points, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
      hp = h.data();
    }
    nfft_plan_validate(dim, N, M, 1, hp, sigma, w);  // error classes before touching the device
    CK(cudaSetDevice(device));
    auto pl = std::make_unique<gs_nfft_plan>();
    pl->device = device;
    pl->P = nfft_plan_build(dim, N, M, 1, hp, sigma, w, 0);
    *out = pl.release();
  });
}

int gs_nfft_plan_destroy(gs_nfft_plan* p) {
  delete p;
  return GS_OK;
}

int gs_nfft_plan_info(const gs_nfft_plan* p, int* dim, int64_t* points, int64_t* grid_size, int* n_over) {
  if (!p) {
    g_err = "null plan";
    return GS_ERR_USAGE;
  }
  if (dim) *dim = p->P->dim;
  if (points) *points = p->P->M;
  if (grid_size) *grid_size = p->P->grid_size();
  if (n_over) {
    n_over[0] = p->P->nov[0];
    n_over[1] = p->P->dim == 2 ? p->P->nov[1] : 0;
  }
  return GS_OK;
}

static int plan_apply(gs_nfft_plan* p, bool adjoint, const double* in, int64_t in_len, double* out, void* stream) {
  return guard_call([&] {
    if (!p || !in || !out) fail(GS_ERR_USAGE, "null argument");
    NfftPlanDev& P = *p->P;
    if (!adjoint && in_len != P.grid_size()) fail(GS_ERR_SHAPE, "grid size mismatch");
    if (adjoint && in_len != P.M) fail(GS_ERR_SHAPE, "sample count mismatch");
    std::lock_guard<std::mutex> lk(p->mu);
    CK(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    const cplx* din = plan_capi::dev_in(in, in_len, p->in, st);
    const int64_t out_len = adjoint ? P.grid_size() : P.M;
    const bool dev_out = is_device_ptr(out);
    if (!dev_out) p->out.alloc(out_len);
    cplx* dout = dev_out ? (cplx*)out : p->out.p;
    if (adjoint) nfft_plan_adjoint(P, din, dout, st);
    else nfft_plan_forward(P, din, dout, st);
    if (!dev_out) CK(cudaMemcpyAsync(out, dout, out_len * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int gs_nfft_plan_forward(gs_nfft_plan* p, const double* grid, int64_t grid_len, double* samples, void* stream) {
  return plan_apply(p, false, grid, grid_len, samples, stream);
}
int gs_nfft_plan_adjoint(gs_nfft_plan* p, const double* samples, int64_t samples_len, double* grid, void* stream) {
  return plan_apply(p, true, samples, samples_len, grid, stream);
}

int gs_uniform_ndft_fft(const double* x, int64_t x_len, int64_t M, double epsilon, int64_t N, double* out,
                        void* stream) {
  return plan_capi::uniform_call(false, x, x_len, M, epsilon, N, out, stream);
}
int gs_uniform_ndft_adjoint_fft(const double* samples, int64_t M, double epsilon, int64_t N, double* out,
                                void* stream) {
  return plan_capi::uniform_call(true, samples, M, M, epsilon, N, out, stream);
}

}  // extern "C"
