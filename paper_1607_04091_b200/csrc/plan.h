// plan.h -- the general-length FFT engine (kernels_fftg.cuh) and the device
// NfftPlan (kernels_plan.cuh) as host objects, shared by the C-ABI of the
// lower-level API (gs_plan.cu: gs_nfft_plan_*, gs_uniform_ndft_*) and the
// operator's general routes (gs_capi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

#include "host_common.cuh"

typedef double2 cplx;

namespace gsb {

// FFT of length L over batched strided lines, any L whose factors fit the
// engine (one CTA per group of lines up to FG_CAP points, four-step beyond).
class FftG {
 public:
  explicit FftG(int L);
  int length() const { return L_; }
  // lines: `count` lines per problem x `batch` problems; element j of line l of
  // problem b at in + b*bstride + l*lstride + j*estride (output likewise);
  // in == out allowed.  sign -1 = FFTW_FORWARD, +1 = BACKWARD (unnormalised).
  void run(const cplx* in, cplx* out, int64_t count, int64_t batch, int64_t lstride, int64_t estride,
           int64_t bstride, int64_t olstride, int64_t oestride, int64_t obstride, int sign, cudaStream_t st);
  // contiguous 1D transforms of `batch` vectors of length L
  void run1d(const cplx* in, cplx* out, int64_t batch, int sign, cudaStream_t st) {
    run(in, out, 1, batch, 0, 1, L_, 0, 1, L_, sign, st);
  }

 private:
  int L_ = 0;
  std::vector<int> f_;
  DBuf<cplx> tw_;
  std::unique_ptr<FftG> sub1_, sub2_;  // four-step factors L = L1 L2
  int L1_ = 0, L2_ = 0;
  DBuf<cplx> tmp_;
};

// Device NfftPlan (nufft.cpp:138-233): batch >= 1 point sets of equal size M
// sharing N, sigma, w.  Points are scaled to [-1/2, 1/2), point-major.
struct NfftPlanDev {
  int dim = 1, batch = 1;
  int vps = 1;          // vectors per point set (forward / adjoint take [batch][vps][...])
  int lo = 0, hi = -1;  // forward embed mask on every axis (operator interiors); -1 = none
  int N[2] = {0, 1};
  int nov[2] = {0, 1};
  int w = 6, S = 13;
  double beta = 0;
  int64_t M = 0;
  DBuf<int> base;       // [B][M][dim] wrapped window origins
  DBuf<double> wts;     // [B][M][dim][S]
  DBuf<double> dec0, dec1;
  DBuf<cplx> G;         // [B][n0 n1] oversampled grid
  std::unique_ptr<FftG> f0, f1;
  int64_t grid_size() const { return (int64_t)N[0] * N[1]; }
  int64_t over_size() const { return (int64_t)nov[0] * nov[1]; }
};

// validation (nufft.cpp:181-188; dim, even N, sigma, w, point range) + device tables;
// d_points: [B][M][dim] device array of scaled points (checked on the host copy h_points)
void nfft_plan_validate(int dim, const int* N, int64_t M, int batch, const double* h_points, double sigma, int w);
std::unique_ptr<NfftPlanDev> nfft_plan_build(int dim, const int* N, int64_t M, int batch, const double* h_points,
                                             double sigma, int w, cudaStream_t st, int vps = 1);
void nfft_plan_forward(NfftPlanDev& P, const cplx* x, cplx* y, cudaStream_t st);   // nufft.cpp:244-306
void nfft_plan_adjoint(NfftPlanDev& P, const cplx* y, cplx* z, cudaStream_t st);   // nufft.cpp:308-365

// The uniform-grid reduction (nufft.cpp:383-459) at any DFT length, batched:
// forward x [batch][N] (only indices [lo, hi) enter; edge slots of an
// operator) -> y [batch][M]; adjoint y [batch][M] -> z [batch][N].
struct UniformDev {
  int64_t M = 0, N = 0, q = 0, n2 = 0;
  double eps = 0;
  int batch = 1;
  std::unique_ptr<FftG> fft;
  DBuf<cplx> z;
};
std::unique_ptr<UniformDev> uniform_build(int64_t M, double eps, int64_t N, int batch);
void uniform_forward(UniformDev& U, const cplx* x, int lo, int hi, cplx* y, cudaStream_t st);
void uniform_adjoint(UniformDev& U, const cplx* y, cplx* z, cudaStream_t st);

}  // namespace gsb
