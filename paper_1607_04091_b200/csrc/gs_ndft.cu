// gs_ndft.cu -- direct NDFT (a14: ndft_forward / ndft_adjoint, nufft.cpp:74-132)
// on the device: launch helpers for the operator's exact route and the C-ABI
// entry points gs_ndft_forward / gs_ndft_adjoint (include/gs_b200.h).
#include <algorithm>
#include <cmath>
#include <vector>

#include "kernels_ndft.cuh"
#include "ndft.h"

namespace gsb {
namespace {

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

NdGeom geom(const NdftShape& s, int lo, int hi) {
  NdGeom g;
  g.dim = s.dim;
  g.N0 = s.N0;
  g.N1 = s.N1;
  g.runs = (s.N1 + ND_RUN - 1) / ND_RUN;
  g.M = s.M;
  g.lo = lo;
  g.hi = hi;
  g.rh0 = s.dim == 1 ? 1 : 2 * (s.N0 / 2);
  g.kh1 = 2 * (s.N1 / 2);
  return g;
}

}  // namespace

void ndft_forward_launch(const NdftShape& s, const double* pts, const cplx* x, cplx* y, int lo, int hi,
                         const cplx* rec, int p, int edges, DBuf<cplx>& part, cudaStream_t st) {
  const NdGeom g = geom(s, lo, hi);
  const int nunits = g.N0 * g.runs;
  const int64_t nb = (s.M + ND_FTHREADS * ND_FPPT - 1) / (ND_FTHREADS * ND_FPPT);
  // split the units so that ~4 CTAs per SM are in flight, at least 8 units per split
  const int64_t want = (int64_t)4 * sm_count();
  int ks = (int)std::max<int64_t>(1, std::min<int64_t>(want / std::max<int64_t>(1, nb * s.batch), nunits / 8));
  const int ups = (nunits + ks - 1) / ks;
  ks = (nunits + ups - 1) / ups;
  part.alloc((size_t)s.batch * ks * s.M);
  k_ndft_fwd<<<dim3((unsigned)nb, ks, s.batch), ND_FTHREADS, 0, st>>>(g, pts, x, ups, part.p);
  pmark("k_ndft_fwd", st);
  k_ndft_fwd_reduce<<<dim3(nblk(s.M * 32, 256), s.batch), 256, 0, st>>>(s.M, ks, part.p, rec, p, edges, x, s.N1, y);
  pmark("k_ndft_fwd_reduce", st);
  CKL();
}

void ndft_adjoint_launch(const NdftShape& s, const double* pts, const cplx* y, cplx* z, int lo, int hi,
                         const cplx* rec, int p, int edges, DBuf<cplx>& part, cudaStream_t st) {
  const NdGeom g = geom(s, 0, s.N1);
  // two units per thread (giant-step chained) once there are enough of them
  const int aupt = (int64_t)g.N0 * g.runs * s.batch >= 8192 ? 2 : 1;
  const int groups = g.N0 * ((g.runs + aupt - 1) / aupt);
  const int64_t nb = (groups + ND_ATHREADS - 1) / ND_ATHREADS;
  const int64_t want = (int64_t)4 * sm_count();
  int64_t ms = std::max<int64_t>(1, std::min<int64_t>(want / std::max<int64_t>(1, nb * s.batch),
                                                      (s.M + ND_ATILE - 1) / ND_ATILE));
  int64_t pps = (s.M + ms - 1) / ms;
  pps = (pps + ND_ATILE - 1) / ND_ATILE * ND_ATILE;
  ms = (s.M + pps - 1) / pps;
  const int64_t nmodes = (int64_t)s.N0 * s.N1;
  part.alloc((size_t)s.batch * ms * nmodes);
  const int Rr = 1 + (edges ? 2 * p : 0);
  if (aupt == 2)
    k_ndft_adj<2><<<dim3((unsigned)nb, (unsigned)ms, s.batch), ND_ATHREADS, 0, st>>>(g, pts, y, rec, Rr, pps, part.p);
  else
    k_ndft_adj<1><<<dim3((unsigned)nb, (unsigned)ms, s.batch), ND_ATHREADS, 0, st>>>(g, pts, y, rec, Rr, pps, part.p);
  pmark("k_ndft_adj", st);
  k_ndft_adj_reduce<<<dim3(nblk(nmodes * 32, 256), s.batch), 256, 0, st>>>(nmodes, (int)ms, part.p, lo, hi, z);
  pmark("k_ndft_adj_reduce", st);
  if (rec && edges) {
    k_ndft_adj_edges<<<dim3(2 * p, s.batch), 256, 0, st>>>(s.M, rec, p, y, s.N1, z);
    pmark("k_ndft_adj_edges", st);
  }
  CKL();
}

void op1d_epilogue_launch(int64_t M, int batch, const cplx* u, const cplx* rec, int p, int edges, const cplx* x, int n,
                          cplx* y, cudaStream_t st) {
  k_ndft_fwd_reduce<<<dim3(nblk(M * 32, 256), batch), 256, 0, st>>>(M, 1, u, rec, p, edges, x, n, y);
  pmark("k_op1d_epilogue", st);
  CKL();
}

void op1d_edges_launch(int64_t M, int batch, const cplx* rec, int p, const cplx* y, int n, cplx* z, cudaStream_t st) {
  k_ndft_adj_edges<<<dim3(2 * p, batch), 256, 0, st>>>(M, rec, p, y, n, z);
  pmark("k_op1d_edges", st);
  CKL();
}

}  // namespace gsb

using namespace gsb;

namespace ndft_capi {

// check_points (nufft.cpp:57-66) + staging of host arrays; returns device pointers
struct Staged {
  DBuf<double> pts;
  DBuf<cplx> in, out;
};

void check_points_host(const double* pts, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!(pts[i] >= -0.5 && pts[i] < 0.5)) fail(GS_ERR_DOMAIN, "scaled point outside [-1/2, 1/2)");
}

__global__ void k_check_points(const double* __restrict__ pts, int64_t n, int* __restrict__ bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && !(pts[i] >= -0.5 && pts[i] < 0.5)) *bad = 1;
}

// per-thread workspaces of the C-ABI calls (grown, never freed per call: a
// cudaFree per call would synchronise the device)
thread_local DBuf<int> t_bad;
thread_local DBuf<cplx> t_part, t_in, t_out;
thread_local DBuf<double> t_pts;

const double* stage_points(const double* pts, int64_t n, Staged& S, cudaStream_t st) {
  (void)S;
  if (is_device_ptr(pts)) {
    DBuf<int>& bad = t_bad;
    bad.alloc(1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    k_check_points<<<nblk(n, 256), 256, 0, st>>>(pts, n, bad.p);
    CKL();
    int h = 0;
    CK(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h) fail(GS_ERR_DOMAIN, "scaled point outside [-1/2, 1/2)");
    return pts;
  }
  check_points_host(pts, n);
  t_pts.upload(pts, n, st);
  return t_pts.p;
}

int ndft_call(bool adjoint, int dim, const int* N, const double* points, int64_t M, const double* in, int64_t in_len,
              double* out, void* stream) {
  return guard_call([&] {
    if (!N || !points || !in || !out) fail(GS_ERR_USAGE, "null argument");
    if (dim != 1 && dim != 2) fail(GS_ERR_DOMAIN, "dim must be 1 or 2");
    cudaStream_t st = (cudaStream_t)stream;
    Staged S;
    // nufft.cpp:57-66: range first, then emptiness
    const double* dp = M > 0 ? stage_points(points, M * dim, S, st) : nullptr;
    if (M <= 0) fail(GS_ERR_SHAPE, "point array size is not a multiple of dim");
    NdftShape s;
    s.dim = dim;
    s.N0 = dim == 2 ? N[0] : 1;
    s.N1 = dim == 2 ? N[1] : N[0];
    s.M = M;
    s.batch = 1;
    if (s.N0 <= 0 || s.N1 <= 0) fail(GS_ERR_DOMAIN, "transform length must be positive");
    const int64_t nmodes = (int64_t)s.N0 * s.N1;
    if (!adjoint && in_len != nmodes) fail(GS_ERR_SHAPE, "grid size mismatch");
    if (adjoint && in_len != M) fail(GS_ERR_SHAPE, "sample count mismatch");
    const int64_t out_len = adjoint ? nmodes : M;
    const cplx* din = (const cplx*)in;
    if (!is_device_ptr(in)) {
      t_in.upload((const cplx*)in, in_len, st);
      din = t_in.p;
    }
    const bool dev_out = is_device_ptr(out);
    cplx* dout = (cplx*)out;
    if (!dev_out) {
      t_out.alloc(out_len);
      dout = t_out.p;
    }
    DBuf<cplx>& part = t_part;
    if (adjoint) ndft_adjoint_launch(s, dp, din, dout, 0, s.N1 * s.N0, nullptr, 1, 0, part, st);
    else ndft_forward_launch(s, dp, din, dout, 0, s.N1, nullptr, 1, 0, part, st);
    if (!dev_out) CK(cudaMemcpyAsync(out, dout, out_len * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

}  // namespace ndft_capi

using ndft_capi::ndft_call;

extern "C" int gs_ndft_forward(int dim, const int* N, const double* points, int64_t M, const double* grid,
                               int64_t grid_len, double* samples, void* stream) {
  return ndft_call(false, dim, N, points, M, grid, grid_len, samples, stream);
}

extern "C" int gs_ndft_adjoint(int dim, const int* N, const double* points, int64_t M, const double* samples,
                               int64_t samples_len, double* grid, void* stream) {
  return ndft_call(true, dim, N, points, M, samples, samples_len, grid, stream);
}
