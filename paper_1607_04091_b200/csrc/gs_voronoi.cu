// gs_voronoi.cu -- exact Voronoi density-compensation weights on the GPU
// (weights.cpp:59-133 semantics): one thread per 2D cell runs
// the same clip-against-neighbours routine as the host harness
// (voronoi_common.h: vor_cell_stream, the host's clip sequence minus its exact
// no-ops, with no candidate buffer), compiled without FMA contraction
// (-fmad=false in the Makefile), so the device doubles equal the host's bit
// for bit.  Cells whose polygon outgrows the thread's buffer are flagged and
// finished on the host with unbounded buffers.  1D weights are a
// sort and midpoints: they stay on the host (gs_voronoi_weights).
#include <cmath>
#include <thread>
#include <vector>

#include "host_common.cuh"
#include "voronoi_common.h"

#define VOR_CAPV 64

namespace {

__global__ void __launch_bounds__(128) k_voronoi_cells(VorGrid g, double* __restrict__ mu, unsigned char* __restrict__ overflow) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= g.M) return;
  double px[VOR_CAPV], py[VOR_CAPV], qx[VOR_CAPV], qy[VOR_CAPV];
  double area = 0.0;
  const int rc = vor_cell_stream(g, m, px, py, qx, qy, VOR_CAPV, &area);
  mu[m] = area;
  overflow[m] = rc != VOR_OK;
}

}  // namespace

using namespace gsb;

extern "C" const char* gs_inputs_last_error(void);
extern "C" int gs_voronoi_weights(int dim, int64_t M, const double* coords, double K, double* mu, int nthreads);

extern "C" int gs_voronoi_weights_gpu(int dim, int64_t M, const double* coords, double K, double* mu, int device,
                                      void* stream) {
  if (dim != 2) return gs_voronoi_weights(dim, M, coords, K, mu, 0);  // 1D: host sort + midpoints
  return guard_call([&] {
    if (!coords || !mu) fail(GS_ERR_USAGE, "null argument");
    if (!(K > 0)) fail(GS_ERR_DOMAIN, "K must be positive");
    if (M <= 0) fail(GS_ERR_SHAPE, "empty point set");
    std::vector<int64_t> start, idx;
    int G = 1;
    double h = 0.0;
    const int rc = vor_grid_build(M, coords, K, start, idx, G, h);  // range + duplicate checks (host)
    if (rc) fail(rc, gs_inputs_last_error());
    CK(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    DBuf<double> dc, dmu;
    DBuf<int64_t> ds, di;
    DBuf<unsigned char> dof;
    dc.upload(coords, 2 * M, st);
    ds.upload(start.data(), start.size(), st);
    di.upload(idx.data(), idx.size(), st);
    dmu.alloc(M);
    dof.alloc(M);
    const VorGrid g{dc.p, ds.p, di.p, M, G, K, h};
    k_voronoi_cells<<<nblk(M, 128), 128, 0, st>>>(g, dmu.p, dof.p);
    pmark("k_voronoi_cells", st);
    CKL();
    std::vector<unsigned char> of(M);
    CK(cudaMemcpyAsync(mu, dmu.p, M * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(of.data(), dof.p, M, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // cells beyond the thread buffers: the same routine on the host, unbounded, threaded
    std::vector<int64_t> todo;
    for (int64_t m = 0; m < M; ++m)
      if (of[m]) todo.push_back(m);
    const VorGrid hg{coords, start.data(), idx.data(), M, G, K, h};
    auto work = [&](size_t lo, size_t hi) {
      int capv = 1024, capc = 4096;
      std::vector<double> px(capv), py(capv), qx(capv), qy(capv), cd(capc);
      std::vector<int64_t> cj(capc);
      for (size_t t = lo; t < hi; ++t) {
        const int64_t m = todo[t];
        while (vor_cell(hg, m, px.data(), py.data(), qx.data(), qy.data(), capv, cd.data(), cj.data(), capc, mu + m,
                        nullptr) != VOR_OK) {
          capv *= 2;
          capc *= 2;
          px.resize(capv);
          py.resize(capv);
          qx.resize(capv);
          qy.resize(capv);
          cd.resize(capc);
          cj.resize(capc);
        }
      }
    };
    const size_t T = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), todo.size() / 16 + 1));
    std::vector<std::thread> th;
    for (size_t t = 0; t < T; ++t) th.emplace_back(work, todo.size() * t / T, todo.size() * (t + 1) / T);
    for (auto& t : th) t.join();
  });
}
