// ndft.h -- host launchers of the direct NDFT kernels (kernels_ndft.cuh),
// shared by the C-ABI entry points (gs_ndft.cu) and the operator's exact
// NDFT route (gs_capi.cu, GS_ROUTE_NDFT_1D).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "host_common.cuh"

typedef double2 cplx;

namespace gsb {

struct NdftShape {
  int dim;      // 1 or 2
  int N0, N1;   // 1D: N0 = 1, N1 = N
  int64_t M;    // points per problem
  int batch;    // independent problems (pts [B][M][dim], modes [B][N0 N1], samples [B][M])
};

// y = NDFT(x) per problem.  lo / hi (1D operator use): only mode indices
// [lo, hi) of x enter; rec != nullptr: operator epilogue (D, L, R records,
// freq2wave.cpp:232-236; p, edges, n = modes) -- else y is the plain sum.
void ndft_forward_launch(const NdftShape& s, const double* pts, const cplx* x, cplx* y, int lo, int hi,
                         const cplx* rec, int p, int edges, DBuf<cplx>& part, cudaStream_t st);
// z = NDFT^H(y) per problem; rec != nullptr: samples weighted by conj(D_m), only
// [lo, hi) written, edge columns from the L / R records (freq2wave.cpp:318-324).
void ndft_adjoint_launch(const NdftShape& s, const double* pts, const cplx* y, cplx* z, int lo, int hi,
                         const cplx* rec, int p, int edges, DBuf<cplx>& part, cudaStream_t st);

// the 1D operator algebra around any core transform u = F(x~) (freq2wave.cpp:232-236,
// 318-324): y = D o u + L x[0:p] + R x[n-p:n]; edge columns z_c = L^H y, R^H y
void op1d_epilogue_launch(int64_t M, int batch, const cplx* u, const cplx* rec, int p, int edges, const cplx* x, int n,
                          cplx* y, cudaStream_t st);
void op1d_edges_launch(int64_t M, int batch, const cplx* rec, int p, const cplx* y, int n, cplx* z, cudaStream_t st);

}  // namespace gsb
