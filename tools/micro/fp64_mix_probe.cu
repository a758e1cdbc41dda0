// Microbenchmark: do the FP64 tensor pipe (mma.sync m8n8k4 f64) and the DFMA pipe
// run concurrently on this GPU?  Warps of a CTA either issue DMMAs, DFMAs, or
// both interleaved; the combined FLOP rate above the single-pipe rate says yes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix_probe fp64_mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// MODE 0: DMMA only; 1: DFMA only; 2: even warps DMMA, odd warps DFMA;
// 3: every warp interleaves 8 DMMA with NF DFMA steps (4 independent chains each)
template <int MODE, int NF>
__global__ void k(double* out, int iters, double seed) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a = seed + lane * 1e-3, b = seed - lane * 1e-3;
  double acc[8][2], f[NF > 0 ? NF : 1][4];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i)
    for (int j = 0; j < 4; ++j) f[i][j] = 0.0;
  const bool dm = MODE == 0 || MODE == 3 || (MODE == 2 && (warp & 1) == 0);
  const bool df = MODE == 1 || MODE == 3 || (MODE == 2 && (warp & 1) == 1);
  for (int it = 0; it < iters; ++it) {
    if (dm) {
#pragma unroll
      for (int i = 0; i < 8; ++i) mma884(acc[i][0], acc[i][1], a, b);
    }
    if (df) {
#pragma unroll
      for (int i = 0; i < (NF > 0 ? NF : 1); ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) f[i][j] = fma(a, b, f[i][j]);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i)
    for (int j = 0; j < 4; ++j) s += f[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int NF>
void run(const char* name, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  for (int bps : {2, 4}) {
    const int grid = 148 * bps, threads = 256, iters = 2000;
    k<MODE, NF><<<grid, threads>>>(out, iters, 1.0);
    cudaEventRecord(e0);
    k<MODE, NF><<<grid, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)grid * threads / 32;
    double dwarps = MODE == 1 ? 0 : (MODE == 2 ? warps / 2 : warps);
    double fwarps = MODE == 0 ? 0 : (MODE == 2 ? warps / 2 : warps);
    const double dmma_fma = dwarps * iters * 8 * 256.0;
    const double dfma_fma = fwarps * iters * (NF > 0 ? NF : 1) * 4 * 32.0;
    printf("%-34s CTAs/SM %d: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms) %s\n", name, bps,
           2 * dmma_fma / (ms * 1e-3) / 1e12, 2 * dfma_fma / (ms * 1e-3) / 1e12,
           2 * (dmma_fma + dfma_fma) / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 4 * 256 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  run<0, 0>("DMMA only", out, e0, e1);
  run<1, 16>("DFMA only (16x4 chains)", out, e0, e1);
  run<2, 16>("half warps DMMA, half DFMA", out, e0, e1);
  run<3, 4>("interleaved 8 DMMA : 4x4 DFMA", out, e0, e1);
  run<3, 8>("interleaved 8 DMMA : 8x4 DFMA", out, e0, e1);
  run<3, 16>("interleaved 8 DMMA : 16x4 DFMA", out, e0, e1);
  return 0;
}
