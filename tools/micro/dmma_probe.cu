// Microbenchmark: FP64 tensor-core (mma.sync f64) vs DFMA throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double* d, double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <int KIND>
__global__ void k(double* out, int iters, double seed) {
  const int lane = threadIdx.x & 31;
  double a = seed + lane * 1e-3, b = seed - lane * 1e-3;
  double acc[8][4];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) mma884(acc[i][0], acc[i][1], a, b);
      else if (KIND == 1) mma1684(acc[i], a, b, b);
      else if (KIND == 2) { double av[4] = {a, b, a, b}; double bv[2] = {b, a}; mma1688(acc[i], av, bv); }
      else {
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a, b, acc[i][j]);
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 16 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"mma m8n8k4 f64", "mma m16n8k4 f64", "mma m16n8k8 f64", "DFMA (fma)"};
  const double fma_per_inst_warp[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 32 * 4};  // per unrolled step per warp
  for (int kind = 0; kind < 4; ++kind) {
    for (int cfg : {0, 1, 2, 3}) {
      const int blocks_per_sm = cfg == 0 ? 2 : (cfg == 1 ? 4 : (cfg == 2 ? 8 : 16));
      const int grid = 148 * blocks_per_sm, threads = 128, iters = 2000;
      auto launch = [&] {
        if (kind == 0) k<0><<<grid, threads>>>(out, iters, 1.0);
        else if (kind == 1) k<1><<<grid, threads>>>(out, iters, 1.0);
        else if (kind == 2) k<2><<<grid, threads>>>(out, iters, 1.0);
        else k<3><<<grid, threads>>>(out, iters, 1.0);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)grid * threads / 32;
      const double fmas = warps * iters * 8 * fma_per_inst_warp[kind];
      printf("%-18s warps/SM %d: %.2f TFLOP/s (%.3f ms) err=%s\n", names[kind], blocks_per_sm * 4, 2 * fmas / (ms * 1e-3) / 1e12,
             ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
