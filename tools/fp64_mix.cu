// Are DFMA and DMMA separate pipes on sm_100a?  Runs a DFMA loop and a DMMA
// loop alone, then in different warps of the same CTA, and reports the
// aggregate FP64 rate (dev tool; informs phase overlap in the engine).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_work(double* out, int iters) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-9 + j;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  double s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ void dmma_work(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mode 0: all warps DFMA, 1: all DMMA, 2: even warps DFMA / odd warps DMMA
__global__ void mix(double* out, int it_f, int it_m, int mode) {
  const int w = threadIdx.x >> 5;
  const bool f = mode == 0 || (mode == 2 && (w & 1) == 0);
  if (f) dfma_work(out, it_f); else dmma_work(out, it_m);
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 4 * 512);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int bs = 512, blocks = sms * 2;  // 32 warps / SM
  // per warp: DFMA work = it_f*128*32 lane-FMA, DMMA work = it_m*32*256 MAC
  const int it_f = 4096, it_m = 2048;    // equal MACs per warp
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      mix<<<blocks, bs>>>(out, it_f, it_m, mode);
      cudaEventRecord(e0);
      mix<<<blocks, bs>>>(out, it_f, it_m, mode);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double macs_per_warp = double(it_f) * 128 * 32;
      const double flops = 2.0 * macs_per_warp * blocks * (bs / 32);
      printf("mode %d (%s): %.3f ms, %.1f TFLOP/s aggregate\n", mode,
             mode == 0 ? "DFMA only" : mode == 1 ? "DMMA only" : "half DFMA + half DMMA warps", ms,
             flops / ms / 1e9);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
