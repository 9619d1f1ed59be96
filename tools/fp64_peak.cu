// FP64 peak probe: DFMA vector loop and DMMA (mma.sync m8n8k4 f64) loop.
// Used to set the FP64 roofline denominator (not in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    for (int bs : {256, 512, 1024}) {
      int blocks = sms * (2048 / bs);
      dfma_loop<<<blocks, bs>>>(out, iters);
      cudaEventRecord(e0);
      dfma_loop<<<blocks, bs>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 16 * double(iters) * blocks * bs;
      printf("DFMA bs=%d: %.2f TFLOP/s (%.3f ms)\n", bs, flops / ms / 1e9, ms);
    }
    for (int bs : {128, 256, 512}) {
      int blocks = sms * 4;
      dmma_loop<<<blocks, bs>>>(out, iters / 4);
      cudaEventRecord(e0);
      dmma_loop<<<blocks, bs>>>(out, iters / 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * 16 * double(iters / 4) * blocks * (bs / 32);
      printf("DMMA bs=%d: %.2f TFLOP/s (%.3f ms)\n", bs, flops / ms / 1e9, ms);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
