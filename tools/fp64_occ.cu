// FP64 issue probe: DFMA / DMMA throughput vs resident warps per SM and
// independent accumulator chains per thread (dev tool; informs the M2L design).
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void dfma_c(double* out, int iters) {
  double a[C];
#pragma unroll
  for (int j = 0; j < C; ++j) a[j] = threadIdx.x * 1e-9 + j;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 128 / C; ++r)
#pragma unroll
      for (int j = 0; j < C; ++j) a[j] = fma(a[j], b, c);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < C; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int C>
__global__ void dmma_c(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[C][2];
  for (int t = 0; t < C; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 32 / C; ++r)
#pragma unroll
      for (int t = 0; t < C; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < C; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
float run(K k, int blocks, int bs, int iters, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks, bs>>>(out, iters);
  cudaEventRecord(e0);
  k<<<blocks, bs>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 2048);
  const int iters = 2048;
  for (int wps : {1, 2, 3, 4, 6, 8}) {  // warps per SMSP: one CTA of 4*wps warps per SM
    const int bs = 128 * wps;
    float m4 = run(dfma_c<4>, sms, bs, iters, out), m8 = run(dfma_c<8>, sms, bs, iters, out);
    float m16 = run(dfma_c<16>, sms, bs, iters, out), m32 = run(dfma_c<32>, sms, bs, iters, out);
    double fl = 2.0 * 128 * double(iters) * sms * bs / 1e9;
    printf("DFMA warps/SMSP=%d: C4 %.1f  C8 %.1f  C16 %.1f  C32 %.1f TF\n", wps, fl / m4, fl / m8, fl / m16, fl / m32);
    float d1 = run(dmma_c<1>, sms, bs, iters / 4, out), d2 = run(dmma_c<2>, sms, bs, iters / 4, out);
    float d4 = run(dmma_c<4>, sms, bs, iters / 4, out), d8 = run(dmma_c<8>, sms, bs, iters / 4, out);
    double fd = 2.0 * 256 * 32 * double(iters / 4) * sms * (bs / 32) / 1e9;
    printf("DMMA warps/SMSP=%d: C1 %.1f  C2 %.1f  C4 %.1f  C8 %.1f TF\n", wps, fd / d1, fd / d2, fd / d4, fd / d8);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
