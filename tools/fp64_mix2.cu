// FP64 pipe probe: DMMA.8x8x4 with DADDs mixed in (the 3-multiplication M2L's
// instruction mix: 5 DADD per 12 DMMA), by resident warps per SM sub-partition.
// Reports the DMMA rate as a fraction of the pure-DMMA peak (dev tool).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// MODE 0: 12 DMMA; 1: + 5 dependent DADD (results feed 4 DMMA b operands and 1 a operand);
// 2: + 5 DADD whose results are used one group later; 3: + 5 DFMA independent of the DMMA
template <int MODE>
__global__ void k(double* out, int iters) {
  double c[12][2];
  for (int t = 0; t < 12; ++t) c[t][0] = c[t][1] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = 1.0 - threadIdx.x * 1e-4, b[4], bi[4], bs[4], as = a0 + a1, x = 1e-9;
  for (int t = 0; t < 4; ++t) { b[t] = 0.5 + t * 1e-3; bi[t] = 0.25 - t * 1e-3; bs[t] = b[t] + bi[t]; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (MODE == 1) {
        as = a0 + a1;
#pragma unroll
        for (int t = 0; t < 4; ++t) bs[t] = b[t] + bi[t];
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        dmma(c[t][0], c[t][1], a0, b[t]);
        dmma(c[4 + t][0], c[4 + t][1], a1, bi[t]);
        dmma(c[8 + t][0], c[8 + t][1], as, bs[t]);
      }
      if (MODE == 2) {
        as = a0 + a1;
#pragma unroll
        for (int t = 0; t < 4; ++t) bs[t] = b[t] + bi[t];
      }
      if (MODE == 3) {
#pragma unroll
        for (int t = 0; t < 5; ++t) x = fma(x, 0.999999, 1e-7);
      }
      if (MODE == 1 || MODE == 2) {  // operands change on the integer pipe, so the DADDs are not hoisted
        a0 = __longlong_as_double(__double_as_longlong(a0) ^ (long long)(r + 1));
#pragma unroll
        for (int t = 0; t < 4; ++t) b[t] = __longlong_as_double(__double_as_longlong(b[t]) ^ (long long)(r + 1));
      }
    }
  }
  double s = x + as;
  for (int t = 0; t < 12; ++t) s += c[t][0] + c[t][1];
  for (int t = 0; t < 4; ++t) s += bs[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
float run(K kern, int blocks, int bs, int iters, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, bs>>>(out, iters);
  cudaEventRecord(e0);
  kern<<<blocks, bs>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 2048);
  const int iters = 4096;
  for (int wps : {1, 2, 3, 4}) {
    const int bs = 128 * wps;
    const double dm = double(sms) * (bs / 32) * iters * 8.0 * 12.0;  // DMMA count
    float m0 = run(k<0>, sms, bs, iters, out), m1 = run(k<1>, sms, bs, iters, out);
    float m2 = run(k<2>, sms, bs, iters, out), m3 = run(k<3>, sms, bs, iters, out);
    auto tf = [&](float ms) { return dm * 512.0 / (ms * 1e-3) / 1e12; };
    printf("warps/SMSP %d: DMMA TFLOP/s  pure %.2f | +5 DADD feeding %.2f | +5 DADD one group ahead %.2f | +5 indep DFMA %.2f\n",
           wps, tf(m0), tf(m1), tf(m2), tf(m3));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
