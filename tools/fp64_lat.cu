// Dependent-issue latency probe (one warp on one SM): DFMA, DADD, DMMA.8x8x4 (accumulator
// chain), SHFL + DADD, LDS.64 + DFMA; clock64 around an unrolled chain (dev tool).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k(double* out, long long* clk) {
  __shared__ double sm[64];
  sm[threadIdx.x] = 1.0 + threadIdx.x * 1e-9;
  sm[threadIdx.x + 32] = 0.5;
  __syncthreads();
  double x = threadIdx.x * 1e-3 + 1.0, b = 0.999999, c = 1e-7;
  const int N = 256;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fma(x, b, c);
  long long t1 = clock64();
  double y = x;
#pragma unroll
  for (int i = 0; i < N; ++i) y = y + c;
  long long t2 = clock64();
  double c0 = y, c1 = x;
#pragma unroll
  for (int i = 0; i < N; ++i) dmma(c0, c1, b, c);
  long long t3 = clock64();
  double s = c0;
#pragma unroll
  for (int i = 0; i < N; ++i) s = s + __shfl_xor_sync(0xffffffffu, s, 1);
  long long t4 = clock64();
  double w = s * 1e-300;
  int idx = threadIdx.x;
#pragma unroll
  for (int i = 0; i < N; ++i) { w = fma(sm[idx], b, w); idx = (idx + (w > 1e300)) & 63; }
  long long t5 = clock64();
  // two independent DFMA chains (issue-limited pair)
  double p = w + 1.0, q2 = w + 2.0;
#pragma unroll
  for (int i = 0; i < N; ++i) { p = fma(p, b, c); q2 = fma(q2, b, c); }
  long long t6 = clock64();
  out[threadIdx.x] = x + y + c0 + c1 + s + w + p + q2;
  if (threadIdx.x == 0) {
    clk[0] = (t1 - t0); clk[1] = (t2 - t1); clk[2] = (t3 - t2); clk[3] = (t4 - t3); clk[4] = (t5 - t4); clk[5] = (t6 - t5);
  }
}

int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 32 * 8); cudaMalloc(&clk, 6 * 8);
  k<<<1, 32>>>(out, clk);
  k<<<1, 32>>>(out, clk);
  long long h[6];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  const double N = 256;
  printf("clocks per dependent op (1 warp): DFMA %.1f | DADD %.1f | DMMA (accumulator chain) %.1f | SHFL+DADD %.1f | LDS.64+DFMA(acc) %.1f | 2 indep DFMA chains, per pair %.1f\n",
         h[0] / N, h[1] / N, h[2] / N, h[3] / N, h[4] / N, h[5] / N);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
