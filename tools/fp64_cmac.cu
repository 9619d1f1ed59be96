// Register-only throughput of the M2L tap-row pattern (complex MACs with three
// distinct 64-bit operands per DFMA) vs the constant-operand DFMA loop: is the
// stencil's FP64 ceiling the pipe or operand delivery?  (dev tool)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

template <bool INNER>
__device__ __forceinline__ void tap_row(double2 (&acc)[8], const double2 (&m)[12], const double2 (&t)[7]) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int dx = -3; dx <= 3; ++dx) {
      auto fd = [](int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); };
      const int a = fd(k) - fd(k - dx);
      const bool xnear = (a < 0 ? -a : a) <= 1;
      const bool adj = INNER && (dx >= -1 && dx <= 1);
      if (xnear && !adj) cmac(acc[k], t[dx + 3], m[k - dx + 2]);
    }
}

__global__ void __launch_bounds__(128, 3) stencil(double* out, int iters) {
  double2 acc[8], m[12], t[7];
  for (int k = 0; k < 8; ++k) acc[k] = make_double2(0, 0);
  for (int i = 0; i < 12; ++i) m[i] = make_double2(threadIdx.x * 1e-3 + i, i * 1e-2);
  for (int j = 0; j < 7; ++j) t[j] = make_double2(1e-3 * j, -1e-3 * j);
  for (int it = 0; it < iters; ++it) {
    tap_row<false>(acc, m, t);
    // perturb the operands a little so nothing is hoisted
#pragma unroll
    for (int j = 0; j < 7; ++j) t[j].x = fma(t[j].x, 0.999, 1e-9);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 3 * 128);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // count the cmacs of tap_row<false>
  int n = 0;
  for (int k = 0; k < 8; ++k) for (int dx = -3; dx <= 3; ++dx) {
    auto fd = [](int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); };
    int a = fd(k) - fd(k - dx); if ((a < 0 ? -a : a) <= 1) ++n;
  }
  const int iters = 20000, blocks = sms * 3;
  stencil<<<blocks, 128>>>(out, iters);
  cudaEventRecord(e0);
  stencil<<<blocks, 128>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = double(blocks) * 128 * iters * (n * 8.0 + 14);
  printf("tap-row register loop: %d cmacs/row, %.1f TFLOP/s (%.3f ms)\n", n, fl / ms / 1e9, ms);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
