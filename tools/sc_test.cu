#include <cstdio>
#include <cmath>
#include "/root/repo/paper_2006_15367_b200/csrc/kernels.cuh"
__global__ void k(double* out, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return; double x = -60.0 + 120.0 * i / n; double s, c; hfmm_b200::sincos_fast(x, &s, &c); out[2*i] = s; out[2*i+1] = c; }
int main() { int n = 1 << 20; double* d; cudaMalloc(&d, 16 * n); k<<<n/256, 256>>>(d, n); double* h = new double[2*n]; cudaMemcpy(h, d, 16*n, cudaMemcpyDeviceToHost); double me = 0; for (int i = 0; i < n; ++i) { double x = -60.0 + 120.0 * i / n; me = fmax(me, fmax(fabs(h[2*i] - sin(x)), fabs(h[2*i+1] - cos(x)))); } printf("max abs err %g\n", me); }
