#include <cstdio>
__global__ void probe(double* out) {
  int lane = threadIdx.x;
  double c0 = 0, c1 = 0;
  double a = lane + 1, b = 1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  out[lane * 4] = c0; out[lane * 4 + 1] = c1;
  c0 = 0; c1 = 0; a = 1; b = lane + 1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  out[lane * 4 + 2] = c0; out[lane * 4 + 3] = c1;
}
int main() {
  double* d; cudaMalloc(&d, 128 * 8); probe<<<1, 32>>>(d);
  double h[128]; cudaMemcpy(h, d, 128 * 8, cudaMemcpyDeviceToHost);
  for (int l = 0; l < 32; ++l) printf("lane %2d: Arow-sums %6.0f %6.0f | Bcol-sums %6.0f %6.0f\n", l, h[4*l], h[4*l+1], h[4*l+2], h[4*l+3]);
}
