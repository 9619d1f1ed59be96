// Standalone check of warp_gemm_rc (DMMA fragment layout) against a CPU GEMM.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2006_15367_b200/csrc/interp_tc.cuh"
using namespace hfmm_b200;

__global__ void kern(int M, int N, int K, const double2* A, int lda, const double* B, double* C) {
  extern __shared__ double2 sm[];
  for (int t = threadIdx.x; t < (M / 2 + 1) * lda; t += blockDim.x) sm[t] = A[t];
  __syncthreads();
  warp_gemm_rc(M, N, K, sm, lda, B, [&](int r, int n, double v) { C[r * N + n] = v; });
}

int main() {
  int M = 36, N = 40, K = 20, lda = 20;
  std::vector<double2> A((M / 2 + 1) * lda);
  std::vector<double> B(K * N), C(M * N, -1), R(M * N, 0);
  srand(1);
  for (auto& a : A) a = make_double2(rand() / double(RAND_MAX) - .5, rand() / double(RAND_MAX) - .5);
  for (auto& b : B) b = rand() / double(RAND_MAX) - .5;
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) {
        double a = (r & 1) ? A[(r >> 1) * lda + k].y : A[(r >> 1) * lda + k].x;
        s += a * B[k * N + n];
      }
      R[r * N + n] = s;
    }
  double2* dA; double *dB, *dC;
  cudaMalloc(&dA, A.size() * 16); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
  kern<<<1, 256, A.size() * 16>>>(M, N, K, dA, lda, dB, dC);
  cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  double mx = 0; int bad = 0;
  for (int i = 0; i < M * N; ++i) { double d = fabs(C[i] - R[i]); if (d > 1e-12) { if (0) printf("bad r=%d n=%d got %f want %f\n", i / N, i % N, C[i], R[i]); ++bad; } mx = fmax(mx, d); }
  printf("max err %g bad %d\n", mx, bad);
  for (int r = 0; r < M; ++r) { int nb = 0; for (int n = 0; n < N; ++n) nb += fabs(C[r*N+n]-R[r*N+n]) > 1e-12; printf("r%d:%d ", r, nb); } printf("\n");
  for (int n = 0; n < N; ++n) printf("%.2f/%.2f ", C[2*N+n], R[2*N+n]); printf("\n");
}
