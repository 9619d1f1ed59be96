// Standalone check of k_m2m_fused for one parent against a CPU restatement.
#include <cstdio>
#include <cstdlib>
#include <complex>
#include <vector>
#include "../paper_2006_15367_b200/csrc/interp.hpp"
#include "../paper_2006_15367_b200/csrc/interp_tc.cuh"
using namespace hfmm_b200;
using cd = std::complex<double>;
int lda_for(int K) { return (K % 8 == 4) ? K : K + 4; }
template <class T> T* up(const std::vector<T>& v) { T* d; cudaMalloc(&d, v.size() * sizeof(T) + 16); cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice); return d; }
int main(int argc, char** argv) {
  const int nc = 18, np = 28, half = np / 2, Sc = nc * nc, Sp = np * np, npar = 216, nch = 8 * npar;
  const int CB = argc > 1 ? atoi(argv[1]) : 4;
  RealRank1 a = real_rank1(nc, 0.0, np, 0.0), b = real_rank1(2 * nc, 0.5, 2 * np, 0.5);
  PassDims phi{a.K, a.N, lda_for(a.K), 0}, th{b.K, b.N, lda_for(b.K), b.N + 4};
  std::vector<double2> X(nch * Sc), sh(8 * Sp, make_double2(1, 0));
  srand(3);
  for (auto& x : X) x = make_double2(rand() / double(RAND_MAX) - .5, rand() / double(RAND_MAX) - .5);
  std::vector<int> coff(npar + 1), ch(nch);
  for (int i = 0; i <= npar; ++i) coff[i] = 8 * i;
  std::vector<uint8_t> oct(nch);
  for (int i = 0; i < nch; ++i) { ch[i] = i; oct[i] = i % 8; }
  // CPU: sum over children of interp (dense complex matrices)
  auto P = resample_matrix(nc, 0, np, 0), T = resample_matrix(2 * nc, .5, 2 * np, .5);
  std::vector<cd> ref(size_t(npar) * Sp, 0);
  for (int c = 0; c < nch; ++c) {
    std::vector<cd> W(nc * np), F(half * 2 * nc), G(half * 2 * np);
    for (int i = 0; i < nc; ++i) for (int j = 0; j < np; ++j) { cd s = 0; for (int k = 0; k < nc; ++k) s += cd(P[2*(j*nc+k)], P[2*(j*nc+k)+1]) * cd(X[c*Sc+i*nc+k].x, X[c*Sc+i*nc+k].y); W[i*np+j] = s; }
    for (int p = 0; p < half; ++p) for (int i = 0; i < 2*nc; ++i) F[p*2*nc+i] = i < nc ? W[i*np+p] : W[(2*nc-1-i)*np+p+half];
    for (int p = 0; p < half; ++p) for (int j = 0; j < 2*np; ++j) { cd s = 0; for (int i = 0; i < 2*nc; ++i) s += cd(T[2*(j*2*nc+i)], T[2*(j*2*nc+i)+1]) * F[p*2*nc+i]; G[p*2*np+j] = s; }
    for (int p = 0; p < half; ++p) for (int j = 0; j < 2*np; ++j) { int s = j < np ? j*np+p : (2*np-1-j)*np+p+half; ref[size_t(c / 8) * Sp + s] += G[p*2*np+j]; }
  }
  double2* dX = up(X); double2* dsh = up(sh); int* dco = up(coff); int* dch = up(ch); uint8_t* doc = up(oct);
  double *dA = up(a.B), *dva = up(a.v), *dB = up(b.B), *dvb = up(b.v);
  double2* dout; cudaMalloc(&dout, size_t(npar) * Sp * 16);
  size_t xs = size_t(CB) * nc * phi.lda, gs = size_t(CB) * half * th.ldo;
  size_t smem = (std::max(xs, gs) + size_t(CB) * half * th.lda) * 16;
  cudaFuncSetAttribute(k_m2m_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_m2m_fused<<<npar, kFusedThreads, smem>>>(nc, np, CB, phi, th, dco, dch, doc, dX, dout, dA, dva, dB, dvb, dsh);
  std::vector<double2> out(size_t(npar) * Sp);
  cudaMemcpy(out.data(), dout, out.size() * 16, cudaMemcpyDeviceToHost);
  printf("CB=%d smem=%zu err=%s\n", CB, smem, cudaGetErrorString(cudaGetLastError()));
  double mx = 0, nr = 0; int bad = 0;
  for (int s = 0; s < npar * Sp; ++s) { double d = std::abs(cd(out[s].x, out[s].y) - ref[s]); mx = std::max(mx, d); nr = std::max(nr, std::abs(ref[s])); if (d > 1e-10 && bad++ < 8) printf("bad par=%d row=%d col=%d\n", s/Sp, (s%Sp)/np, s%np); }
  printf("max err %g (max |ref| %g) bad %d\n", mx, nr, bad);
}
