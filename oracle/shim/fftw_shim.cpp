// Mixed-radix FFT behind the FFTW3 API subset the reference uses.
// TEST INFRASTRUCTURE ONLY (oracle/). See fftw3.h for the contract.
//
// Recursive decimation-in-time Cooley-Tukey over the prime factorisation of
// n; each radix-p butterfly is a direct p-point DFT with table twiddles.
// Sizes in the reference are 2L+2 and 2*n_theta (even, small primes up to a
// few hundred), so the cost is O(n * sum(p)) -- within a small factor of
// FFTW_ESTIMATE for these lengths.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

using cd = std::complex<double>;

struct fftw_plan_s {
  int n = 0;
  int sign = -1;
  std::vector<int> factors;
  std::vector<cd> w;  // w[e] = exp(sign * 2 pi i e / n)
  fftw_complex* in = nullptr;
  fftw_complex* out = nullptr;
};

namespace {

void transform(const fftw_plan_s& P, const cd* in, std::size_t stride, cd* out,
               int n, std::size_t fi, cd* scratch) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  int p = P.factors[fi];
  int m = n / p;
  for (int r = 0; r < p; ++r)
    transform(P, in + r * stride, stride * std::size_t(p), out + std::size_t(r) * m, m,
              fi + 1, scratch);
  const std::size_t step_n = std::size_t(P.n / n);  // W_n^e = w[e * step_n]
  const std::size_t step_p = std::size_t(P.n / p);  // W_p^e = w[e * step_p]
  cd* t = scratch;
  for (int k = 0; k < m; ++k) {
    for (int r = 0; r < p; ++r)
      t[r] = out[std::size_t(r) * m + k] * P.w[(std::size_t(r) * k * step_n) % P.n];
    if (p == 2) {
      out[k] = t[0] + t[1];
      out[k + m] = t[0] - t[1];
      continue;
    }
    for (int q = 0; q < p; ++q) {
      cd acc = t[0];
      for (int r = 1; r < p; ++r)
        acc += t[r] * P.w[(std::size_t(r * q) % std::size_t(p)) * step_p];
      t[p + q] = acc;
    }
    for (int q = 0; q < p; ++q) out[k + std::size_t(q) * m] = t[p + q];
  }
}

}  // namespace

extern "C" {

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned) {
  if (n <= 0) return nullptr;
  auto* P = new fftw_plan_s;
  P->n = n;
  P->sign = sign;
  P->in = in;
  P->out = out;
  int v = n;
  for (int f = 2; f * f <= v; ++f)
    while (v % f == 0) {
      P->factors.push_back(f);
      v /= f;
    }
  if (v > 1) P->factors.push_back(v);
  P->w.resize(std::size_t(n));
  for (int e = 0; e < n; ++e) {
    double ang = double(sign) * 2.0 * M_PI * double(e) / double(n);
    P->w[std::size_t(e)] = cd(std::cos(ang), std::sin(ang));
  }
  return P;
}

void fftw_execute_dft(const fftw_plan P, fftw_complex* in, fftw_complex* out) {
  const std::size_t n = std::size_t(P->n);
  int maxp = 2;
  for (int f : P->factors) maxp = f > maxp ? f : maxp;
  thread_local std::vector<cd> src, dst, scratch;
  src.resize(n);
  dst.resize(n);
  scratch.resize(2 * std::size_t(maxp));
  std::memcpy(src.data(), in, n * sizeof(cd));
  transform(*P, src.data(), 1, dst.data(), P->n, 0, scratch.data());
  std::memcpy(out, dst.data(), n * sizeof(cd));
}

void fftw_execute(const fftw_plan P) { fftw_execute_dft(P, P->in, P->out); }

void fftw_destroy_plan(fftw_plan P) { delete P; }

}  // extern "C"
