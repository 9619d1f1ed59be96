// Dense linear maps equivalent to the reference's FFT resampling.
//
// resample_circle (/root/reference/proj/src/sphere_grid.cpp:128-155) is linear:
// with n_in samples at (i + s_in) 2pi/n_in and n_out at (j + s_out) 2pi/n_out and
// the asymmetric mode window m in [-K/2, K/2 - 1], K = min(n_in, n_out) (even),
//
//   out[j] = sum_i M[j][i] in[i],
//   M[j][i] = (1/n_in) sum_m exp(2 pi i m ((j + s_out)/n_out - (i + s_in)/n_in)).
//
// The device applies these matrices per theta row (phi pass, shift 0) and per
// folded great circle (theta pass, shift 0.5), which reproduces fft_interpolate
// (:183-192) and fft_anterpolate (:194-204) to roundoff (SURVEY.md §7 hard part 3).
#ifndef HFMM_B200_INTERP_HPP
#define HFMM_B200_INTERP_HPP

#include <cmath>
#include <cstdint>
#include <vector>

namespace hfmm_b200 {

// Row-major n_out x n_in complex matrix (re, im interleaved).  Angles are
// reduced exactly in integer arithmetic and the sum is carried in long
// double, so entries are accurate to ~1 ulp.
inline std::vector<double> resample_matrix(int64_t n_in, double s_in, int64_t n_out,
                                           double s_out) {
  const int64_t K = std::min(n_in, n_out);
  std::vector<double> M(size_t(2 * n_out * n_in));
  // angle = 2 pi m ((2j + 2 s_out) n_in - (2i + 2 s_in) n_out) / (2 n_in n_out)
  const int64_t den = 2 * n_in * n_out;
  const int64_t so2 = int64_t(std::llround(2 * s_out)), si2 = int64_t(std::llround(2 * s_in));
  const int64_t m_lo = (K % 2 == 0) ? -K / 2 : -(K - 1) / 2;
  const int64_t m_hi = (K % 2 == 0) ? K / 2 - 1 : (K - 1) / 2;
  const long double two_pi = 6.283185307179586476925286766559L;
  for (int64_t j = 0; j < n_out; ++j)
    for (int64_t i = 0; i < n_in; ++i) {
      const int64_t num = (2 * j + so2) * n_in - (2 * i + si2) * n_out;
      // Geometric sum of exp(i m t), t = 2 pi num / den, by a long-double
      // rotation recurrence started from the exactly reduced first angle.
      int64_t r0 = (m_lo * num) % den;
      if (r0 < 0) r0 += den;
      int64_t r1 = num % den;
      if (r1 < 0) r1 += den;
      const long double a0 = two_pi * (long double)r0 / (long double)den;
      const long double a1 = two_pi * (long double)r1 / (long double)den;
      long double cr = cosl(a0), ci = sinl(a0);
      const long double sr = cosl(a1), si = sinl(a1);
      long double re = 0, im = 0;
      for (int64_t m = m_lo; m <= m_hi; ++m) {
        re += cr;
        im += ci;
        const long double nr = cr * sr - ci * si;
        ci = cr * si + ci * sr;
        cr = nr;
      }
      M[size_t(2 * (j * n_in + i))] = double(re / (long double)n_in);
      M[size_t(2 * (j * n_in + i) + 1)] = double(im / (long double)n_in);
    }
  return M;
}

}  // namespace hfmm_b200

#endif
