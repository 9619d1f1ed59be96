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

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
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

// Real + rank-1 split of a resampling map, M = R + i u v^T, laid out as the
// B operand of the fused tensor-core passes: B is (K x N) row-major with
// B[k][n] = R[n][k] (k < n_in), B[n_in][n] = u[n], zero padding elsewhere;
// K = round_up(n_in + 1, 4), N = round_up(n_out, 8).  row_scale / col_scale
// (optional, length n_out / n_in) multiply M from the left / right.
struct RealRank1 {
  int K = 0, N = 0;
  std::vector<double> B;  // K*N
  std::vector<double> v;  // n_in
};

inline RealRank1 real_rank1(int64_t n_in, double s_in, int64_t n_out, double s_out,
                            const std::vector<double>* row_scale = nullptr,
                            const std::vector<double>* col_scale = nullptr) {
  const std::vector<double> M = resample_matrix(n_in, s_in, n_out, s_out);
  const int64_t Kw = std::min(n_in, n_out);
  const long double pi = 3.141592653589793238462643383279503L;
  // Im(M)[j][i] = -(1/n_in) sin(K pi (a_j - b_i)) = u1_j v1_i + u2_j v2_i
  std::vector<long double> u1(static_cast<size_t>(n_out)), u2(static_cast<size_t>(n_out)), v1(static_cast<size_t>(n_in)), v2(static_cast<size_t>(n_in));
  for (int64_t j = 0; j < n_out; ++j) {
    const long double a = ((long double)j + s_out) / (long double)n_out;
    u1[size_t(j)] = -sinl(Kw * pi * a) / (long double)n_in;
    u2[size_t(j)] = cosl(Kw * pi * a) / (long double)n_in;
  }
  for (int64_t i = 0; i < n_in; ++i) {
    const long double b = ((long double)i + s_in) / (long double)n_in;
    v1[size_t(i)] = cosl(Kw * pi * b);
    v2[size_t(i)] = sinl(Kw * pi * b);
  }
  auto amax = [](const std::vector<long double>& x) {
    long double m = 0;
    for (auto e : x) m = std::max(m, e < 0 ? -e : e);
    return m;
  };
  const bool use1 = amax(u1) * amax(v1) >= amax(u2) * amax(v2);
  const std::vector<long double>& u = use1 ? u1 : u2;
  const std::vector<long double>& v = use1 ? v1 : v2;
  if ((use1 ? amax(u2) * amax(v2) : amax(u1) * amax(v1)) > 1e-13L)
    throw std::logic_error("real_rank1: imaginary part is not rank one");
  RealRank1 out;
  out.K = int((n_in + 1 + 3) / 4 * 4);
  out.N = int((n_out + 7) / 8 * 8);
  out.B.assign(size_t(out.K) * size_t(out.N), 0.0);
  out.v.resize(size_t(n_in));
  for (int64_t j = 0; j < n_out; ++j) {
    const double rs = row_scale ? (*row_scale)[size_t(j)] : 1.0;
    for (int64_t i = 0; i < n_in; ++i) {
      const double cs = col_scale ? (*col_scale)[size_t(i)] : 1.0;
      const double re = M[size_t(2 * (j * n_in + i))];
      const double im = M[size_t(2 * (j * n_in + i) + 1)];
      if (std::fabs(im - double(u[size_t(j)] * v[size_t(i)])) > 1e-14)
        throw std::logic_error("real_rank1: rank-one factors do not reproduce the map");
      out.B[size_t(i) * out.N + size_t(j)] = rs * re * cs;
    }
    out.B[size_t(n_in) * out.N + size_t(j)] = rs * double(u[size_t(j)]);
  }
  for (int64_t i = 0; i < n_in; ++i)
    out.v[size_t(i)] = double(v[size_t(i)]) * (col_scale ? (*col_scale)[size_t(i)] : 1.0);
  return out;
}

// ---------------------------------------------------------------------------
// Even / odd halving of the theta passes.
//
// The theta pass resamples a folded great circle of n_in = 2 n_c points at
// (i + 1/2) 2 pi / n_in to n_out = 2 n_p points.  Both point sets are symmetric
// under t -> -t (i <-> n_in - 1 - i, j <-> n_out - 1 - j) and the kernel is a
// function of the angle difference with an even real part, so the real matrix
// is centrosymmetric: R[J j][J i] = R[j][i].  With x_e = x + J x and
// x_o = x - J x (first halves),
//     y[j]   = Ye[j] + Yo[j],      Ye = Be x_e,  Be[j][i] = (R[j][i] + R[j][J i]) / 2,
//     y[J j] = Ye[j] - Yo[j],      Yo = Bo x_o,  Bo[j][i] = (R[j][i] - R[j][J i]) / 2,
// for j < n_out / 2: two half-size products, half the multiply-adds.  The
// rank-1 part i u (v . x) splits the same way (u into its symmetric and
// antisymmetric parts, v . x into v_e . x_e + v_o . x_o).
//
// Layout (B operand of the DMMA passes): B is (2 KH4) x NH row-major,
// KH4 = round_up(n_in / 2 + 1, 4), NH = round_up(n_out / 2, 8): rows [0, KH4)
// hold Be (row n_in / 2 = symmetric part of u), rows [KH4, 2 KH4) hold Bo
// (row KH4 + n_in / 2 = antisymmetric part of u); v has 2 KH4 entries, laid
// out like the rows.
struct EvenOdd {
  int KH4 = 0, NH = 0;
  std::vector<double> B;  // 2 KH4 x NH
  std::vector<double> v;  // 2 KH4
};

inline EvenOdd even_odd(const RealRank1& m, int64_t n_in, int64_t n_out) {
  if (n_in % 2 || n_out % 2) throw std::logic_error("even_odd: odd circle length");
  const int64_t hi = n_in / 2, ho = n_out / 2;
  auto Bm = [&](int64_t k, int64_t n) { return m.B[size_t(k) * size_t(m.N) + size_t(n)]; };
  double amax = 0;
  for (int64_t k = 0; k < n_in; ++k)
    for (int64_t n = 0; n < n_out; ++n) amax = std::max(amax, std::fabs(Bm(k, n)));
  for (int64_t k = 0; k < n_in; ++k)
    for (int64_t n = 0; n < n_out; ++n)
      if (std::fabs(Bm(k, n) - Bm(n_in - 1 - k, n_out - 1 - n)) > 1e-13 * amax)
        throw std::logic_error("even_odd: the theta map is not centrosymmetric");
  EvenOdd out;
  out.KH4 = int((hi + 1 + 3) / 4 * 4);
  out.NH = int((ho + 7) / 8 * 8);
  out.B.assign(size_t(2 * out.KH4) * size_t(out.NH), 0.0);
  out.v.assign(size_t(2 * out.KH4), 0.0);
  for (int64_t n = 0; n < ho; ++n) {
    for (int64_t k = 0; k < hi; ++k) {
      out.B[size_t(k) * out.NH + size_t(n)] = 0.5 * (Bm(k, n) + Bm(n_in - 1 - k, n));
      out.B[size_t(out.KH4 + k) * out.NH + size_t(n)] = 0.5 * (Bm(k, n) - Bm(n_in - 1 - k, n));
    }
    out.B[size_t(hi) * out.NH + size_t(n)] = 0.5 * (Bm(n_in, n) + Bm(n_in, n_out - 1 - n));
    out.B[size_t(out.KH4 + hi) * out.NH + size_t(n)] = 0.5 * (Bm(n_in, n) - Bm(n_in, n_out - 1 - n));
  }
  for (int64_t k = 0; k < hi; ++k) {
    out.v[size_t(k)] = 0.5 * (m.v[size_t(k)] + m.v[size_t(n_in - 1 - k)]);
    out.v[size_t(out.KH4 + k)] = 0.5 * (m.v[size_t(k)] - m.v[size_t(n_in - 1 - k)]);
  }
  return out;
}

// M2M phi pass with the fold into (x_e, x_o) baked into its output columns:
// column 2 p + h of the result is column p of M plus (h = 0) or minus (h = 1)
// column p + n_out / 2 -- the two phi samples that land on circle p's
// positions i and J i.  Same K, N as the plain map.
inline RealRank1 fold_columns(const RealRank1& m, int64_t n_in, int64_t n_out) {
  RealRank1 out = m;
  const int64_t half = n_out / 2;
  for (int64_t k = 0; k <= n_in; ++k)
    for (int64_t p = 0; p < half; ++p) {
      const double a = m.B[size_t(k) * m.N + size_t(p)], b = m.B[size_t(k) * m.N + size_t(p + half)];
      out.B[size_t(k) * m.N + size_t(2 * p)] = a + b;
      out.B[size_t(k) * m.N + size_t(2 * p + 1)] = a - b;
    }
  return out;
}

// L2L phi pass reading (Ye, Yo) pairs: input column 2 p + h stands for
// Ye_p (h = 0) or Yo_p (h = 1), where the plain inputs are x[p] = Ye + Yo and
// x[p + n_in / 2] = Ye - Yo; rows of B and entries of v combine accordingly.
inline RealRank1 unfold_rows(const RealRank1& m, int64_t n_in, int64_t n_out) {
  RealRank1 out = m;
  const int64_t half = n_in / 2;
  (void)n_out;
  for (int64_t p = 0; p < half; ++p) {
    for (int64_t n = 0; n < m.N; ++n) {
      const double a = m.B[size_t(p) * m.N + size_t(n)], b = m.B[size_t(p + half) * m.N + size_t(n)];
      out.B[size_t(2 * p) * m.N + size_t(n)] = a + b;
      out.B[size_t(2 * p + 1) * m.N + size_t(n)] = a - b;
    }
    out.v[size_t(2 * p)] = m.v[size_t(p)] + m.v[size_t(p + half)];
    out.v[size_t(2 * p + 1)] = m.v[size_t(p)] - m.v[size_t(p + half)];
  }
  return out;
}

}  // namespace hfmm_b200

#endif
