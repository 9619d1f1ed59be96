// Frozen seeded input generator for the BASELINE configurations.
//
// The reference has no random-cube / random-sphere generator (its generators
// are lattices and a Fibonacci sphere, /root/reference/proj/src/geometry.cpp:75-127),
// so this recipe is the single definition shared by the
// product library (bench inputs) and the oracle driver (reference inputs).
// Both are built by the same g++/libstdc++, so std::uniform_real_distribution
// produces identical bits on both sides.
//
//   rng = std::mt19937_64(seed)
//   positions first, one statement per draw (no argument-order ambiguity):
//     cube:   x = U*side; y = U*side; z = U*side
//     sphere: z = 2U-1; phi = 2 pi U; rho = sqrt(max(0, 1-z^2));
//             p = (R + R rho cos phi, R + R rho sin phi, R + R z)
//   then charges: re = U(-1,1); im = U(-1,1)
#ifndef HFMM_B200_INPUTS_HPP
#define HFMM_B200_INPUTS_HPP

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <random>

namespace hfmm_b200 {

enum InputShape { kShapeCube = 0, kShapeSphere = 1 };

// xyz: n*3 doubles (AoS), q: n*2 doubles (re, im).
inline void generate_inputs(int shape, std::size_t n, double extent,
                            std::uint64_t seed, double* xyz, double* q) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  std::uniform_real_distribution<double> u11(-1.0, 1.0);
  for (std::size_t i = 0; i < n; ++i) {
    if (shape == kShapeCube) {
      double x = u01(rng) * extent;
      double y = u01(rng) * extent;
      double z = u01(rng) * extent;
      xyz[3 * i] = x;
      xyz[3 * i + 1] = y;
      xyz[3 * i + 2] = z;
    } else {
      const double R = extent;
      double z = 2.0 * u01(rng) - 1.0;
      double ph = 2.0 * M_PI * u01(rng);
      double rho = std::sqrt(std::max(0.0, 1.0 - z * z));
      xyz[3 * i] = R + R * rho * std::cos(ph);
      xyz[3 * i + 1] = R + R * rho * std::sin(ph);
      xyz[3 * i + 2] = R + R * z;
    }
  }
  for (std::size_t i = 0; i < n; ++i) {
    double re = u11(rng);
    double im = u11(rng);
    q[2 * i] = re;
    q[2 * i + 1] = im;
  }
}

}  // namespace hfmm_b200

#endif
