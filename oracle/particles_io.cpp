// Runs the reference's particle-file I/O (geometry.cpp:128-159) out of
// process (its iostreams clash with the Python process's C++ runtime).
// TEST INFRASTRUCTURE for tests/test_io.py:
//   particles_io write <raw.bin> <out.txt> <header>   raw = u64 n, n*3 xyz, n*2 q (f64)
//   particles_io read  <in.txt>  <raw.bin>            exit 2 + message on parse errors
#include <cstdint>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "hfmm/geometry.hpp"

int main(int argc, char** argv) {
  if (argc < 4) return 1;
  const std::string cmd = argv[1];
  try {
    if (cmd == "write") {
      FILE* f = std::fopen(argv[2], "rb");
      if (!f) return 1;
      uint64_t n = 0;
      if (std::fread(&n, 8, 1, f) != 1) return 1;
      std::vector<double> xyz(3 * n), q(2 * n);
      if (std::fread(xyz.data(), 8, 3 * n, f) != 3 * n || std::fread(q.data(), 8, 2 * n, f) != 2 * n) return 1;
      std::fclose(f);
      std::vector<hfmm::Particle> p(n);
      for (uint64_t i = 0; i < n; ++i) {
        p[i].position = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
        p[i].intensity = {q[2 * i], q[2 * i + 1]};
      }
      hfmm::write_particles(argv[3], p, argc > 4 ? argv[4] : "");
      return 0;
    }
    if (cmd == "read") {
      const auto p = hfmm::read_particles(argv[2]);
      FILE* f = std::fopen(argv[3], "wb");
      if (!f) return 1;
      const uint64_t n = p.size();
      std::fwrite(&n, 8, 1, f);
      for (const auto& e : p) std::fwrite(&e.position.x, 8, 3, f);
      for (const auto& e : p) {
        const double c[2] = {e.intensity.real(), e.intensity.imag()};
        std::fwrite(c, 8, 2, f);
      }
      std::fclose(f);
      return 0;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  }
  return 1;
}
