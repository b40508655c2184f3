// dropin_bench.cpp -- times the reference's own API entry xpcs::ttc_raw +
// xpcs::g2_from_ttc (correlate.hpp:10,26) as a reference program would call
// it, linked against integration/correlate_b200.cpp (the B200 drop-in).
// Built by `make -C oracle acceptance` next to the acceptance binaries (it
// links reference sources, so it lives in oracle/_ref, git-ignored).
// Usage: dropin_bench frames.u8 n m reps  -> one JSON line.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "xpcsvd/correlate.hpp"

int main(int argc, char** argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: %s frames.u8 n m reps\n", argv[0]);
    return 2;
  }
  const std::size_t n = std::strtoull(argv[2], nullptr, 10), m = std::strtoull(argv[3], nullptr, 10);
  const int reps = std::atoi(argv[4]);
  std::vector<unsigned char> u8(n * m);
  std::ifstream(argv[1], std::ios::binary).read(reinterpret_cast<char*>(u8.data()), n * m);
  xpcs::Matrix x(n, m);
  for (std::size_t i = 0; i < n * m; ++i) x.data()[i] = u8[i];
  xpcs::FrameSeries fs(std::move(x), 1.0);
  double best = 1e30, sum = 0.0, chk = 0.0;
  for (int r = 0; r < reps + 1; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    const xpcs::TTCMatrix g = xpcs::ttc_raw(fs);
    const xpcs::G2Curve c = xpcs::g2_from_ttc(g, 1.0);
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (r > 0) {  // the first call creates the context and buffers
      best = dt < best ? dt : best;
      sum += dt;
    }
    chk = c.values[1];
  }
  std::printf("{\"ms_best\": %.4f, \"ms_mean\": %.4f, \"g2_1\": %.17g}\n", best * 1e3,
              sum / reps * 1e3, chk);
  return 0;
}
