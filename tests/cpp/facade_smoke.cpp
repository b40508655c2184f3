// facade_smoke.cpp -- exercises include/xpcs_b200.hpp from C++ (built by
// __graft_entry__.build(), run by tests/test_gpu_facade.py on the GPU box).
// Reads a u8 frame file (n x m) and a ring map (m int32), prints the int
// Gram diagonal checksum, the f64 TTC checksum and g2[0..2] of every ring.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "xpcs_b200.hpp"

int main(int argc, char** argv) {
  if (argc != 6) {
    std::fprintf(stderr, "usage: %s frames.u8 ring.i32 n m q\n", argv[0]);
    return 2;
  }
  const int64_t n = std::atoll(argv[3]), m = std::atoll(argv[4]);
  const int q = std::atoi(argv[5]);
  std::vector<uint8_t> frames(static_cast<size_t>(n * m));
  std::vector<int32_t> ring(static_cast<size_t>(m));
  std::ifstream(argv[1], std::ios::binary).read(reinterpret_cast<char*>(frames.data()), n * m);
  std::ifstream(argv[2], std::ios::binary).read(reinterpret_cast<char*>(ring.data()), m * 4);
  try {
    xpcs_b200::Context ctx(0);
    std::vector<std::vector<int64_t>> masks(q);
    for (int64_t p = 0; p < m; ++p) masks[ring[p]].push_back(p);
    xpcs_b200::RingLayout layout(ctx, m, masks);
    xpcs_b200::Series s(layout, n);
    s.load(frames.data(), n);
    s.ttc_raw();
    for (int r = 0; r < q; ++r) {
      const auto c = s.ttc(r);
      double sum = 0.0;
      for (double v : c) sum += v;
      const auto g2 = s.g2(r);
      std::printf("ring %d sum %.17g g2 %.17g %.17g %.17g\n", r, sum, g2[0], g2[1], g2[2]);
    }
    // device basis, compressed TTC, analysis and formats through the facade
    {
      xpcs_b200::Basis b(layout, 4);
      const auto rank = s.build_basis(4, &b);
      s.compress(b);
      s.ttc_compressed();
      const auto bg = s.ttc_background(2);
      const auto fits = s.fit_kww(1.0, 1.0, static_cast<double>(n / 2));
      std::printf("basis rank %lld bg %.6g fit status %d\n", (long long)rank[0], bg[0], fits[0].status);
      s.write_xcmp(0, "/tmp/facade_r0.xcmp", 42);
      s.write_ttc(0, "/tmp/facade_r0.xttc", XG_I32_GRAM);
      xpcs_b200::Series s3(layout, n);
      s3.load_xfsr("/tmp/facade_frames.xfsr");  // written by the test (u8 XFSR)
      s3.ttc_raw();
      std::printf("xfsr load %s\n", s3.ttc(0) == s.ttc(0) ? "equal" : "DIFFERENT");
    }
    // reference-facing exact entry on the same ring 0 data
    std::vector<double> x0;
    for (int64_t t = 0; t < n; ++t)
      for (int64_t p : masks[0]) x0.push_back(frames[t * m + p]);
    const auto g = xpcs_b200::ttc_raw(x0, n, static_cast<int64_t>(masks[0].size()));
    double sum = 0.0;
    for (double v : g) sum += v;
    std::printf("exact ring 0 sum %.17g\n", sum);
    // f64 intensities: integral counts load through the u8 path (same C)
    {
      std::vector<double> fd(frames.begin(), frames.end());
      xpcs_b200::Series s2(layout, n);
      s2.load(fd.data(), n, m);
      s2.ttc_raw();
      const auto c0 = s2.ttc(0), c1 = s.ttc(0);
      std::printf("f64 load %s\n", c0 == c1 ? "equal" : "DIFFERENT");
      fd[3] = 1.5;
      try {
        s2.load(fd.data(), n, m);
        std::printf("missing ContractError\n");
        return 1;
      } catch (const xpcs_b200::ContractError&) {
        std::printf("ContractError non-integer\n");
      }
    }
    try {
      std::vector<double> z(static_cast<size_t>(3 * 4), 1.0);
      for (int p = 0; p < 4; ++p) z[4 + p] = 0.0;
      xpcs_b200::ttc_raw(z, 3, 4);
      std::printf("missing NormalizationError\n");
      return 1;
    } catch (const xpcs_b200::NormalizationError& e) {
      std::printf("NormalizationError frame %zu\n", e.frame_index());
    }
    // round-2 entries: a split ring summed from two half-shares equals the
    // whole ring's Gram; the batch push equals n single pushes
    {
      const auto& m0 = masks[0];
      const size_t half = m0.size() / 2;
      std::vector<std::vector<int64_t>> ma{std::vector<int64_t>(m0.begin(), m0.begin() + half)};
      std::vector<std::vector<int64_t>> mb{std::vector<int64_t>(m0.begin() + half, m0.end())};
      xpcs_b200::RingLayout la(ctx, m, ma), lb(ctx, m, mb);
      xpcs_b200::Series sa(la, n), sb(lb, n);
      sa.load(frames.data(), n);
      sb.load(frames.data(), n);
      sa.ttc_raw();
      sb.ttc_raw();
      auto pa = sa.export_partial(0);
      const auto pb = sb.export_partial(0);
      for (size_t i = 0; i < pa.gram.size(); ++i) pa.gram[i] += pb.gram[i];
      for (size_t i = 0; i < pa.norm2.size(); ++i) pa.norm2[i] += pb.norm2[i];
      sa.import_partial(0, pa);
      std::printf("split ring %s\n", sa.gram(0) == s.gram(0) ? "equal" : "DIFFERENT");
      xpcs_b200::Stream st1(layout, n), st2(layout, n);
      for (int64_t t = 0; t < n; ++t) st1.push(frames.data() + t * m);
      st2.push_batch(frames.data(), n);
      std::printf("push batch %s\n", st1.g2(0) == st2.g2(0) ? "equal" : "DIFFERENT");
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
