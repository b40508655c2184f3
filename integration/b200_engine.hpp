// b200_engine.hpp -- shared state of the drop-in xpcs:: sources
// (integration/correlate_b200.cpp, integration/compress_b200.cpp): one
// process-wide B200 context, and the photon-count fast path of ttc_raw.
//
// Routing of xpcs::ttc_raw(const FrameSeries&) (correlate.hpp:10):
//   * intensities that are integer photon counts in [0, 255] (what an XPCS
//     detector delivers; the reference's f64 carries them exactly) go through
//     the u8 tensor-core path: ring permutation (K1), exact u8 x u8 -> int32
//     Gram (K2), f64 normalisation on readback.  The integer Gram equals the
//     reference's gram(counts) bitwise; C is within ~1e-13 of the reference's
//     gram(row_normalize(X)) (SURVEY finding 3; the reference's own oracle
//     tolerance is 1e-12, test_correlate.cpp:43);
//   * anything else -- and every call when XPCS_B200_EXACT=1 -- runs the
//     reference-order f64 replica (xg_f64_ttc_raw), which returns the
//     reference's bits.
// The context is created on first use (device XPCS_B200_DEVICE, default 0)
// and guarded by a mutex: the reference's functions may be called from
// several threads; the GPU work is serialised.
#ifndef XPCS_B200_ENGINE_HPP_
#define XPCS_B200_ENGINE_HPP_

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "xpcs_b200.h"

namespace xpcs_b200_dropin {

inline bool exact_only() {
  static const bool v = [] {
    const char* e = std::getenv("XPCS_B200_EXACT");
    return e && e[0] == '1';
  }();
  return v;
}

// True when every value is an integer count in [0, 255]; packs them to u8.
// Branch-free per element (the range and integrality test folded into one
// flag, so the loop vectorises) over contiguous slices on XPCS_THREADS (the
// reference's own thread knob, linalg.cpp:62-91) or all hardware threads.
inline bool pack_counts(const double* x, std::size_t n, std::vector<uint8_t>& out) {
  out.resize(n);
  auto slice = [x, &out](std::size_t lo, std::size_t hi) {
    bool ok = true;
    uint8_t* o = out.data();
    for (std::size_t i = lo; i < hi; ++i) {
      const double v = x[i];
      const double c = v >= 0.0 && v <= 255.0 ? v : 0.0;
      const uint8_t b = static_cast<uint8_t>(static_cast<int>(c));
      ok &= (static_cast<double>(b) == v);  // NaN, out of range, fractional -> false
      o[i] = b;
    }
    return ok;
  };
  unsigned nt = std::thread::hardware_concurrency();
  if (const char* e = std::getenv("XPCS_THREADS")) nt = static_cast<unsigned>(std::atoi(e));
  nt = std::max(1u, std::min<unsigned>(nt ? nt : 1u, static_cast<unsigned>(n / (1u << 20) + 1)));
  if (nt == 1) return slice(0, n);
  std::vector<char> ok(nt, 0);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&, t] { ok[t] = slice(n * t / nt, n * (t + 1) / nt) ? 1 : 0; });
  for (auto& th : pool) th.join();
  for (char v : ok)
    if (!v) return false;
  return true;
}

struct Engine {
  std::mutex mu;
  xg_ctx* ctx = nullptr;
  int ctx_rc = -1;
  xg_layout* layout = nullptr;  // one ring = every pixel of the series
  int64_t layout_m = -1;
  xg_series* series = nullptr;
  int64_t series_n = -1;

  // 0 = ready; else an xg_status (no device, ...)
  int ensure(int64_t n, int64_t m) {
    if (!ctx) {
      const char* d = std::getenv("XPCS_B200_DEVICE");
      ctx_rc = xg_ctx_create(d ? std::atoi(d) : 0, nullptr, &ctx);
      if (ctx_rc != XG_OK) {
        ctx = nullptr;
        return ctx_rc;
      }
    }
    if (layout_m != m) {
      if (series) xg_series_destroy(series);
      series = nullptr;
      series_n = -1;
      if (layout) xg_layout_destroy(layout);
      layout = nullptr;
      std::vector<int64_t> off{0, m}, idx(static_cast<std::size_t>(m));
      for (int64_t i = 0; i < m; ++i) idx[static_cast<std::size_t>(i)] = i;
      const int rc = xg_layout_create(ctx, m, 1, off.data(), idx.data(), &layout);
      if (rc != XG_OK) return rc;
      layout_m = m;
    }
    if (series_n < n) {
      if (series) xg_series_destroy(series);
      series = nullptr;
      const int rc = xg_series_create(ctx, layout, n, &series);
      if (rc != XG_OK) return rc;
      series_n = n;
    }
    return XG_OK;
  }

  ~Engine() {
    if (series) xg_series_destroy(series);
    if (layout) xg_layout_destroy(layout);
    if (ctx) xg_ctx_destroy(ctx);
  }
};

inline Engine& engine() {
  static Engine e;
  return e;
}

// ttc_raw of integer counts on the tensor-core path.  Returns XG_OK and fills
// out (n x n f64), or an xg_status with msg/frame set (NormalizationError:
// *frame = the zero frame).  XG_ERR_INVALID: not counts -> caller falls back.
inline int ttc_raw_counts(const double* x, int64_t n, int64_t m, double* out, std::string& msg,
                          int64_t* frame) {
  if (exact_only()) return XG_ERR_INVALID;
  std::vector<uint8_t> u8;
  if (!pack_counts(x, static_cast<std::size_t>(n * m), u8)) return XG_ERR_INVALID;
  Engine& e = engine();
  std::lock_guard<std::mutex> lock(e.mu);
  int rc = e.ensure(n, m);
  if (rc == XG_OK) rc = xg_series_load_frames(e.series, u8.data(), n, 0);
  if (rc == XG_OK) rc = xg_ttc_raw(e.series, XG_STRICT);
  if (rc == XG_OK) rc = xg_series_get_ttc(e.series, 0, XG_F64, out, n, 0);
  if (rc != XG_OK && e.ctx) {
    msg = xg_last_error(e.ctx);
    int32_t ring = -1;
    *frame = xg_last_error_payload(e.ctx, &ring);
  } else if (rc != XG_OK) {
    msg = "no sm_100 device for the B200 path";
  }
  return rc;
}

}  // namespace xpcs_b200_dropin

#endif  // XPCS_B200_ENGINE_HPP_
