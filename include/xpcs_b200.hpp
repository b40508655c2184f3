// xpcs_b200.hpp -- header-only C++ facade over the C ABI (xpcs_b200.h).
//
// Mirrors the reference's C++ operator API (namespace xpcs,
// /root/reference/proj/include/xpcsvd/{correlate,compress,model,errors}.hpp):
// the same exception hierarchy, and two layers:
//   * reference-facing free functions on row-major f64 buffers with the
//     reference's exact arithmetic (ttc_raw, ttc_compressed, ttc_extend,
//     g2_from_ttc, ttc_rel_error, compress_series, compress_frame);
//   * RAII handles for the high-throughput photon-count path (Context,
//     RingLayout, Series, Basis, Stream): u8 frames in, every q-ring's TTC,
//     compressed TTC and g2 out, computed by the sm_100a kernels.
// No CPU compute path: every number comes from libxpcs_b200.so's kernels.
#ifndef XPCS_B200_HPP_
#define XPCS_B200_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "xpcs_b200.h"

namespace xpcs_b200 {

// ------------------------------------------------------------- errors
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ShapeError : public Error { public: using Error::Error; };
class ContractError : public Error { public: using Error::Error; };
class MaskError : public Error { public: using Error::Error; };
class BindingError : public Error { public: using Error::Error; };
class FormatError : public Error { public: using Error::Error; };
class DeviceError : public Error { public: using Error::Error; };
class NormalizationError : public Error {
 public:
  NormalizationError(const std::string& m, std::size_t frame, int ring = -1)
      : Error(m), frame_(frame), ring_(ring) {}
  std::size_t frame_index() const { return frame_; }
  int ring() const { return ring_; }

 private:
  std::size_t frame_;
  int ring_;
};
class RankError : public Error {
 public:
  RankError(const std::string& m, std::size_t rank) : Error(m), rank_(rank) {}
  std::size_t achievable_rank() const { return rank_; }

 private:
  std::size_t rank_;
};

namespace detail {
[[noreturn]] inline void raise(int rc, const std::string& msg, int64_t payload, int ring) {
  switch (rc) {
    case XG_ERR_SHAPE: throw ShapeError(msg);
    case XG_ERR_CONTRACT: throw ContractError(msg);
    case XG_ERR_MASK: throw MaskError(msg);
    case XG_ERR_NORMALIZATION: throw NormalizationError(msg, static_cast<std::size_t>(payload), ring);
    case XG_ERR_RANK: throw RankError(msg, static_cast<std::size_t>(payload));
    case XG_ERR_BINDING: throw BindingError(msg);
    case XG_ERR_FORMAT: throw FormatError(msg);
    default: throw DeviceError(msg + " (status " + std::to_string(rc) + ")");
  }
}
inline void f64(int rc) {
  if (rc != XG_OK) raise(rc, xg_f64_last_error(), xg_f64_last_payload(), -1);
}
}  // namespace detail

// ------------------------------------------ reference-facing (exact f64)
inline std::vector<double> ttc_raw(const std::vector<double>& x, int64_t n, int64_t m) {
  std::vector<double> g(static_cast<size_t>(n * n));
  detail::f64(xg_f64_ttc_raw(x.data(), n, m, g.data()));
  return g;
}
inline std::pair<std::vector<double>, bool> ttc_compressed(const std::vector<double>& y,
                                                           int64_t n, int64_t k) {
  std::vector<double> g(static_cast<size_t>(n * n));
  int ll = 0;
  detail::f64(xg_f64_ttc_compressed(y.data(), n, k, g.data(), &ll));
  return {std::move(g), ll != 0};
}
inline std::pair<std::vector<double>, bool> ttc_extend(const std::vector<double>& g, int64_t n,
                                                       const std::vector<double>& y, int64_t k,
                                                       const std::vector<double>& row) {
  std::vector<double> out(static_cast<size_t>((n + 1) * (n + 1)));
  int ll = 0;
  detail::f64(xg_f64_ttc_extend(g.data(), n, y.data(), k, row.data(), out.data(), &ll));
  return {std::move(out), ll != 0};
}
struct G2Curve {
  std::vector<double> lags, values;
  std::vector<int64_t> counts;
};
inline G2Curve g2_from_ttc(const std::vector<double>& g, int64_t n, double frame_period) {
  G2Curve c{std::vector<double>(n), std::vector<double>(n), std::vector<int64_t>(n)};
  detail::f64(xg_f64_g2_from_ttc(g.data(), n, frame_period, c.lags.data(), c.values.data(),
                                 c.counts.data()));
  return c;
}
inline double ttc_rel_error(const std::vector<double>& a, const std::vector<double>& b) {
  if (a.size() != b.size()) throw ShapeError("ttc_rel_error: size mismatch");
  double out = 0.0;
  detail::f64(xg_f64_ttc_rel_error(a.data(), b.data(), static_cast<int64_t>(a.size()), &out));
  return out;
}
inline std::pair<std::vector<double>, std::vector<double>> compress_series(
    const std::vector<double>& x, int64_t n, int64_t m, const std::vector<double>& v, int64_t k) {
  std::vector<double> y(static_cast<size_t>(n * k)), norms(static_cast<size_t>(n));
  detail::f64(xg_f64_compress_series(x.data(), n, m, v.data(), k, y.data(), norms.data()));
  return {std::move(y), std::move(norms)};
}

// --------------------------------------------- photon-count fast path
class Context {
 public:
  explicit Context(int device = 0, void* cuda_stream = nullptr) {
    const int rc = xg_ctx_create(device, cuda_stream, &h_);
    if (rc != XG_OK) throw DeviceError("xg_ctx_create failed (an sm_100 B200 is required)");
  }
  ~Context() { xg_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  xg_ctx* get() const { return h_; }
  void check(int rc) const {
    if (rc == XG_OK) return;
    int32_t ring = -1;
    const int64_t payload = xg_last_error_payload(h_, &ring);
    detail::raise(rc, xg_last_error(h_), payload, ring);
  }
  void synchronize() const { check(xg_synchronize(h_)); }

 private:
  xg_ctx* h_ = nullptr;
};

// A set of PixelMask (one per q-ring), each strictly ascending.
class RingLayout {
 public:
  RingLayout(const Context& ctx, int64_t full_pixels, const std::vector<std::vector<int64_t>>& masks)
      : ctx_(ctx) {
    std::vector<int64_t> off(1, 0), idx;
    for (const auto& m : masks) {
      idx.insert(idx.end(), m.begin(), m.end());
      off.push_back(static_cast<int64_t>(idx.size()));
    }
    ctx.check(xg_layout_create(ctx.get(), full_pixels, static_cast<int32_t>(masks.size()),
                               off.data(), idx.data(), &h_));
    rings_ = static_cast<int32_t>(masks.size());
  }
  // a height x width row-major detector (2D ingest bands on wide detectors)
  RingLayout(const Context& ctx, int64_t height, int64_t width,
             const std::vector<std::vector<int64_t>>& masks)
      : ctx_(ctx) {
    std::vector<int64_t> off(1, 0), idx;
    for (const auto& m : masks) {
      idx.insert(idx.end(), m.begin(), m.end());
      off.push_back(static_cast<int64_t>(idx.size()));
    }
    ctx.check(xg_layout_create_2d(ctx.get(), height, width, static_cast<int32_t>(masks.size()),
                                  off.data(), idx.data(), &h_));
    rings_ = static_cast<int32_t>(masks.size());
  }
  ~RingLayout() { xg_layout_destroy(h_); }
  RingLayout(const RingLayout&) = delete;
  RingLayout& operator=(const RingLayout&) = delete;
  xg_layout* get() const { return h_; }
  const Context& ctx() const { return ctx_; }
  int32_t rings() const { return rings_; }

 private:
  const Context& ctx_;
  xg_layout* h_ = nullptr;
  int32_t rings_ = 0;
};

class Basis {
 public:
  Basis(const RingLayout& L, int32_t k, int32_t digits = 3) : L_(L) {
    L.ctx().check(xg_basis_create(L.ctx().get(), L.get(), k, digits, &h_));
  }
  ~Basis() { xg_basis_destroy(h_); }
  Basis(const Basis&) = delete;
  Basis& operator=(const Basis&) = delete;
  // v: M_q x k row-major, mask order
  void set_ring(int32_t ring, const double* v) { L_.ctx().check(xg_basis_set_ring(h_, ring, v)); }
  xg_basis* get() const { return h_; }

 private:
  const RingLayout& L_;
  xg_basis* h_ = nullptr;
};

class Series {
 public:
  Series(const RingLayout& L, int64_t max_frames) : L_(L) {
    L.ctx().check(xg_series_create(L.ctx().get(), L.get(), max_frames, &h_));
  }
  ~Series() { xg_series_destroy(h_); }
  Series(const Series&) = delete;
  Series& operator=(const Series&) = delete;
  void load(const uint8_t* frames, int64_t n, bool on_device = false) {
    L_.ctx().check(xg_series_load_frames(h_, frames, n, on_device ? 1 : 0));
  }
  // The reference's f64 FrameSeries intensities (model.hpp:26-36): accepted
  // when every value is an integer photon count in [0, 255] (packed to u8
  // here, exact); anything else is a ContractError, never a silent wrap.
  void load(const double* intensities, int64_t n, int64_t full_pixels) {
    std::vector<uint8_t> u8(static_cast<size_t>(n * full_pixels));
    for (size_t i = 0; i < u8.size(); ++i) {
      const double v = intensities[i];
      if (!(v >= 0.0 && v <= 255.0) || v != static_cast<double>(static_cast<int>(v)))
        throw ContractError("frame intensities must be integer photon counts in [0, 255] for "
                            "the u8 tensor-core path (value " + std::to_string(v) + " at " +
                            std::to_string(i) + ")");
      u8[i] = static_cast<uint8_t>(v);
    }
    load(u8.data(), n, false);
  }
  void ttc_raw(uint32_t flags = 0) { L_.ctx().check(xg_ttc_raw(h_, flags)); }
  // load + ttc_raw for host frames: PCIe transfer overlapped with the compute
  void ttc_raw_host(const uint8_t* frames, int64_t n, uint32_t flags = 0) {
    L_.ctx().check(xg_series_ttc_raw_host(h_, frames, n, flags));
  }
  // Photon-event frames (CSR by frame: offsets[n + 1], raster pixel,
  // count): the same series as load() of the dense frames
  void load_events(const int64_t* frame_off, const int32_t* pix, const uint8_t* val, int64_t n,
                   bool on_device = false) {
    L_.ctx().check(xg_series_load_events(h_, frame_off, pix, val, n, on_device ? 1 : 0));
  }
  void ttc_raw_events_host(const int64_t* frame_off, const int32_t* pix, const uint8_t* val,
                           int64_t n, uint32_t flags = 0) {
    L_.ctx().check(xg_series_ttc_raw_events_host(h_, frame_off, pix, val, n, flags));
  }
  void compress(const Basis& b, uint32_t flags = 0) { L_.ctx().check(xg_compress(h_, b.get(), flags)); }
  void ttc_compressed(uint32_t flags = 0) { L_.ctx().check(xg_ttc_compressed(h_, flags)); }
  int64_t frames() const { return xg_series_frames(h_); }
  std::vector<double> ttc(int32_t ring) const {
    const int64_t n = frames();
    std::vector<double> out(static_cast<size_t>(n * n));
    L_.ctx().check(xg_series_get_ttc(h_, ring, XG_F64, out.data(), n, 0));
    return out;
  }
  // the exact int32 Gram (full symmetric n x n)
  std::vector<int32_t> gram(int32_t ring) const {
    const int64_t n = frames();
    std::vector<int32_t> out(static_cast<size_t>(n * n));
    L_.ctx().check(xg_series_get_ttc(h_, ring, XG_I32_GRAM, out.data(), n, 0));
    return out;
  }
  // Split rings (multi-GPU): this process's share of a ring as packed upper
  // pair tiles + |x_t|^2, and the summed total installed back (host buffers
  // here; the C ABI also takes device buffers for NCCL).
  struct Partial {
    std::vector<int32_t> gram;
    std::vector<int64_t> norm2;
  };
  Partial export_partial(int32_t ring) {
    Partial p{std::vector<int32_t>(static_cast<size_t>(xg_series_partial_elems(h_))),
              std::vector<int64_t>(static_cast<size_t>(frames()))};
    L_.ctx().check(xg_series_export_partial(h_, ring, p.gram.data(), p.norm2.data(), 0));
    return p;
  }
  void import_partial(int32_t ring, const Partial& p, uint32_t flags = 0) {
    L_.ctx().check(xg_series_import_partial(h_, ring, p.gram.data(), p.norm2.data(), 0, flags));
  }
  std::vector<double> g2(int32_t ring, std::vector<int64_t>* counts = nullptr) const {
    const int64_t n = frames();
    std::vector<double> v(static_cast<size_t>(n));
    std::vector<int64_t> c(static_cast<size_t>(n));
    L_.ctx().check(xg_series_get_g2(h_, ring, v.data(), c.data()));
    if (counts) *counts = std::move(c);
    return v;
  }
  // build_online_from_frames per ring on the device (k = 0: build_offline);
  // fills b (k > 0) and returns each ring's numerical rank
  std::vector<int64_t> build_basis(int32_t k, Basis* b = nullptr) {
    std::vector<int64_t> rank(static_cast<size_t>(rings()));
    L_.ctx().check(xg_series_build_basis(h_, k, nullptr, nullptr, 0, rank.data(),
                                         b ? b->get() : nullptr));
    return rank;
  }
  // analysis.cpp on the device: ttc_background per ring; fit_kww per ring
  // (KwwFit fields B, C, t0, rms + status 0 ok / 1 degenerate / 2 no
  // convergence / 3 contract)
  std::vector<double> ttc_background(int64_t exclusion = 0, bool compressed = false) {
    std::vector<double> out(static_cast<size_t>(rings()));
    L_.ctx().check(xg_series_ttc_background(h_, compressed ? 1 : 0, exclusion, out.data()));
    return out;
  }
  struct KwwFit {
    double baseline, contrast, relaxation_time, residual_rms;
    int32_t status;
  };
  std::vector<KwwFit> fit_kww(double frame_period, double min_lag, double max_lag,
                              bool compressed = false) {
    const int32_t q = rings();
    std::vector<double> o(static_cast<size_t>(4 * q));
    std::vector<int32_t> st(static_cast<size_t>(q));
    L_.ctx().check(xg_series_fit_kww(h_, compressed ? 1 : 0, frame_period, min_lag, max_lag,
                                     o.data(), st.data()));
    std::vector<KwwFit> out;
    for (int32_t r = 0; r < q; ++r) out.push_back({o[4 * r], o[4 * r + 1], o[4 * r + 2], o[4 * r + 3], st[r]});
    return out;
  }
  // io.cpp formats next to the device buffers
  void write_xcmp(int32_t ring, const std::string& path, uint64_t encoder_hash, bool append = false) {
    L_.ctx().check(xg_series_write_xcmp(h_, ring, path.c_str(), encoder_hash, append ? 1 : 0));
  }
  double load_xfsr(const std::string& path) {
    double period = 0.0;
    L_.ctx().check(xg_series_load_xfsr(h_, path.c_str(), &period));
    return period;
  }
  void write_ttc(int32_t ring, const std::string& path, xg_dtype dtype = XG_F64,
                 bool compressed = false) {
    L_.ctx().check(xg_series_write_ttc(h_, ring, compressed ? 1 : 0, dtype, path.c_str()));
  }
  int32_t rings() const { return L_.rings(); }
  xg_series* get() const { return h_; }

 private:
  const RingLayout& L_;
  xg_series* h_ = nullptr;
};

class Stream {
 public:
  Stream(const RingLayout& L, int64_t max_frames, const Basis* b = nullptr, uint32_t flags = 0)
      : L_(L) {
    L.ctx().check(xg_stream_create(L.ctx().get(), L.get(), b ? b->get() : nullptr, max_frames,
                                   flags, &h_));
  }
  ~Stream() { xg_stream_destroy(h_); }
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
  void push(const uint8_t* frame, bool on_device = false) {
    L_.ctx().check(xg_stream_push(h_, frame, on_device ? 1 : 0));
  }
  void push_batch(const uint8_t* frames, int64_t n, bool on_device = false) {
    L_.ctx().check(xg_stream_push_batch(h_, frames, n, on_device ? 1 : 0));
  }
  int64_t frames() const { return xg_stream_frames(h_); }
  std::vector<double> g2(int32_t ring, bool compressed = false) const {
    std::vector<double> v(static_cast<size_t>(frames()));
    L_.ctx().check(xg_stream_get_g2(h_, ring, compressed ? 1 : 0, v.data(), nullptr));
    return v;
  }

 private:
  const RingLayout& L_;
  xg_stream* h_ = nullptr;
};

}  // namespace xpcs_b200

#endif  // XPCS_B200_HPP_
