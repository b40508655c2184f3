// compress_b200.cpp -- drop-in replacement for /root/reference/proj/src/
// compress.cpp: compress_series / compress_frame on the B200 through the
// xg_f64_* reference-order entries of libxpcs_b200.so (bit-identical to the
// reference, including zero-pixel skipping and the first-zero-frame error);
// series of integer photon counts are shipped as u8 and widened on the device.
// decompress is validation-only (out of scope): it stays a
// host loop over the reference's own xpcs::dot.
#include "xpcsvd/compress.hpp"

#include <string>
#include <vector>

#include "b200_engine.hpp"
#include "xpcs_b200.h"

namespace xpcs {

namespace {

void check(int rc) {
  if (rc == XG_OK) return;
  const std::string msg = xg_f64_last_error();
  if (rc == XG_ERR_NORMALIZATION)
    throw NormalizationError(msg, static_cast<std::size_t>(xg_f64_last_payload()));
  if (rc == XG_ERR_SHAPE) throw ShapeError(msg);
  if (rc == XG_ERR_CONTRACT) throw ContractError(msg);
  throw Error("xpcs_b200: " + msg + " (status " + std::to_string(rc) + ")");
}

void check_pixels(std::size_t frame_pixels, const EncodingMatrix& enc) {
  if (frame_pixels != enc.n_pixels())
    throw ShapeError("frame has " + std::to_string(frame_pixels) + " pixels, encoder expects " +
                     std::to_string(enc.n_pixels()));
}

}  // namespace

std::pair<std::vector<double>, double> compress_frame(std::span<const double> frame,
                                                      const EncodingMatrix& enc) {
  check_pixels(frame.size(), enc);
  std::vector<double> coeffs(enc.k());
  double norm = 0.0;
  check(xg_f64_compress_frame(frame.data(), static_cast<int64_t>(frame.size()),
                              enc.v().data().data(), static_cast<int64_t>(enc.k()), coeffs.data(),
                              &norm));
  return {std::move(coeffs), norm};
}

CompressedSeries compress_series(const FrameSeries& frames, const EncodingMatrix& enc) {
  check_pixels(frames.n_pixels(), enc);
  const std::size_t n = frames.n_frames(), k = enc.k();
  std::vector<double> coeffs(n * k), norms(n);
  const double* x = frames.intensities.data().data();
  const int64_t m = static_cast<int64_t>(frames.n_pixels());
  // integer photon counts cross PCIe as u8 (1 B instead of 8 per pixel) and
  // are widened on the device: the same kernels, the same bits
  std::vector<uint8_t> u8;
  if (!xpcs_b200_dropin::exact_only() && n > 0 &&
      xpcs_b200_dropin::pack_counts(x, n * frames.n_pixels(), u8))
    check(xg_f64_compress_series_u8(u8.data(), static_cast<int64_t>(n), m, enc.v().data().data(),
                                    static_cast<int64_t>(k), coeffs.data(), norms.data()));
  else
    check(xg_f64_compress_series(x, static_cast<int64_t>(n), m, enc.v().data().data(),
                                 static_cast<int64_t>(k), coeffs.data(), norms.data()));
  return CompressedSeries(k, content_hash_u64(enc), std::move(coeffs), std::move(norms));
}

Matrix decompress(const CompressedSeries& y, const EncodingMatrix& enc) {
  if (y.encoder_id() != content_hash_u64(enc))
    throw BindingError("store was compressed with a different encoder (content hash mismatch)");
  const auto snap = y.snapshot();
  const Matrix ym = snap.coefficient_matrix();
  Matrix out(ym.rows(), enc.n_pixels());
  for (std::size_t i = 0; i < ym.rows(); ++i)
    for (std::size_t p = 0; p < enc.n_pixels(); ++p) out(i, p) = dot(ym.row(i), enc.v().row(p));
  return out;
}

}  // namespace xpcs
