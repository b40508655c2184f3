// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile with the
// reference's own Release flags into oracle/_ref/libxpcsvd_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (oracle/xpcs_oracle.c) and to generate tests/golden/, and by bench.py's
// `--impl reference` / cpu_baseline legs to time the reference's own CPU
// path.  The product never links it.
//
// Error codes mirror the C-ABI of the product (include/xpcs_b200.h):
// 0 ok, 1 ShapeError, 2 ContractError, 3 MaskError, 4 NormalizationError,
// 5 RankError, 6 BindingError, 7 FormatError, 99 other.
#include <cstdint>
#include <cstring>
#include <vector>

#include "xpcsvd/analysis.hpp"
#include "xpcsvd/compress.hpp"
#include "xpcsvd/correlate.hpp"
#include "xpcsvd/encoder.hpp"
#include "xpcsvd/io.hpp"
#include "xpcsvd/linalg.hpp"
#include "xpcsvd/model.hpp"
#include "xpcsvd/rng.hpp"

using namespace xpcs;

namespace {

thread_local int64_t g_payload = -1;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError&) {
    return 1;
  } catch (const ContractError&) {
    return 2;
  } catch (const MaskError&) {
    return 3;
  } catch (const NormalizationError& e) {
    g_payload = static_cast<int64_t>(e.frame_index());
    return 4;
  } catch (const RankError& e) {
    g_payload = static_cast<int64_t>(e.achievable_rank());
    return 5;
  } catch (const BindingError&) {
    return 6;
  } catch (const Error&) {
    return 99;
  }
}

Matrix to_matrix(const double* p, int64_t rows, int64_t cols) {
  return Matrix(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols),
                std::vector<double>(p, p + rows * cols));
}

void copy_out(const Matrix& m, double* out) {
  std::memcpy(out, m.data().data(), sizeof(double) * m.data().size());
}

EncodingMatrix to_encoder(const double* v, int64_t m, int64_t k) {
  // Spectrum is only checked for monotonicity; a flat one is valid.
  return EncodingMatrix(to_matrix(v, m, k), std::vector<double>(k, 1.0),
                        EncoderMode::kOnlineRelated);
}

}  // namespace

extern "C" {

int64_t ref_last_payload() { return g_payload; }

int ref_gram(const double* x, int64_t n, int64_t m, double* out) {
  return guarded([&] { copy_out(gram(to_matrix(x, n, m)), out); });
}

int ref_row_normalize(const double* x, int64_t n, int64_t m, double* out, double* norms) {
  return guarded([&] {
    auto r = row_normalize(to_matrix(x, n, m));
    copy_out(r.first, out);
    std::memcpy(norms, r.second.data(), sizeof(double) * r.second.size());
  });
}

int ref_ttc_raw(const double* x, int64_t n, int64_t m, double* out) {
  return guarded([&] { copy_out(ttc_raw(FrameSeries(to_matrix(x, n, m))).values(), out); });
}

int ref_ttc_compressed(const double* y, const double* norms, int64_t n, int64_t k,
                       double* out, int* lossless) {
  return guarded([&] {
    CompressedSeries s(static_cast<std::size_t>(k), 0,
                       std::vector<double>(y, y + n * k), std::vector<double>(norms, norms + n));
    TTCMatrix g = ttc_compressed(s);
    copy_out(g.values(), out);
    *lossless = g.lossless() ? 1 : 0;
  });
}

// Streams n frames through the reference's ttc_extend / append loop (the
// acceptance criterion 9 pattern): the first two rows seed ttc_compressed,
// every further row is ttc_extend-ed, then appended.
int ref_ttc_extend_stream(const double* y, const double* norms, int64_t n, int64_t k,
                          double* out) {
  return guarded([&] {
    CompressedSeries s(static_cast<std::size_t>(k), 0);
    s.append({y, static_cast<std::size_t>(k)}, norms[0]);
    s.append({y + k, static_cast<std::size_t>(k)}, norms[1]);
    TTCMatrix g = ttc_compressed(s);
    for (int64_t t = 2; t < n; ++t) {
      std::span<const double> row{y + t * k, static_cast<std::size_t>(k)};
      g = ttc_extend(g, s, row);
      s.append(row, norms[t]);
    }
    copy_out(g.values(), out);
  });
}

int ref_ttc_extend(const double* g, int64_t n, const double* y, const double* norms,
                   int64_t k, const double* row, double* out) {
  return guarded([&] {
    CompressedSeries s(static_cast<std::size_t>(k), 0,
                       std::vector<double>(y, y + n * k), std::vector<double>(norms, norms + n));
    TTCMatrix in(to_matrix(g, n, n), false);
    copy_out(ttc_extend(in, s, {row, static_cast<std::size_t>(k)}).values(), out);
  });
}

int ref_g2_from_ttc(const double* g, int64_t n, double period, double* lags, double* values,
                    int64_t* counts) {
  return guarded([&] {
    G2Curve c = g2_from_ttc(TTCMatrix(to_matrix(g, n, n), false), period);
    for (int64_t d = 0; d < n; ++d) {
      lags[d] = c.lags[d];
      values[d] = c.values[d];
      counts[d] = static_cast<int64_t>(c.counts[d]);
    }
  });
}

// content_hash_u64 (model.cpp:99-114) of an encoder with this V and mode.
int ref_content_hash(const double* v, int64_t m, int64_t k, int mode, uint64_t* out) {
  return guarded([&] {
    EncodingMatrix e(to_matrix(v, m, k), std::vector<double>(k, 1.0), static_cast<EncoderMode>(mode));
    *out = content_hash_u64(e);
  });
}

int ref_ttc_rel_error(const double* a, const double* b, int64_t n, double* out) {
  return guarded([&] { *out = ttc_rel_error(to_matrix(a, n, n), to_matrix(b, n, n)); });
}

int ref_compress_series(const double* x, int64_t n, int64_t m, const double* v, int64_t k,
                        double* coeffs, double* norms) {
  return guarded([&] {
    CompressedSeries s = compress_series(FrameSeries(to_matrix(x, n, m)), to_encoder(v, m, k));
    auto snap = s.snapshot();
    std::memcpy(coeffs, snap.coefficients.data(), sizeof(double) * snap.coefficients.size());
    std::memcpy(norms, snap.norms.data(), sizeof(double) * snap.norms.size());
  });
}

int ref_compress_frame(const double* frame, int64_t m, const double* v, int64_t k,
                       double* coeffs, double* norm) {
  return guarded([&] {
    auto r = compress_frame({frame, static_cast<std::size_t>(m)}, to_encoder(v, m, k));
    std::memcpy(coeffs, r.first.data(), sizeof(double) * r.first.size());
    *norm = r.second;
  });
}

// Basis from a prior measurement (encoder.cpp:53-60): V (m x k) and the
// first min(n, spectrum) singular values.
int ref_build_online_from_frames(const double* x, int64_t n, int64_t m, int64_t k, double* v,
                                 double* spectrum, int64_t* spectrum_len) {
  return guarded([&] {
    EncodingMatrix e = build_online_from_frames(FrameSeries(to_matrix(x, n, m)),
                                                static_cast<std::size_t>(k));
    copy_out(e.v(), v);
    *spectrum_len = static_cast<int64_t>(e.spectrum().size());
    std::memcpy(spectrum, e.spectrum().data(), sizeof(double) * e.spectrum().size());
  });
}

int ref_build_offline(const double* x, int64_t n, int64_t m, double* v, int64_t* k_out) {
  return guarded([&] {
    EncodingMatrix e = build_offline(FrameSeries(to_matrix(x, n, m)));
    copy_out(e.v(), v);
    *k_out = static_cast<int64_t>(e.k());
  });
}

int ref_apply_mask(const double* x, int64_t n, int64_t m_full, const int64_t* idx, int64_t mq,
                   double* out) {
  return guarded([&] {
    std::vector<std::size_t> ind(idx, idx + mq);
    FrameSeries f = apply_mask(FrameSeries(to_matrix(x, n, m_full)),
                               PixelMask(static_cast<std::size_t>(m_full), ind));
    copy_out(f.intensities, out);
  });
}

// io::read_compressed (io.cpp:334-360): call with coeffs == null for the
// dimensions, then with buffers.  FormatError -> 7 (payload = offset).
int ref_read_compressed(const char* path, int64_t* k, uint64_t* hash, int64_t* n, double* coeffs,
                        double* norms) {
  try {
    CompressedSeries cs = io::read_compressed(path);
    auto snap = cs.snapshot();
    *k = static_cast<int64_t>(snap.k);
    *hash = snap.encoder_id;
    *n = static_cast<int64_t>(snap.n_frames());
    if (coeffs) std::memcpy(coeffs, snap.coefficients.data(), snap.coefficients.size() * 8);
    if (norms) std::memcpy(norms, snap.norms.data(), snap.norms.size() * 8);
    return 0;
  } catch (const FormatError& e) {
    g_payload = static_cast<int64_t>(e.offset());
    return 7;
  } catch (const Error&) {
    return 99;
  }
}

// io::write_encoder / read_encoder (io.cpp:273-321).
int ref_write_encoder(const char* path, const double* v, int64_t m, int64_t k, const double* spec,
                      int64_t sl, int mode) {
  return guarded([&] {
    io::write_encoder(path, EncodingMatrix(to_matrix(v, m, k), std::vector<double>(spec, spec + sl),
                                           static_cast<EncoderMode>(mode)));
  });
}
int ref_read_encoder(const char* path, int64_t* m, int64_t* k, int64_t* sl, int* mode, double* v,
                     double* spec) {
  try {
    EncodingMatrix e = io::read_encoder(path);
    *m = static_cast<int64_t>(e.n_pixels());
    *k = static_cast<int64_t>(e.k());
    *sl = static_cast<int64_t>(e.spectrum().size());
    *mode = static_cast<int>(e.mode());
    if (v) std::memcpy(v, e.v().data().data(), e.v().data().size() * 8);
    if (spec) std::memcpy(spec, e.spectrum().data(), e.spectrum().size() * 8);
    return 0;
  } catch (const FormatError& ex) {
    g_payload = static_cast<int64_t>(ex.offset());
    return 7;
  } catch (const Error&) {
    return 99;
  }
}

// io::write_frames (io.cpp:150-184) with dtype 0 u16, 1 f32, 2 f64.
int ref_write_frames(const char* path, const double* x, int64_t n, int64_t m, double period,
                     int dtype) {
  return guarded([&] {
    io::write_frames(path, FrameSeries(to_matrix(x, n, m), period),
                     static_cast<io::FrameDtype>(dtype));
  });
}

// io::read_frames status only (FormatError -> 7, payload = offset).
int ref_read_frames_status(const char* path, int64_t* n, int64_t* m) {
  try {
    FrameSeries f = io::read_frames(path);
    *n = static_cast<int64_t>(f.n_frames());
    *m = static_cast<int64_t>(f.n_pixels());
    return 0;
  } catch (const FormatError& e) {
    g_payload = static_cast<int64_t>(e.offset());
    return 7;
  } catch (const Error&) {
    return 99;
  }
}

// ttc_background (analysis.cpp:202-235) of an n x n TTC.
int ref_ttc_background(const double* g, int64_t n, int64_t exclusion, double* out) {
  return guarded([&] {
    *out = ttc_background(TTCMatrix(to_matrix(g, n, n), false), static_cast<std::size_t>(exclusion));
  });
}

// fit_kww (analysis.cpp:77-172) of a g2 curve; out = {B, C, t0, rms}.
// Status 10: FitDegenerateError, 11: FitError (out = its best()).
int ref_fit_kww(const double* lags, const double* values, int64_t n, double min_lag,
                double max_lag, double* out) {
  try {
    G2Curve c;
    c.lags.assign(lags, lags + n);
    c.values.assign(values, values + n);
    c.counts.assign(static_cast<std::size_t>(n), 1);
    const KwwFit f = fit_kww(c, LagWindow{min_lag, max_lag});
    out[0] = f.baseline;
    out[1] = f.contrast;
    out[2] = f.relaxation_time;
    out[3] = f.residual_rms;
    return 0;
  } catch (const FitDegenerateError&) {
    return 10;
  } catch (const FitError& e) {
    out[0] = e.best().baseline;
    out[1] = e.best().contrast;
    out[2] = e.best().relaxation_time;
    out[3] = e.best().residual_rms;
    return 11;
  } catch (const ContractError&) {
    return 2;
  } catch (const Error&) {
    return 99;
  }
}

uint64_t ref_rng_bits(uint64_t seed, uint64_t tag, uint64_t index) {
  return CounterRng(seed).substream(tag).bits(index);
}
double ref_rng_normal(uint64_t seed, uint64_t tag, uint64_t index) {
  return CounterRng(seed).substream(tag).normal(index);
}
double ref_rng_exponential(uint64_t seed, uint64_t tag, uint64_t index) {
  return CounterRng(seed).substream(tag).exponential(index);
}

}  // extern "C"
