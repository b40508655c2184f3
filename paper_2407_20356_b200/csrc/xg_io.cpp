// xg_io.cpp -- on-disk formats next to the device buffers (SURVEY 8(f)
// item 3; the reference's src/io.cpp).  Host code: the device entry points
// in xg_api.cu copy the rows out and call these.
//
//   XCMP store (io.cpp:319-441): "XCMP", u32 1, u64 K, u64 encoder hash,
//     u64 N, then N records (f64 norm, K f64 coefficients), little-endian.
//     xg_io_write_xcmp writes a new store or, like CompressedFileAppender,
//     validates an existing one (k -> ShapeError, hash -> BindingError,
//     layout -> FormatError) and appends, rewriting N at offset 24.
//   XFSR frames (io.cpp:150-225): "XFSR", u32 1, u32 dtype, u64 N, u64 M,
//     f64 frame_period, N*M values.  dtype 0 u16, 1 f32, 2 f64 as the
//     reference; dtype 3 = u8 photon counts is new here (1 byte per pixel,
//     the detector's own width).  The reader applies the reference's checks
//     (magic, version, dtype, plausible dims, period, exact size -> FormatError
//     with the byte offset) and accepts only integer counts in [0, 255] for
//     the u8 device path (ContractError otherwise).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/xpcs_b200.h"

namespace {

thread_local char g_err[320];
thread_local int64_t g_payload = -1;

int io_fail(int code, int64_t payload, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
int io_fail(int code, int64_t payload, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  g_payload = payload;
  return code;
}

void put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_f64(std::vector<uint8_t>& b, double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  put_u64(b, u);
}
uint32_t get_u32(const uint8_t* p) {
  uint32_t v = 0;
  for (int i = 3; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
uint64_t get_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
double get_f64(const uint8_t* p) {
  const uint64_t u = get_u64(p);
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

bool read_all(const char* path, std::vector<uint8_t>& bytes) {
  File fh;
  fh.f = fopen(path, "rb");
  if (!fh.f) return false;
  if (fseek(fh.f, 0, SEEK_END) != 0) return false;
  const long sz = ftell(fh.f);
  if (sz < 0) return false;
  rewind(fh.f);
  bytes.resize(static_cast<size_t>(sz));
  return sz == 0 || fread(bytes.data(), 1, bytes.size(), fh.f) == bytes.size();
}

}  // namespace

extern "C" {

XG_API const char* xg_io_last_error(void) { return g_err; }
XG_API int64_t xg_io_last_payload(void) { return g_payload; }

XG_API int xg_io_write_xcmp(const char* path, int64_t k, uint64_t hash, int64_t n,
                            const double* norms, const double* coeffs, int32_t append) {
  if (!path || n < 0 || (n > 0 && (!norms || !coeffs))) return XG_ERR_INVALID;
  if (k < 1) return io_fail(XG_ERR_CONTRACT, -1, "appender needs k >= 1");
  for (int64_t i = 0; i < n; ++i) {  // CompressedSeries::append (model.cpp:177-193)
    if (!(norms[i] > 0.0) || !std::isfinite(norms[i]))
      return io_fail(XG_ERR_NORMALIZATION, i, "store row %lld: frame norm must be positive and finite",
                     (long long)i);
    double sq = 0.0;
    for (int64_t j = 0; j < k; ++j) {
      const double v = coeffs[i * k + j];
      if (!std::isfinite(v))
        return io_fail(XG_ERR_CONTRACT, i, "store row %lld: non-finite coefficient", (long long)i);
      sq += v * v;
    }
    // the reader rebuilds the store through append(), which rejects rows
    // above unit norm: such a file could never be read back
    if (sq > (1.0 + 1e-10) * (1.0 + 1e-10))
      return io_fail(XG_ERR_CONTRACT, i,
                     "store row %lld: coefficient row norm %.17g exceeds 1 (not a projection "
                     "of a unit row)", (long long)i, std::sqrt(sq));
  }
  uint64_t n_old = 0;
  std::vector<uint8_t> head;
  File fh;
  if (append) {
    std::vector<uint8_t> old;
    if (read_all(path, old) && !old.empty()) {
      // read_compressed's validation of the existing store (io.cpp:334-360)
      if (old.size() < 4 || std::memcmp(old.data(), "XCMP", 4) != 0)
        return io_fail(XG_ERR_FORMAT, 0, "bad magic, expected \"XCMP\" for compressed store");
      if (old.size() < 32) return io_fail(XG_ERR_FORMAT, (int64_t)old.size(), "compressed store file truncated");
      if (get_u32(old.data() + 4) != 1)
        return io_fail(XG_ERR_FORMAT, 4, "unsupported compressed store version %u", get_u32(old.data() + 4));
      const uint64_t ok = get_u64(old.data() + 8), oh = get_u64(old.data() + 16);
      n_old = get_u64(old.data() + 24);
      if (ok < 1 || ok > (1ull << 30) || n_old > (1ull << 40) / (ok + 1))
        return io_fail(XG_ERR_FORMAT, 8, "implausible store dimensions");
      const uint64_t want = 32 + n_old * 8 * (ok + 1);
      if (old.size() != want)
        return io_fail(XG_ERR_FORMAT, (int64_t)std::min<uint64_t>(old.size(), want),
                       "compressed store file length %zu, expected %llu", old.size(),
                       (unsigned long long)want);
      if ((int64_t)ok != k)
        return io_fail(XG_ERR_SHAPE, -1, "existing store has k = %llu, appender configured with k = %lld",
                       (unsigned long long)ok, (long long)k);
      if (oh != hash)
        return io_fail(XG_ERR_BINDING, -1, "existing store was written with a different encoder");
      fh.f = fopen(path, "r+b");
      if (!fh.f || fseek(fh.f, 0, SEEK_END) != 0)
        return io_fail(XG_ERR_FORMAT, -1, "cannot reopen store file %s", path);
    } else {
      append = 0;
    }
  }
  if (!append) {
    fh.f = fopen(path, "wb");
    if (!fh.f) return io_fail(XG_ERR_FORMAT, -1, "cannot create store file %s", path);
    head.insert(head.end(), {'X', 'C', 'M', 'P'});
    put_u32(head, 1);
    put_u64(head, static_cast<uint64_t>(k));
    put_u64(head, hash);
    put_u64(head, 0);  // N, rewritten below
    if (fwrite(head.data(), 1, head.size(), fh.f) != head.size())
      return io_fail(XG_ERR_FORMAT, -1, "failed writing compressed store file %s", path);
  }
  std::vector<uint8_t> rec;
  rec.reserve(static_cast<size_t>(8 * (k + 1)) * 64);
  for (int64_t i = 0; i < n; ++i) {
    put_f64(rec, norms[i]);
    for (int64_t j = 0; j < k; ++j) put_f64(rec, coeffs[i * k + j]);
    if (rec.size() >= static_cast<size_t>(8 * (k + 1)) * 63 || i + 1 == n) {
      if (fwrite(rec.data(), 1, rec.size(), fh.f) != rec.size())
        return io_fail(XG_ERR_FORMAT, -1, "store append failed");
      rec.clear();
    }
  }
  std::vector<uint8_t> nb;
  put_u64(nb, n_old + static_cast<uint64_t>(n));
  if (fseek(fh.f, 24, SEEK_SET) != 0 || fwrite(nb.data(), 1, 8, fh.f) != 8)
    return io_fail(XG_ERR_FORMAT, -1, "store close failed");
  if (fclose(fh.f) != 0) {
    fh.f = nullptr;
    return io_fail(XG_ERR_FORMAT, -1, "store close failed");
  }
  fh.f = nullptr;
  return XG_OK;
}

XG_API int xg_io_write_xfsr_u8(const char* path, const uint8_t* frames, int64_t n, int64_t m,
                               double frame_period) {
  if (!path || !frames || n < 1 || m < 1) return XG_ERR_INVALID;
  if (!(frame_period > 0.0) || !std::isfinite(frame_period))
    return io_fail(XG_ERR_CONTRACT, -1, "frame_period must be positive and finite");
  File fh;
  fh.f = fopen(path, "wb");
  if (!fh.f) return io_fail(XG_ERR_FORMAT, -1, "cannot create frames file %s", path);
  std::vector<uint8_t> h;
  h.insert(h.end(), {'X', 'F', 'S', 'R'});
  put_u32(h, 1);
  put_u32(h, 3);  // u8 photon counts
  put_u64(h, static_cast<uint64_t>(n));
  put_u64(h, static_cast<uint64_t>(m));
  put_f64(h, frame_period);
  const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(m);
  if (fwrite(h.data(), 1, h.size(), fh.f) != h.size() || fwrite(frames, 1, bytes, fh.f) != bytes)
    return io_fail(XG_ERR_FORMAT, -1, "failed writing frames file %s", path);
  if (fclose(fh.f) != 0) {
    fh.f = nullptr;
    return io_fail(XG_ERR_FORMAT, -1, "failed writing frames file %s", path);
  }
  fh.f = nullptr;
  return XG_OK;
}

// Two calls: out == null returns the dimensions only; then out receives
// n * m u8 counts (out_cap >= n * m).
XG_API int xg_io_read_xfsr_u8(const char* path, uint8_t* out, int64_t out_cap, int64_t* n_out,
                              int64_t* m_out, double* period_out) {
  if (!path || !n_out || !m_out) return XG_ERR_INVALID;
  // header + size checks first, then the payload in 16 MB pieces (the file
  // is never held in memory whole)
  File fh;
  fh.f = fopen(path, "rb");
  if (!fh.f) return io_fail(XG_ERR_FORMAT, -1, "cannot open frames file %s", path);
  if (fseeko(fh.f, 0, SEEK_END) != 0) return io_fail(XG_ERR_FORMAT, -1, "cannot read frames file %s", path);
  const uint64_t size = static_cast<uint64_t>(ftello(fh.f));
  rewind(fh.f);
  uint8_t h[36];
  const size_t got = fread(h, 1, sizeof h, fh.f);
  if (got < 4 || std::memcmp(h, "XFSR", 4) != 0)
    return io_fail(XG_ERR_FORMAT, 0, "bad magic, expected \"XFSR\" for frames");
  if (got < 8) return io_fail(XG_ERR_FORMAT, (int64_t)got, "frames file truncated, need 4 more bytes");
  if (get_u32(h + 4) != 1) return io_fail(XG_ERR_FORMAT, 4, "unsupported frames version %u", get_u32(h + 4));
  if (got < 36) return io_fail(XG_ERR_FORMAT, (int64_t)got, "frames file truncated");
  const uint32_t dtype = get_u32(h + 8);
  if (dtype > 3) return io_fail(XG_ERR_FORMAT, 8, "unknown frames dtype %u", dtype);
  const uint64_t n = get_u64(h + 12), m = get_u64(h + 20);
  if (n < 1 || m < 1 || m > (1ull << 40) / n)
    return io_fail(XG_ERR_FORMAT, 12, "implausible frame dimensions %llux%llu", (unsigned long long)n,
                   (unsigned long long)m);
  const double period = get_f64(h + 28);
  if (!(period > 0.0) || !std::isfinite(period))
    return io_fail(XG_ERR_FORMAT, 28, "frame period must be positive");
  const uint64_t elem = dtype == 0 ? 2 : dtype == 1 ? 4 : dtype == 2 ? 8 : 1;
  const uint64_t want = 36 + n * m * elem;
  if (size != want)
    return io_fail(XG_ERR_FORMAT, (int64_t)std::min<uint64_t>(size, want),
                   "frames file length %llu, expected %llu", (unsigned long long)size,
                   (unsigned long long)want);
  *n_out = static_cast<int64_t>(n);
  *m_out = static_cast<int64_t>(m);
  if (period_out) *period_out = period;
  if (!out) return XG_OK;
  if (out_cap < static_cast<int64_t>(n * m)) return XG_ERR_INVALID;
  const uint64_t total = n * m, per = (16u << 20) / elem;
  std::vector<uint8_t> buf(static_cast<size_t>(std::min<uint64_t>(total, per) * elem));
  for (uint64_t i0 = 0; i0 < total; i0 += per) {
    const uint64_t cnt = std::min<uint64_t>(per, total - i0);
    if (fread(buf.data(), 1, cnt * elem, fh.f) != cnt * elem)
      return io_fail(XG_ERR_FORMAT, (int64_t)(36 + i0 * elem), "cannot read frames file %s", path);
    const uint8_t* p = buf.data();
    for (uint64_t j = 0; j < cnt; ++j) {
      double v;
      switch (dtype) {
        case 0: v = static_cast<double>(p[2 * j] | (uint32_t(p[2 * j + 1]) << 8)); break;
        case 1: {
          const uint32_t u = get_u32(p + 4 * j);
          float f;
          std::memcpy(&f, &u, 4);
          v = f;
          break;
        }
        case 2: v = get_f64(p + 8 * j); break;
        default: v = p[j];
      }
      if (!(v >= 0.0 && v <= 255.0) || v != std::floor(v))
        return io_fail(XG_ERR_CONTRACT, static_cast<int64_t>(36 + (i0 + j) * elem),
                       "frame value %g is not a photon count in [0, 255]", v);
      out[i0 + j] = static_cast<uint8_t>(v);
    }
  }
  return XG_OK;
}

// XENC encoder (io.cpp:273-321): "XENC", u32 1, u8 mode, u64 M, u64 K, u64
// spectrum length, spectrum f64, M*K f64 row-major.  A device-built basis
// saved for the reference (or read back); the content hash that binds an
// XCMP store is xg_content_hash over the same V and mode.
XG_API int xg_io_write_xenc(const char* path, int32_t mode, int64_t m, int64_t k,
                            const double* spectrum, int64_t spectrum_len, const double* v) {
  if (!path || !v || !spectrum || m < 1 || k < 1 || spectrum_len < k) return XG_ERR_INVALID;
  if (mode < 0 || mode > 2) return io_fail(XG_ERR_CONTRACT, -1, "unknown encoder mode %d", mode);
  File fh;
  fh.f = fopen(path, "wb");
  if (!fh.f) return io_fail(XG_ERR_FORMAT, -1, "cannot create encoder file %s", path);
  std::vector<uint8_t> b;
  b.insert(b.end(), {'X', 'E', 'N', 'C'});
  put_u32(b, 1);
  b.push_back(static_cast<uint8_t>(mode));
  put_u64(b, static_cast<uint64_t>(m));
  put_u64(b, static_cast<uint64_t>(k));
  put_u64(b, static_cast<uint64_t>(spectrum_len));
  for (int64_t i = 0; i < spectrum_len; ++i) put_f64(b, spectrum[i]);
  for (int64_t i = 0; i < m * k; ++i) {
    put_f64(b, v[i]);
    if (b.size() >= (8u << 20) || i + 1 == m * k) {
      if (fwrite(b.data(), 1, b.size(), fh.f) != b.size())
        return io_fail(XG_ERR_FORMAT, -1, "failed writing encoder file %s", path);
      b.clear();
    }
  }
  if (fclose(fh.f) != 0) {
    fh.f = nullptr;
    return io_fail(XG_ERR_FORMAT, -1, "failed writing encoder file %s", path);
  }
  fh.f = nullptr;
  return XG_OK;
}

// Two calls: v == null returns mode, M, K and the spectrum length; then v
// (M*K) and spectrum (spectrum_len) receive the payload.  read_encoder's
// layout checks; the orthonormality check is the caller's (Basis.set_ring /
// the tests), as EncodingMatrix's constructor is in the reference.
XG_API int xg_io_read_xenc(const char* path, int32_t* mode, int64_t* m, int64_t* k,
                           int64_t* spectrum_len, double* spectrum, double* v) {
  if (!path || !mode || !m || !k || !spectrum_len) return XG_ERR_INVALID;
  std::vector<uint8_t> b;
  if (!read_all(path, b)) return io_fail(XG_ERR_FORMAT, -1, "cannot open encoder file %s", path);
  if (b.size() < 4 || std::memcmp(b.data(), "XENC", 4) != 0)
    return io_fail(XG_ERR_FORMAT, 0, "bad magic, expected \"XENC\" for encoder");
  if (b.size() < 33) return io_fail(XG_ERR_FORMAT, (int64_t)b.size(), "encoder file truncated");
  if (get_u32(b.data() + 4) != 1)
    return io_fail(XG_ERR_FORMAT, 4, "unsupported encoder version %u", get_u32(b.data() + 4));
  if (b[8] > 2) return io_fail(XG_ERR_FORMAT, 8, "unknown encoder mode %u", b[8]);
  const uint64_t mm = get_u64(b.data() + 9), kk = get_u64(b.data() + 17),
                 sl = get_u64(b.data() + 25);
  if (mm < 1 || kk < 1 || kk > mm || sl < kk || sl > (1ull << 40) || mm > (1ull << 40) / kk)
    return io_fail(XG_ERR_FORMAT, 9, "implausible encoder dimensions");
  const uint64_t want = 33 + 8 * sl + 8 * mm * kk;
  if (b.size() != want)
    return io_fail(XG_ERR_FORMAT, (int64_t)std::min<uint64_t>(b.size(), want),
                   "encoder file length %zu, expected %llu", b.size(), (unsigned long long)want);
  *mode = b[8];
  *m = static_cast<int64_t>(mm);
  *k = static_cast<int64_t>(kk);
  *spectrum_len = static_cast<int64_t>(sl);
  if (!v) return XG_OK;
  if (spectrum)
    for (uint64_t i = 0; i < sl; ++i) spectrum[i] = get_f64(b.data() + 33 + 8 * i);
  const uint8_t* pv = b.data() + 33 + 8 * sl;
  for (uint64_t i = 0; i < mm * kk; ++i) v[i] = get_f64(pv + 8 * i);
  return XG_OK;
}

}  // extern "C"
