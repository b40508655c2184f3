// xg_hash.cpp -- content_hash_u64 of an encoding basis (model.cpp:99-114):
// 64-bit FNV-1a over "XENC", the mode byte, m, k (little-endian u64) and the
// f64 bits of V.  Host metadata only; the basis itself is built on the
// device (K9, xg_api.cu: xg_series_build_basis / xg_build_basis).
#include <cstdint>
#include <cstring>

#include "../../include/xpcs_b200.h"

extern "C" {

XG_API uint64_t xg_content_hash(const double* v, int64_t m, int64_t k, int32_t mode) {
  uint64_t h = 0xCBF29CE484222325ULL;
  auto feed = [&](const unsigned char* p, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      h ^= p[i];
      h *= 0x100000001B3ULL;
    }
  };
  auto feed_u64 = [&](uint64_t x) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(x >> (8 * i));
    feed(b, 8);
  };
  feed(reinterpret_cast<const unsigned char*>("XENC"), 4);
  const unsigned char md = static_cast<unsigned char>(mode);
  feed(&md, 1);
  feed_u64(static_cast<uint64_t>(m));
  feed_u64(static_cast<uint64_t>(k));
  for (int64_t i = 0; i < m * k; ++i) {
    uint64_t bits;
    std::memcpy(&bits, v + i, 8);
    feed_u64(bits);
  }
  return h;
}

}  // extern "C"
