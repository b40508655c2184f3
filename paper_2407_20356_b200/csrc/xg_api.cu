// xg_api.cu -- host runtime behind the C ABI (include/xpcs_b200.h).
//
// Owns device memory, the CUDA stream, TMA tensor maps and the tile lists;
// validates arguments with the reference's error taxonomy
// (include/xpcsvd/errors.hpp) and launches the sm_100a kernels.  There is no
// CPU compute path: every numeric result comes from a kernel in this library.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/xpcs_b200.h"
#include "xg_kernels.h"

using namespace xg;

namespace {

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

struct Status {
  int code;
};

}  // namespace

struct xg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 0;
  std::string err;
  int64_t payload = -1;
  int32_t payload_ring = -1;
  int* d_err = nullptr;  // device error word (pipeline timeouts, overflow)
  int64_t launches = 0;
  PFN_encodeTiled encode = nullptr;
  cudaStream_t copy_stream = nullptr;    // host -> device copies overlapped with compute
  std::vector<cudaEvent_t> events;       // chunk-arrival events (reused)
  void* scratch = nullptr;               // readback staging (grown, reused: no malloc/free
  size_t scratch_cap = 0;                // per call, so pinned readbacks run at PCIe speed)
};

struct xg_layout {
  xg_ctx* ctx = nullptr;
  int64_t pixels = 0;
  int32_t rings = 0;
  int32_t band = 16384;
  int32_t n_bands = 0;
  int64_t ktot = 0;
  int32_t max_words = 0, max_bytes = 0, max_band_pieces = 0;
  std::vector<int64_t> ring_pixels, kpad, koff;
  std::vector<int64_t> mask_off;  // [rings + 1] offsets into colpos (mask order)
  std::vector<int64_t> colpos;    // ring-major column of every mask entry
  std::vector<int32_t> colpix;    // [ktot] detector pixel of every column (-1 = padding)
  int32_t* d_band_piece = nullptr;
  Piece* d_pieces = nullptr;
  int32_t* d_band_word = nullptr;
  uint16_t* d_words = nullptr;
  int32_t* d_band_byte = nullptr;
  uint16_t* d_bytes = nullptr;
  int32_t* d_ring_koff = nullptr;
  int32_t* d_ring_nkb = nullptr;
  int32_t width = 0, height = 0, blocks_x = 0;  // 2D bands (xg_layout_create_2d)
  // Ring-major frames (and basis digits) ring-BLOCKED -- ring q's frames a
  // contiguous [rows][kpad_q] block -- when a ring-major row is long (C3-C5:
  // a TMA box of 128 frame rows then spans 128 kpad_q bytes instead of
  // 128 ktot, C4 K2 104.7 -> 82.6 ms, C5 K3 2.2x); else rows interleaved
  // [frame][ktot] (C2: one frame's ingest writes stay in 262 KB, 0.39 ms vs
  // 0.43 ms blocked).
  bool blocked = false;
};

// Ring q's part of a [rows] x ktot ring-major buffer: element offset of its
// first row and its row stride.
static int64_t ring_base(const xg_layout* L, int64_t rows, int32_t q) {
  return L->blocked ? rows * L->koff[q] : L->koff[q];
}
static int64_t ring_ld(const xg_layout* L, int32_t q) {
  return L->blocked ? L->kpad[q] : L->ktot;
}

struct xg_series {
  xg_ctx* ctx = nullptr;
  const xg_layout* L = nullptr;
  int64_t tmax = 0;
  int64_t t = 0;
  int64_t tp = 0;  // padded frame count (Gram leading dimension)
  uint8_t* d_raster = nullptr;
  uint8_t* d_x = nullptr;
  // photon-event loads (xg_series_load_events): pixel -> (ring, column)
  // table and grow-only staging for host event lists
  int32_t* d_pixcol = nullptr;
  int64_t* d_evoff = nullptr;
  int32_t* d_evpix = nullptr;
  uint8_t* d_evval = nullptr;
  int64_t evoff_cap = 0, ev_cap = 0;
  int64_t* d_norm2 = nullptr;
  double* d_norms = nullptr;
  double* d_inv = nullptr;
  float2* d_inv2 = nullptr;        // (hi, lo) split of d_inv for the FP32 g2
  int64_t* d_zero = nullptr;
  int64_t* d_first_zero = nullptr;
  int64_t* d_max_norm2 = nullptr;  // max |x_t|^2 over all frames and rings
  int32_t* d_gram = nullptr;
  double* d_g2 = nullptr;
  int64_t* d_g2cnt = nullptr;
  double* d_g2part = nullptr;
  int64_t* d_g2pcnt = nullptr;
  uint32_t* d_nz_bits = nullptr;   // [ring][nz_words] nonzero-frame bitmask
  int32_t nz_words = 0;
  float2* d_g2tile = nullptr;      // [ntiles][384] fused-g2 tile diagonal sums (hi, lo)
  double* d_g2runs = nullptr;      // [ring][2 nbj][384] their per-delta run sums (g2 fold)
  int32_t tiles_per_ring = 0;
  TileDesc* d_tiles = nullptr;
  TileDesc* d_tiles2 = nullptr;    // 256 x 256 pair tiles
  int32_t ntiles2 = 0;
  TileDesc* d_tiles2_j = nullptr;  // the same tiles ordered by column block J
  std::vector<int32_t> tiles2_joff;  // [nbj + 1] offsets of each J in d_tiles2_j
  int32_t ntiles = 0;
  int64_t tiles_for_t = -1;
  size_t g2part_cap = 0;
  bool have_raw = false;
  bool raw_stored = false, cmp_stored = false;  // TTC tiles written (not XG_NO_STORE)
  int64_t xmax = 0;    // frames the ring-major buffer holds (= tmax unless chunked)
  int64_t x_row0 = 0;  // series frame index of ring-major row 0  // TTC tiles written (not XG_NO_STORE)
  // compressed path (allocated on first xg_compress)
  int32_t ck = 0, ckp = 0;         // rank and plane row length of the last compress
  double* d_y = nullptr;           // [ring][tp][k] coefficients
  __nv_bfloat16* d_planes = nullptr;  // [(ring*3+s)*tp + t][kp]
  float* d_cgram = nullptr;        // [ring][tp][tp] C~ upper tiles
  double* d_cg2 = nullptr;
  int64_t* d_cg2cnt = nullptr;
  bool have_y = false, have_cttc = false;
  bool raw_g2 = false, cmp_g2 = false;  // g2 curves current (not XG_NO_G2)
  void* d_spec = nullptr;           // XG_G2_SPECTRAL scratch (kept for the next call)
  size_t spec_cap = 0;
  TileDesc* d_ptiles = nullptr;    // projection tiles
  int32_t n_ptiles = 0;
  int64_t ptiles_key = -1;
  unsigned int* d_wave = nullptr;  // K2 wave-gate counter (zeroed before each launch)
  CUtensorMap* d_xmaps = nullptr;  // per-ring TMA maps of the ring blocks of x
  int64_t xmaps_rows = -1;         // frame rows they were encoded for (zero fill beyond)
};

struct xg_basis {
  xg_ctx* ctx = nullptr;
  const xg_layout* L = nullptr;
  int32_t k = 0, digits = 3, kt = 0, ntiles_n = 0;
  int64_t vrows = 0;               // digit rows = ntiles_n * digits * kt
  std::vector<int8_t> h_vd;        // [vrows][ktot]
  std::vector<double> h_scale;     // [rings][k]
  std::vector<uint8_t> ring_set;
  int8_t* d_vd = nullptr;           // ring-blocked digits: ring q at vrows koff_q, [vrows][kpad_q]
  double* d_scale = nullptr;
  CUtensorMap* d_vmaps = nullptr;   // per-ring TMA maps of the digit blocks
  bool dirty = true;
};

namespace {

constexpr int64_t kNoZero = 0x7F7F7F7F7F7F7F7FLL;  // "no zero frame" sentinel

int fail(xg_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (code != XG_ERR_NORMALIZATION && code != XG_ERR_RANK) {
      c->payload = -1;
      c->payload_ring = -1;
    }
  }
  return code;
}

int cuda_fail(xg_ctx* c, cudaError_t e, const char* what) {
  return fail(c, XG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define XG_CUDA(c, expr)                                  \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return cuda_fail((c), _e, #expr); \
  } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int make_map_bf16_box(xg_ctx* c, CUtensorMap* map, const void* base, int64_t cols, int64_t rows,
                      uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 2)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, XG_ERR_CUDA, "cuTensorMapEncodeTiled(bf16) failed (%d)", (int)r);
  return XG_OK;
}

int make_map_bf16(xg_ctx* c, CUtensorMap* map, const void* base, int64_t cols, int64_t rows) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 2)};
  cuuint32_t box[2] = {64, 128};  // 128-byte rows
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, XG_ERR_CUDA, "cuTensorMapEncodeTiled(bf16) failed (%d)", (int)r);
  return XG_OK;
}

// 32-bit output map for the Gram epilogue's 32 x 32 TMA stores
int make_map_out32(xg_ctx* c, CUtensorMap* map, const void* base, int64_t ld, int64_t rows) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, XG_ERR_CUDA, "cuTensorMapEncodeTiled(out) failed (%d)", (int)r);
  return XG_OK;
}

int make_map_u8(xg_ctx* c, CUtensorMap* map, const void* base, int64_t cols, int64_t rows,
                int64_t row_stride, uint32_t box_cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, XG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return XG_OK;
}

// Per-ring 2D TMA maps (128-byte x box_rows boxes, 128B swizzle) of ring-
// blocked u8 data: ring q's block starts at base + rows_cap * koff_q and holds
// `rows` valid rows of kpad_q bytes (rows beyond read as zeros).  Encoded on
// the host and copied (stream-ordered) to the device array *dev.
int upload_ring_maps(xg_ctx* c, const xg_layout* L, const uint8_t* base, int64_t rows_cap,
                     int64_t rows, uint32_t box_rows, CUtensorMap** dev) {
  std::vector<CUtensorMap> maps(static_cast<size_t>(L->rings));
  for (int32_t r = 0; r < L->rings; ++r) {
    const int rc = make_map_u8(c, &maps[r], base + ring_base(L, rows_cap, r), L->kpad[r], rows,
                               ring_ld(L, r), 128, box_rows);
    if (rc) return rc;
  }
  if (!*dev) XG_CUDA(c, dalloc(dev, maps.size()));
  // pageable source: staged before the call returns; stream-ordered after
  // every earlier kernel that read the previous maps
  XG_CUDA(c, cudaMemcpyAsync(*dev, maps.data(), maps.size() * sizeof(CUtensorMap),
                             cudaMemcpyHostToDevice, c->stream));
  return XG_OK;
}

// The context's readback staging buffer, at least `bytes` large.
cudaError_t ctx_scratch(xg_ctx* c, size_t bytes, void** out) {
  if (bytes > c->scratch_cap) {
    if (c->scratch) {
      cudaStreamSynchronize(c->stream);
      cudaFree(c->scratch);
      c->scratch = nullptr;
      c->scratch_cap = 0;
    }
    const cudaError_t e = cudaMalloc(&c->scratch, bytes);
    if (e != cudaSuccess) return e;
    c->scratch_cap = bytes;
  }
  *out = c->scratch;
  return cudaSuccess;
}

// Device error word: bit0 pipeline timeout, bit2 int32 Gram overflow.
int check_device_error(xg_ctx* c) {
  int h = 0;
  XG_CUDA(c, cudaMemcpyAsync(&h, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  if (h & 1) {
    cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream);
    return fail(c, XG_ERR_DEVICE, "tensor-core pipeline self-check failed (mbarrier timeout)");
  }
  if (h & 4) {
    cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream);
    return fail(c, XG_ERR_CONTRACT,
                "ttc_raw: a frame norm^2 exceeds 2^31-1; the exact int32 Gram would overflow");
  }
  if (h & 8) {
    cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream);
    return fail(c, XG_ERR_SHAPE, "load_events: a pixel index outside [0, full_pixels)");
  }
  return XG_OK;
}

}  // namespace

extern "C" {

int xg_version(void) { return 100; }

int xg_ctx_create(int device, void* stream, xg_ctx** out) {
  if (!out) return XG_ERR_INVALID;
  *out = nullptr;
  xg_ctx* c = new xg_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete c;
    return XG_ERR_CUDA;
  }
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess || prop.major != 10) {
    delete c;
    return XG_ERR_DEVICE;  // sm_100a kernels only
  }
  c->num_sms = prop.multiProcessorCount;
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    c->own_stream = true;
  }
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn) {
    delete c;
    return XG_ERR_CUDA;
  }
  c->encode = reinterpret_cast<PFN_encodeTiled>(fn);
  if (cudaMalloc(&c->d_err, sizeof(int)) != cudaSuccess) {
    delete c;
    return XG_ERR_CUDA;
  }
  cudaMemset(c->d_err, 0, sizeof(int));
  *out = c;
  return XG_OK;
}

void xg_ctx_destroy(xg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->d_err) cudaFree(c->d_err);
  if (c->scratch) cudaFree(c->scratch);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (cudaEvent_t ev : c->events) cudaEventDestroy(ev);
  delete c;
}

const char* xg_last_error(const xg_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t xg_last_error_payload(const xg_ctx* c, int32_t* ring) {
  if (!c) return -1;
  if (ring) *ring = c->payload_ring;
  return c->payload;
}

int xg_synchronize(xg_ctx* c) {
  if (!c) return XG_ERR_INVALID;
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

int64_t xg_kernel_launches(const xg_ctx* c) { return c ? c->launches : -1; }

// ------------------------------------------------------------------ layout
// Layout builder.  width > 0 (a height x width row-major detector wider than
// one 512-pixel piece): K1 bands are blocks of 32 rows x 512 columns, else
// 16384-pixel raster strips.  A ring's pixels in one band form one segment
// of its ring-major row.
static int layout_build(xg_ctx* c, int64_t full_pixels, int64_t height, int64_t width,
                        int32_t n_rings, const int64_t* offsets, const int64_t* indices,
                        xg_layout** out) {
  if (!c || !out || !offsets || !indices) return XG_ERR_INVALID;
  *out = nullptr;
  if (full_pixels < 1) return fail(c, XG_ERR_CONTRACT, "layout: full_pixels must be >= 1");
  if (n_rings < 1) return fail(c, XG_ERR_CONTRACT, "layout: need at least one ring");
  // PixelMask validation (model.cpp:10-26) for every ring.
  for (int32_t r = 0; r < n_rings; ++r) {
    const int64_t b = offsets[r], e = offsets[r + 1];
    if (e <= b) return fail(c, XG_ERR_MASK, "pixel mask %d selects no pixels", r);
    for (int64_t i = b; i < e; ++i) {
      if (indices[i] < 0 || indices[i] >= full_pixels)
        return fail(c, XG_ERR_MASK, "mask %d index %lld out of range for %lld pixels", r,
                    (long long)indices[i], (long long)full_pixels);
      if (i > b && indices[i] <= indices[i - 1])
        return fail(c, XG_ERR_MASK, "mask %d indices not strictly ascending at position %lld",
                    r, (long long)(i - b));
    }
  }
  xg_layout* L = new xg_layout();
  L->ctx = c;
  L->pixels = full_pixels;
  L->rings = n_rings;
  // 16384-pixel bands: a consumer pass moves twice the bytes of an 8192
  // band for the same bookkeeping (measured: K1 0.475 -> 0.441 ms at C2;
  // 4096 and >= 24576 are slower: fewer passes vs fewer CTAs per SM).  On a
  // wide detector a 16384-pixel raster strip is only 16384 / W rows tall, so
  // an annulus crosses it in many short segments (C5: 8 rows, ~200 segments
  // per band, K1 at 0.45 of HBM): 2D bands of 32 rows x 512 columns keep the
  // segments as long as on a 512-wide detector (the band of C2), and keep
  // the shared-memory layout (one 512-byte piece per row).  128 x 128 blocks
  // were slower (short row runs -> few whole words: C5 8.8 -> 10.8 ms).
  const bool two_d = width > kBandW && width % 16 == 0;
  if (two_d) {
    L->width = static_cast<int32_t>(width);
    L->height = static_cast<int32_t>(height);
    L->blocks_x = static_cast<int32_t>((width + kBandW - 1) / kBandW);
    L->band = kBandH * kBandW;
    L->n_bands = L->blocks_x * static_cast<int32_t>((height + kBandH - 1) / kBandH);
  } else {
    L->band = static_cast<int32_t>(std::min<int64_t>(16384, round_up(full_pixels, 16)));
    L->n_bands = static_cast<int32_t>((full_pixels + L->band - 1) / L->band);
  }
  const int32_t nb = L->n_bands;
  // band of a detector pixel and its index e inside the band (2D: row-major
  // in a 512-wide block, so e's shared-memory byte is ingest_smem_offset(e)
  // in both forms)
  auto band_of = [&](int64_t px) -> int32_t {
    if (!two_d) return static_cast<int32_t>(px / L->band);
    return static_cast<int32_t>((px / width) / kBandH * L->blocks_x + (px % width) / kBandW);
  };
  auto e_of = [&](int64_t px) -> int32_t {
    if (!two_d) return static_cast<int32_t>(px % L->band);
    return static_cast<int32_t>((px / width) % kBandH * kBandW + (px % width) % kBandW);
  };
  auto smem_of = [&](int32_t e) -> int32_t { return ingest_smem_offset(e); };
  // mask entries bucketed by band: ring order, ascending inside a ring
  std::vector<int64_t> cnt(static_cast<size_t>(n_rings) * nb, 0);
  std::vector<int64_t> bstart(static_cast<size_t>(nb) + 1, 0);
  for (int32_t r = 0; r < n_rings; ++r)
    for (int64_t i = offsets[r]; i < offsets[r + 1]; ++i) {
      const int32_t b = band_of(indices[i]);
      cnt[(size_t)r * nb + b]++;
      bstart[b + 1]++;
    }
  for (int32_t b = 0; b < nb; ++b) bstart[b + 1] += bstart[b];
  std::vector<int64_t> bucket(static_cast<size_t>(offsets[n_rings]));
  {
    std::vector<int64_t> fill(bstart.begin(), bstart.end() - 1);
    for (int32_t r = 0; r < n_rings; ++r)
      for (int64_t i = offsets[r]; i < offsets[r + 1]; ++i) bucket[fill[band_of(indices[i])]++] = i;
  }
  L->ring_pixels.resize(n_rings);
  L->mask_off.assign(offsets, offsets + n_rings + 1);
  L->colpos.assign(static_cast<size_t>(offsets[n_rings]), 0);
  L->kpad.resize(n_rings);
  L->koff.resize(n_rings);
  std::vector<int64_t> segoff(static_cast<size_t>(n_rings) * nb, 0);
  int64_t koff = 0;
  for (int32_t r = 0; r < n_rings; ++r) {
    int64_t k = 0;
    for (int32_t b = 0; b < nb; ++b) {
      segoff[(size_t)r * nb + b] = k;
      k += round_up(cnt[(size_t)r * nb + b], 4);  // 4-byte segments: K1 stores words
    }
    L->ring_pixels[r] = offsets[r + 1] - offsets[r];
    L->kpad[r] = std::max<int64_t>(128, round_up(k, 128));
    L->koff[r] = koff;
    koff += L->kpad[r];
  }
  L->ktot = koff;
  L->blocked = L->ktot > 400000;
  if (L->ktot > INT32_MAX) {
    delete L;
    return fail(c, XG_ERR_CONTRACT, "layout: padded ring width exceeds 2^31 bytes");
  }
  // Per band: segments in ring order.  A segment's output is its whole
  // source words (round-robin over smem banks, so the 32 words a warp loads
  // at once sit in distinct banks) followed by its remaining pixels packed
  // 4 per group; colpos records where every mask entry lands.
  const int32_t bstride = ingest_band_stride(L->band);
  const uint16_t zero_at = static_cast<uint16_t>(bstride - 16);
  std::vector<int32_t> band_word(nb + 1, 0), band_byte(nb + 1, 0);
  std::vector<uint16_t> words, bytes;
  std::vector<Piece> pieces;
  constexpr int kWarps = INGEST_CONSUMERS;
  std::vector<int32_t> band_piece((size_t)nb * (kWarps + 1) + 1, 0);
  std::vector<int64_t> pos(static_cast<size_t>(L->band), -1);  // band pixel -> mask entry
  struct Seg { int32_t ring, dst, nw, woff, nb, boff; };
  for (int32_t b = 0; b < nb; ++b) {
    band_word[b] = static_cast<int32_t>(words.size());
    band_byte[b] = static_cast<int32_t>(bytes.size() / 4);
    std::vector<Seg> sg;
    int64_t cur = bstart[b];
    for (int32_t r = 0; r < n_rings; ++r) {
      const int64_t n = cnt[(size_t)r * nb + b];
      if (n == 0) continue;
      const int64_t* ent = bucket.data() + cur;  // this ring's mask entries in the band
      std::vector<int32_t> ex(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) {
        ex[i] = e_of(indices[ent[i]]);
        pos[ex[i]] = ent[i];
      }
      std::vector<int32_t> bank_words[32], left;
      for (int64_t i = 0; i < n; ++i) {
        const int32_t e = ex[i];
        if ((e & 3) == 0 && i + 3 < n && ex[i + 3] == e + 3) {  // ascending => all 4 in ring
          bank_words[(smem_of(e) / 4) & 31].push_back(e);
          i += 3;
        } else {
          left.push_back(e);
        }
      }
      Seg s;
      s.ring = r;
      s.dst = static_cast<int32_t>(L->koff[r] + segoff[(size_t)r * nb + b]);
      s.woff = static_cast<int32_t>(words.size()) - band_word[b];
      s.boff = static_cast<int32_t>(bytes.size() / 4) - band_byte[b];
      int32_t g = 0;
      size_t next[32] = {0};
      for (bool any = true; any;) {
        any = false;
        for (int k = 0; k < 32; ++k) {
          if (next[k] == bank_words[k].size()) continue;
          const int32_t e = bank_words[k][next[k]++];
          any = true;
          words.push_back(static_cast<uint16_t>(smem_of(e) / 4));
          for (int j = 0; j < 4; ++j) L->colpos[pos[e + j]] = s.dst + 4 * g + j;
          ++g;
        }
      }
      s.nw = g;
      const size_t nl = left.size(), nlp = static_cast<size_t>(round_up((int64_t)nl, 4));
      for (size_t q = 0; q < nlp; ++q) {
        if (q < nl) {
          bytes.push_back(static_cast<uint16_t>(smem_of(left[q])));
          L->colpos[pos[left[q]]] = s.dst + 4 * g + static_cast<int64_t>(q);
        } else {
          bytes.push_back(zero_at);
        }
      }
      s.nb = static_cast<int32_t>(nlp / 4);
      sg.push_back(s);
      cur += n;
    }
    // Split the band's groups over the consumer warps by estimated cost
    // (a word group ~2 shared-memory wavefronts, a byte group ~5).
    std::vector<int64_t> seg_cost(sg.size() + 1, 0);
    for (size_t i = 0; i < sg.size(); ++i) seg_cost[i + 1] = seg_cost[i] + 2 * sg[i].nw + 5 * sg[i].nb;
    const int64_t total = seg_cost.back();
    size_t si = 0;
    int32_t j0 = 0;  // next unassigned group of segment si
    for (int w = 0; w < kWarps; ++w) {
      band_piece[(size_t)b * (kWarps + 1) + w] = static_cast<int32_t>(pieces.size());
      const int64_t target = total * (w + 1) / kWarps;
      while (si < sg.size()) {
        const Seg& s = sg[si];
        const int32_t ng = s.nw + s.nb;
        // groups of this segment that fit below the target
        int32_t j1 = ng;
        if (w + 1 < kWarps) {
          int64_t c = seg_cost[si];
          j1 = 0;
          while (j1 < ng && c + (j1 < s.nw ? 2 : 5) <= target) c += (j1++ < s.nw ? 2 : 5);
          // c now includes groups [0, j1)
          if (j1 < j0) j1 = j0;
        }
        if (j1 > j0) {
          Piece pc{};
          pc.ring = s.ring;
          pc.dst = s.dst + 4 * j0;
          pc.n_word = std::max(0, std::min(j1, s.nw) - j0);
          pc.word_off = s.woff + std::min(j0, s.nw);
          pc.n_byte = (j1 - j0) - pc.n_word;
          pc.byte_off = s.boff + std::max(0, j0 - s.nw);
          // K1 writes frame row r of the piece at x + xmax koff + r kpad + (dst - koff):
          // ring-blocked, or (koff 0, kpad ktot) the interleaved rows
          pc.koff = L->blocked ? static_cast<int32_t>(L->koff[s.ring]) : 0;
          pc.kpad = static_cast<int32_t>(L->blocked ? L->kpad[s.ring] : L->ktot);
          pieces.push_back(pc);
        }
        if (j1 < ng) { j0 = j1; break; }
        ++si;
        j0 = 0;
      }
    }
    band_piece[(size_t)b * (kWarps + 1) + kWarps] = static_cast<int32_t>(pieces.size());
    L->max_words = std::max(L->max_words, static_cast<int32_t>(words.size()) - band_word[b]);
    L->max_bytes =
        std::max(L->max_bytes, static_cast<int32_t>(bytes.size() / 4) - band_byte[b]);
    L->max_band_pieces = std::max(
        L->max_band_pieces, band_piece[(size_t)b * (kWarps + 1) + kWarps] -
                                band_piece[(size_t)b * (kWarps + 1)]);
  }
  L->colpix.assign(static_cast<size_t>(L->ktot), -1);
  for (int64_t i = 0; i < offsets[n_rings]; ++i) L->colpix[L->colpos[i]] = static_cast<int32_t>(indices[i]);
  band_word[nb] = static_cast<int32_t>(words.size());
  band_byte[nb] = static_cast<int32_t>(bytes.size() / 4);
  if (words.empty()) words.push_back(0);
  if (bytes.empty()) bytes.assign(4, zero_at);
  if (pieces.empty()) pieces.push_back(Piece{});
  std::vector<int32_t> rk(n_rings), rn(n_rings);
  for (int32_t r = 0; r < n_rings; ++r) {
    rk[r] = static_cast<int32_t>(L->koff[r]);
    rn[r] = static_cast<int32_t>(L->kpad[r] / 128);
  }
  cudaError_t e = cudaSuccess;
  if ((e = dalloc(&L->d_band_piece, band_piece.size())) != cudaSuccess ||
      (e = dalloc(&L->d_pieces, pieces.size())) != cudaSuccess ||
      (e = dalloc(&L->d_band_word, band_word.size())) != cudaSuccess ||
      (e = dalloc(&L->d_words, words.size())) != cudaSuccess ||
      (e = dalloc(&L->d_band_byte, band_byte.size())) != cudaSuccess ||
      (e = dalloc(&L->d_bytes, bytes.size())) != cudaSuccess ||
      (e = dalloc(&L->d_ring_koff, rk.size())) != cudaSuccess ||
      (e = dalloc(&L->d_ring_nkb, rn.size())) != cudaSuccess) {
    xg_layout_destroy(L);
    return cuda_fail(c, e, "layout alloc");
  }
  cudaMemcpy(L->d_band_piece, band_piece.data(), band_piece.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(L->d_pieces, pieces.data(), pieces.size() * sizeof(Piece), cudaMemcpyHostToDevice);
  cudaMemcpy(L->d_band_word, band_word.data(), band_word.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(L->d_words, words.data(), words.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(L->d_band_byte, band_byte.data(), band_byte.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(L->d_bytes, bytes.data(), bytes.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(L->d_ring_koff, rk.data(), rk.size() * 4, cudaMemcpyHostToDevice);
  e = cudaMemcpy(L->d_ring_nkb, rn.data(), rn.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    xg_layout_destroy(L);
    return cuda_fail(c, e, "layout upload");
  }
  *out = L;
  return XG_OK;
}

int xg_layout_create(xg_ctx* c, int64_t full_pixels, int32_t n_rings, const int64_t* offsets,
                     const int64_t* indices, xg_layout** out) {
  return layout_build(c, full_pixels, 0, 0, n_rings, offsets, indices, out);
}

int xg_layout_create_2d(xg_ctx* c, int64_t height, int64_t width, int32_t n_rings,
                        const int64_t* offsets, const int64_t* indices, xg_layout** out) {
  if (!c) return XG_ERR_INVALID;
  if (height < 1 || width < 1 || height > INT32_MAX || width > INT32_MAX)
    return fail(c, XG_ERR_CONTRACT, "layout: detector height and width must be >= 1");
  return layout_build(c, height * width, height, width, n_rings, offsets, indices, out);
}

void xg_layout_destroy(xg_layout* L) {
  if (!L) return;
  dfree(L->d_band_piece);
  dfree(L->d_pieces);
  dfree(L->d_band_word);
  dfree(L->d_words);
  dfree(L->d_band_byte);
  dfree(L->d_bytes);
  dfree(L->d_ring_koff);
  dfree(L->d_ring_nkb);
  delete L;
}

int64_t xg_layout_ring_pixels(const xg_layout* L, int32_t ring) {
  if (!L || ring < 0 || ring >= L->rings) return -1;
  return L->ring_pixels[ring];
}

// ------------------------------------------------------------------ series
int xg_series_create(xg_ctx* c, const xg_layout* L, int64_t max_frames, xg_series** out) {
  return xg_series_create2(c, L, max_frames, max_frames, out);
}

int xg_series_create2(xg_ctx* c, const xg_layout* L, int64_t max_frames, int64_t x_frames,
                      xg_series** out) {
  if (!c || !L || !out) return XG_ERR_INVALID;
  *out = nullptr;
  if (max_frames < 2) return fail(c, XG_ERR_CONTRACT, "series: need at least 2 frames");
  if (x_frames < 1 || x_frames > max_frames)
    return fail(c, XG_ERR_CONTRACT, "series: x_frames must be in [1, max_frames]");
  xg_series* s = new xg_series();
  s->ctx = c;
  s->L = L;
  s->tmax = max_frames;
  s->xmax = x_frames;
  s->tp = round_up(max_frames, 256);
  const int64_t Q = L->rings;
  cudaError_t e = cudaSuccess;
  // d_raster (the H2D staging raster) is allocated on the first host load:
  // device-resident frames never need it (C4: 17 GB saved)
  if ((e = dalloc(&s->d_x, (size_t)x_frames * L->ktot)) != cudaSuccess ||
      (e = dalloc(&s->d_norm2, (size_t)max_frames * Q)) != cudaSuccess ||
      (e = dalloc(&s->d_norms, (size_t)s->tp * Q)) != cudaSuccess ||
      (e = dalloc(&s->d_inv, (size_t)s->tp * Q)) != cudaSuccess ||
      (e = dalloc(&s->d_inv2, (size_t)s->tp * Q)) != cudaSuccess ||
      (e = dalloc(&s->d_zero, (size_t)Q)) != cudaSuccess ||
      (e = dalloc(&s->d_first_zero, (size_t)Q)) != cudaSuccess ||
      (e = dalloc(&s->d_max_norm2, (size_t)1)) != cudaSuccess ||
      (e = dalloc(&s->d_g2, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_g2cnt, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_g2part, (size_t)Q * 8 * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_g2pcnt, (size_t)Q * 8 * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_nz_bits, (size_t)Q * (s->tp / 32))) != cudaSuccess) {
    xg_series_destroy(s);
    return cuda_fail(c, e, "series alloc");
  }
  s->g2part_cap = (size_t)Q * 8 * s->tp;
  // padding columns of the ring-major rows must stay zero forever
  e = cudaMemsetAsync(s->d_x, 0, (size_t)x_frames * L->ktot, c->stream);
  if (e != cudaSuccess) {
    xg_series_destroy(s);
    return cuda_fail(c, e, "series memset");
  }
  *out = s;
  return XG_OK;
}

void xg_series_destroy(xg_series* s) {
  if (!s) return;
  dfree(s->d_raster);
  dfree(s->d_pixcol);
  dfree(s->d_evoff);
  dfree(s->d_evpix);
  dfree(s->d_evval);
  dfree(s->d_x);
  dfree(s->d_norm2);
  dfree(s->d_norms);
  dfree(s->d_inv);
  dfree(s->d_inv2);
  dfree(s->d_zero);
  dfree(s->d_first_zero);
  dfree(s->d_max_norm2);
  dfree(s->d_gram);
  dfree(s->d_g2);
  dfree(s->d_g2cnt);
  dfree(s->d_g2part);
  dfree(s->d_g2pcnt);
  dfree(s->d_tiles);
  dfree(s->d_tiles2);
  dfree(s->d_tiles2_j);
  dfree(s->d_nz_bits);
  dfree(s->d_g2tile);
  dfree(s->d_g2runs);
  dfree(s->d_y);
  dfree(s->d_planes);
  dfree(s->d_cgram);
  dfree(s->d_cg2);
  dfree(s->d_spec);
  dfree(s->d_cg2cnt);
  dfree(s->d_ptiles);
  dfree(s->d_wave);
  dfree(s->d_xmaps);
  delete s;
}

int64_t xg_series_frames(const xg_series* s) { return s ? s->t : -1; }

// Stored-TTC geometry (ttc_off, xg_kernels.h): one slab of packed upper pair
// tiles per ring, sized for the series' capacity; the tiles of the current
// frames use ttc_nb(s) per row.
static int64_t slab_elems(const xg_series* s) { return ttc_slab(s->tp / 256); }
static int32_t ttc_nb(const xg_series* s) { return static_cast<int32_t>((s->t + 255) / 256); }

// Per-ring TMA maps of the series' ring blocks for `rows` valid frames.
static int ensure_xmaps(xg_series* s, int64_t rows) {
  if (s->xmaps_rows == rows && s->d_xmaps) return XG_OK;
  const int rc = upload_ring_maps(s->ctx, s->L, s->d_x, s->xmax, rows, 128, &s->d_xmaps);
  if (rc) return rc;
  s->xmaps_rows = rows;
  return XG_OK;
}

// The staging raster for frames that arrive from host memory.
static int ensure_raster(xg_series* s) {
  if (s->d_raster) return XG_OK;
  XG_CUDA(s->ctx, dalloc(&s->d_raster, (size_t)s->xmax * s->L->pixels));
  return XG_OK;
}

// New frames replace the series: every result derived from the old ones
// (raw TTC, coefficients, compressed TTC, both g2 curves) stops being valid.
static void invalidate_results(xg_series* s) {
  s->have_raw = false;
  s->raw_stored = false;
  s->raw_g2 = false;
  s->have_y = false;
  s->have_cttc = false;
  s->cmp_stored = false;
  s->cmp_g2 = false;
}

// Ingest frames [t0, t0 + n) from a device raster whose first frame is t0:
// K1 (ring permutation + |x|^2 per (frame, ring)) and K1b (norms, 1/|x|,
// zero-frame bookkeeping).  reset_stats() must have run for this series.
static int ingest_range(xg_series* s, const uint8_t* raster, int64_t t0, int64_t n) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  IngestParams p;
  p.raster = raster;
  p.x = s->d_x;
  p.xmax = s->xmax;
  p.blocked = L->blocked ? 1 : 0;
  p.pixels = L->pixels;
  p.ktot = L->ktot;
  p.band = L->band;
  p.n_bands = L->n_bands;
  p.n_rings = L->rings;
  p.band_piece = L->d_band_piece;
  p.pieces = L->d_pieces;
  p.band_word = L->d_band_word;
  p.words = L->d_words;
  p.band_byte = L->d_band_byte;
  p.bytes = L->d_bytes;
  p.max_words = L->max_words;
  p.max_bytes = L->max_bytes;
  p.max_band_pieces = L->max_band_pieces;
  p.t0 = t0;
  p.x_row0 = s->x_row0;
  p.n_frames = n;
  p.width = L->width;
  p.height = L->height;
  p.blocks_x = L->blocks_x;
  // one wave of ~4 resident CTAs per SM, each streaming a run of frames of one band
  const int64_t want = std::max<int64_t>(1, (int64_t)c->num_sms * 4 / std::max(1, L->n_bands));
  p.frames_per_cta = static_cast<int32_t>(std::max<int64_t>(1, (n + want - 1) / want));
  p.norm2 = reinterpret_cast<unsigned long long*>(s->d_norm2);
  XG_CUDA(c, cudaMemsetAsync(s->d_norm2 + t0 * L->rings, 0, (size_t)n * L->rings * 8, c->stream));
  XG_CUDA(c, launch_ingest(p, c->stream));
  NormParams np;
  np.t0 = t0;
  np.norm2 = s->d_norm2;
  np.n_frames = n;
  np.ld = s->tp;
  np.n_rings = L->rings;
  np.norms = s->d_norms;
  np.inv = s->d_inv;
  np.inv2 = s->d_inv2;
  np.zero_count = s->d_zero;
  np.first_zero = s->d_first_zero;
  np.nz_bits = s->d_nz_bits;
  np.nz_words = s->nz_words;
  np.max_norm2 = reinterpret_cast<unsigned long long*>(s->d_max_norm2);
  np.err = nullptr;  // the int32 overflow is checked by K2, where the raw Gram is formed
  XG_CUDA(c, launch_norms(np, c->stream));
  c->launches += 2;
  return XG_OK;
}

// Series-wide statistics that the per-range ingests accumulate into.
static int reset_stats(xg_series* s, int64_t n) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  s->nz_words = static_cast<int32_t>((n + 31) / 32);
  XG_CUDA(c, cudaMemsetAsync(s->d_max_norm2, 0, 8, c->stream));
  XG_CUDA(c, cudaMemsetAsync(s->d_nz_bits, 0, (size_t)L->rings * s->nz_words * 4, c->stream));
  XG_CUDA(c, cudaMemsetAsync(s->d_zero, 0, (size_t)L->rings * 8, c->stream));
  XG_CUDA(c, cudaMemsetAsync(s->d_first_zero, 0x7F, (size_t)L->rings * 8, c->stream));
  return XG_OK;
}

int xg_series_load_frames(xg_series* s, const uint8_t* frames, int64_t n, int on_device) {
  if (!s || !frames) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (n < 1 || n > s->xmax)
    return fail(c, XG_ERR_SHAPE, "load_frames: %lld frames, capacity %lld", (long long)n,
                (long long)s->xmax);
  s->x_row0 = 0;
  const uint8_t* src = frames;
  if (!on_device) {
    if (int rc0 = ensure_raster(s)) return rc0;
    XG_CUDA(c, cudaMemcpyAsync(s->d_raster, frames, (size_t)n * L->pixels,
                               cudaMemcpyHostToDevice, c->stream));
    src = s->d_raster;
  }
  int rc = reset_stats(s, n);
  if (rc) return rc;
  invalidate_results(s);
  rc = ingest_range(s, src, 0, n);
  if (rc) return rc;
  s->t = n;
  return XG_OK;
}

// Photon-event loads: the pixel -> (ring, column) table, host-side checks of
// the offsets, staging capacity, and the per-range scatter + norms.
static int events_prepare(xg_series* s, int64_t n) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (n < 1 || n > s->xmax)
    return fail(c, XG_ERR_SHAPE, "load_events: %lld frames, capacity %lld", (long long)n,
                (long long)s->xmax);
  if (L->ktot >= (1 << 22) || L->rings > 512)
    return fail(c, XG_ERR_CONTRACT, "load_events: at most 2^22 columns and 512 rings");
  if (!s->d_pixcol) {
    std::vector<int32_t> pc(static_cast<size_t>(L->pixels), -1);
    for (int32_t r = 0; r < L->rings; ++r)
      for (int64_t col = L->koff[r]; col < L->koff[r] + L->kpad[r]; ++col)
        if (L->colpix[col] >= 0) pc[L->colpix[col]] = (r << 22) | static_cast<int32_t>(col);
    XG_CUDA(c, dalloc(&s->d_pixcol, pc.size()));
    XG_CUDA(c, cudaMemcpy(s->d_pixcol, pc.data(), pc.size() * 4, cudaMemcpyHostToDevice));
  }
  return XG_OK;
}

static int events_stage(xg_series* s, const int64_t* frame_off, const int32_t* pix,
                        const uint8_t* val, int64_t n) {
  xg_ctx* c = s->ctx;
  if (frame_off[0] != 0) return fail(c, XG_ERR_SHAPE, "load_events: frame_off[0] must be 0");
  for (int64_t f = 0; f < n; ++f)
    if (frame_off[f + 1] < frame_off[f])
      return fail(c, XG_ERR_SHAPE, "load_events: frame_off must be non-decreasing");
  const int64_t nnz = frame_off[n];
  if (nnz > 0 && (!pix || !val)) return XG_ERR_INVALID;
  if (s->evoff_cap < n + 1) {
    dfree(s->d_evoff);
    s->evoff_cap = 0;
    XG_CUDA(c, dalloc(&s->d_evoff, (size_t)(n + 1)));
    s->evoff_cap = n + 1;
  }
  if (s->ev_cap < nnz) {
    dfree(s->d_evpix);
    dfree(s->d_evval);
    s->ev_cap = 0;
    XG_CUDA(c, dalloc(&s->d_evpix, (size_t)nnz));
    XG_CUDA(c, dalloc(&s->d_evval, (size_t)nnz));
    s->ev_cap = nnz;
  }
  return XG_OK;
}

// clear rows [0, n) of the ring-major buffer (zero pixels, ring padding)
static int events_clear(xg_series* s, int64_t n) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (L->blocked) {
    for (int32_t r = 0; r < L->rings; ++r)
      XG_CUDA(c, cudaMemsetAsync(s->d_x + ring_base(L, s->xmax, r), 0,
                                 (size_t)n * ring_ld(L, r), c->stream));
  } else {
    XG_CUDA(c, cudaMemsetAsync(s->d_x, 0, (size_t)n * L->ktot, c->stream));
  }
  return XG_OK;
}

// K1e + K1b for frames [t0, t0 + n) of device event lists (global offsets)
static int events_ingest(xg_series* s, const int64_t* d_off, const int32_t* d_pix,
                         const uint8_t* d_val, int64_t t0, int64_t n) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  EventIngestParams ep;
  ep.frame_off = d_off;
  ep.t0 = t0;
  ep.pix = d_pix;
  ep.val = d_val;
  ep.n_frames = n;
  ep.pixels = L->pixels;
  ep.pixcol = s->d_pixcol;
  ep.ring_koff = L->d_ring_koff;
  ep.ring_nkb = L->d_ring_nkb;
  ep.n_rings = L->rings;
  ep.x = s->d_x;
  ep.xmax = s->xmax;
  ep.ktot = L->ktot;
  ep.blocked = L->blocked ? 1 : 0;
  ep.norm2 = reinterpret_cast<unsigned long long*>(s->d_norm2);
  ep.err = c->d_err;
  XG_CUDA(c, launch_ingest_events(ep, c->stream));
  NormParams np;
  np.t0 = t0;
  np.norm2 = s->d_norm2;
  np.n_frames = n;
  np.ld = s->tp;
  np.n_rings = L->rings;
  np.norms = s->d_norms;
  np.inv = s->d_inv;
  np.inv2 = s->d_inv2;
  np.zero_count = s->d_zero;
  np.first_zero = s->d_first_zero;
  np.nz_bits = s->d_nz_bits;
  np.nz_words = s->nz_words;
  np.max_norm2 = reinterpret_cast<unsigned long long*>(s->d_max_norm2);
  np.err = nullptr;  // the int32 overflow is checked by K2, where the raw Gram is formed
  XG_CUDA(c, launch_norms(np, c->stream));
  c->launches += 2;
  return XG_OK;
}

int xg_series_load_events(xg_series* s, const int64_t* frame_off, const int32_t* pix,
                          const uint8_t* val, int64_t n, int on_device) {
  if (!s || !frame_off) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  int rc = events_prepare(s, n);
  if (rc) return rc;
  const int64_t* d_off = frame_off;
  const int32_t* d_pix = pix;
  const uint8_t* d_val = val;
  if (!on_device) {
    rc = events_stage(s, frame_off, pix, val, n);
    if (rc) return rc;
    const int64_t nnz = frame_off[n];
    XG_CUDA(c, cudaMemcpyAsync(s->d_evoff, frame_off, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice,
                               c->stream));
    if (nnz > 0) {
      XG_CUDA(c, cudaMemcpyAsync(s->d_evpix, pix, (size_t)nnz * 4, cudaMemcpyHostToDevice, c->stream));
      XG_CUDA(c, cudaMemcpyAsync(s->d_evval, val, (size_t)nnz, cudaMemcpyHostToDevice, c->stream));
    }
    d_off = s->d_evoff;
    d_pix = s->d_evpix;
    d_val = s->d_evval;
  }
  s->x_row0 = 0;
  rc = reset_stats(s, n);
  if (rc) return rc;
  invalidate_results(s);
  rc = events_clear(s, n);
  if (rc) return rc;
  rc = events_ingest(s, d_off, d_pix, d_val, 0, n);
  if (rc) return rc;
  s->t = n;
  return XG_OK;
}

static int build_tiles(xg_series* s) {
  xg_ctx* c = s->ctx;
  if (s->tiles_for_t == s->t) return XG_OK;
  std::vector<TileDesc> tiles;
  const int64_t nbi = (s->t + 127) / 128, nbj = (s->t + 255) / 256;
  for (int32_t r = 0; r < s->L->rings; ++r)
    for (int64_t ib = 0; ib < nbi; ++ib)
      for (int64_t jb = (ib * 128) / 256; jb < nbj; ++jb) {
        TileDesc d;
        d.ring = r;
        d.i0 = static_cast<int32_t>(ib * 128);
        d.j0 = static_cast<int32_t>(jb * 256);
        d.pad = 0;
        tiles.push_back(d);
      }
  // tile offset of each tile row within a ring (pair-tile pad indices below)
  std::vector<int32_t> iboff(nbi + 1, 0);
  for (int64_t ib = 0; ib < nbi; ++ib) iboff[ib + 1] = iboff[ib] + static_cast<int32_t>(nbj - ib / 2);
  s->tiles_per_ring = iboff[nbi];
  dfree(s->d_tiles);
  dfree(s->d_g2tile);
  dfree(s->d_g2runs);
  XG_CUDA(c, dalloc(&s->d_tiles, tiles.size()));
  XG_CUDA(c, dalloc(&s->d_g2tile, tiles.size() * 384));
  XG_CUDA(c, dalloc(&s->d_g2runs, (size_t)s->L->rings * 2 * nbj * 384));
  XG_CUDA(c, cudaMemcpy(s->d_tiles, tiles.data(), tiles.size() * sizeof(TileDesc),
                        cudaMemcpyHostToDevice));
  s->ntiles = static_cast<int32_t>(tiles.size());
  // 256 x 256 pair tiles (k_gram2): pad = 1-CTA index of the upper half tile.
  // The persistent kernel deals consecutive tiles to the CTA pairs, so ~one
  // wave of (SMs / 2) consecutive tiles is in flight at once.  Tiles are
  // listed ring by ring in 8 x 8 super-tiles (row-major inside): a wave then
  // reads ~16 row/column blocks of the ring's frames instead of ~75 column
  // blocks, so the operands stay in L2 even when a ring's frames do not fit
  // (C4: 172 MB per ring); the order does not change any result.
  std::vector<TileDesc> tiles2;
  const int64_t nbi2 = (s->t + 255) / 256;
  constexpr int64_t SUPER = 8;  // C4 ncu: DRAM reads 425 GB (row-major) -> 294 GB
  for (int32_t r = 0; r < s->L->rings; ++r)
    for (int64_t SI = 0; SI < nbi2; SI += SUPER)
      for (int64_t SJ = SI; SJ < nbj; SJ += SUPER)
        for (int64_t I = SI; I < std::min(nbi2, SI + SUPER); ++I)
          for (int64_t J = std::max(I, SJ); J < std::min(nbj, SJ + SUPER); ++J) {
            TileDesc d;
            d.ring = r;
            d.i0 = static_cast<int32_t>(I * 256);
            d.j0 = static_cast<int32_t>(J * 256);
            d.pad = static_cast<int32_t>((int64_t)r * s->tiles_per_ring + iboff[2 * I] + (J - I));
            tiles2.push_back(d);
          }
  dfree(s->d_tiles2);
  XG_CUDA(c, dalloc(&s->d_tiles2, tiles2.size()));
  XG_CUDA(c, cudaMemcpy(s->d_tiles2, tiles2.data(), tiles2.size() * sizeof(TileDesc),
                        cudaMemcpyHostToDevice));
  s->ntiles2 = static_cast<int32_t>(tiles2.size());
  // the same tiles grouped by column block J: a tile needs frames < 256 (J+1)
  // only, so the host-overlapped path runs group J as soon as those arrive
  s->tiles2_joff.assign(static_cast<size_t>(nbj + 1), 0);
  for (const TileDesc& d : tiles2) s->tiles2_joff[d.j0 / 256 + 1]++;
  for (int64_t J = 0; J < nbj; ++J) s->tiles2_joff[J + 1] += s->tiles2_joff[J];
  std::vector<TileDesc> byj(tiles2.size());
  {
    std::vector<int32_t> fill(s->tiles2_joff.begin(), s->tiles2_joff.end() - 1);
    for (const TileDesc& d : tiles2) byj[fill[d.j0 / 256]++] = d;  // stable within J
  }
  dfree(s->d_tiles2_j);
  XG_CUDA(c, dalloc(&s->d_tiles2_j, byj.size()));
  XG_CUDA(c, cudaMemcpy(s->d_tiles2_j, byj.data(), byj.size() * sizeof(TileDesc),
                        cudaMemcpyHostToDevice));
  s->tiles_for_t = s->t;
  return XG_OK;
}

// K2/K4 launch: the CTA-pair kernel over the pair tiles (or a J-group of them).
static cudaError_t launch_gram_any(xg_series* s, int mode, const CUtensorMap& in,
                                   const CUtensorMap& out, GramParams gp,
                                   const TileDesc* tiles2 = nullptr, int32_t ntiles2 = -1) {
  gp.g2_nbi = static_cast<int32_t>((s->t + 127) / 128);
  gp.g2_nbj = static_cast<int32_t>((s->t + 255) / 256);
  gp.tiles = tiles2 ? tiles2 : s->d_tiles2;
  gp.ntiles = ntiles2 >= 0 ? ntiles2 : s->ntiles2;
  if (gp.ntiles == 0) return cudaSuccess;
  if (gp.wave_ctr) {
    // the wave gate pays where a ring's frames overflow L2 (C4: 172 MB per
    // ring, 109.6 -> 105.5 ms); where they fit (C2: 33 MB) it only costs
    const double ring_bytes = (double)s->t * (double)s->L->ktot / std::max(1, s->L->rings);
    if (ring_bytes <= 64e6) {
      gp.wave_ctr = nullptr;
    } else {
      gp.gate_lag = 2;  // C4 (ring-blocked): 86.1 ms ungated, 82.4 ms at lag 2
      const cudaError_t e = cudaMemsetAsync(gp.wave_ctr, 0, sizeof(unsigned int), s->ctx->stream);
      if (e != cudaSuccess) return e;
    }
  }
  return mode == 0 ? launch_gram2_u8(in, out, gp, s->ctx->num_sms, s->ctx->stream)
                   : launch_gram2_cmp(in, out, gp, s->ctx->num_sms, s->ctx->stream);
}

static int run_g2(xg_series* s, int mode, int32_t ring0 = 0, int32_t n_rings = -1) {
  xg_ctx* c = s->ctx;
  if (n_rings < 0) n_rings = s->L->rings - ring0;
  // <= 8 segments of >= 1024 frames: bounded partial storage, long serial chains split
  const int32_t seg = static_cast<int32_t>(std::max<int64_t>(1024, (s->t + 7) / 8));
  const int32_t nseg = static_cast<int32_t>((s->t + seg - 1) / seg);
  // partials: [ring][nseg][t] <= Q * tp entries since nseg * t <= tp * ceil(t/seg)...
  // allocated at creation as Q * tp; grow once if a long series needs more.
  const size_t need = (size_t)s->L->rings * nseg * s->t;
  if (need > s->g2part_cap) {
    dfree(s->d_g2part);
    dfree(s->d_g2pcnt);
    XG_CUDA(c, dalloc(&s->d_g2part, need));
    XG_CUDA(c, dalloc(&s->d_g2pcnt, need));
    s->g2part_cap = need;
  }
  G2Params g;
  g.gram = s->d_gram + (int64_t)ring0 * slab_elems(s);
  g.cf32 = nullptr;
  g.ring_stride = slab_elems(s);
  g.ld = static_cast<int32_t>(s->tp);
  g.nb = ttc_nb(s);
  g.inv = s->d_inv + (int64_t)ring0 * s->tp;
  g.inv_ld = s->tp;
  g.n_frames = s->t;
  g.n_rings = n_rings;
  g.seg = seg;
  g.n_seg = nseg;
  g.partial = s->d_g2part;
  g.pcount = s->d_g2pcnt;
  g.g2 = s->d_g2 + (int64_t)ring0 * s->tp;
  g.counts = s->d_g2cnt + (int64_t)ring0 * s->tp;
  g.g2_ld = s->tp;
  XG_CUDA(c, launch_g2(g, mode, c->stream));
  c->launches += 2;
  return XG_OK;
}

// Fold the per-tile diagonal sums left by a K2/K4 launch into g2 (fixed order).
static int fold_g2(xg_series* s, double* g2, int64_t* cnt, bool single = false) {
  xg_ctx* c = s->ctx;
  G2FoldParams f;
  f.g2_partial = s->d_g2tile;
  f.single = single ? 1 : 0;
  f.runs = s->d_g2runs;
  f.tiles_per_ring = s->tiles_per_ring;
  f.nbi = static_cast<int32_t>((s->t + 127) / 128);
  f.nbj = static_cast<int32_t>((s->t + 255) / 256);
  f.n_frames = s->t;
  f.n_rings = s->L->rings;
  f.nz_bits = s->d_nz_bits;
  f.nz_words = s->nz_words;
  f.zero_count = s->d_zero;
  f.g2 = g2;
  f.counts = cnt;
  f.g2_ld = s->tp;
  XG_CUDA(c, launch_g2_fold(f, c->stream));
  c->launches++;
  return XG_OK;
}

// K2 launch parameters and tensor maps of a raw pass over the series.
static int raw_gram_setup(xg_series* s, bool g2, bool store, GramParams& gp, CUtensorMap& map,
                          CUtensorMap& omap) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (store && !s->d_gram)  // the packed int32 TTC (upper pair tiles), allocated on first use
    XG_CUDA(c, dalloc(&s->d_gram, (size_t)L->rings * slab_elems(s)));
  int rc = build_tiles(s);
  if (rc) return rc;
  rc = ensure_xmaps(s, s->t);
  if (rc) return rc;
  // the kernel's parameter map is unused in raw mode (per-ring maps above)
  rc = make_map_u8(c, &map, s->d_x, L->kpad[0], s->t, L->kpad[0], 128, 128);
  if (rc) return rc;
  gp.xmaps = s->d_xmaps;
  gp.tiles = s->d_tiles;
  gp.ntiles = s->ntiles;
  gp.ring_koff = L->d_ring_koff;
  gp.ring_nkb = L->d_ring_nkb;
  gp.gram = reinterpret_cast<uint32_t*>(s->d_gram);
  gp.ring_stride = slab_elems(s);
  gp.ld = static_cast<int32_t>(s->tp);
  gp.nb = ttc_nb(s);
  gp.err = c->d_err;
  gp.max_norm2 = reinterpret_cast<const unsigned long long*>(s->d_max_norm2);
  gp.inv = s->d_inv;
  gp.inv2 = s->d_inv2;
  gp.inv_ld = s->tp;
  gp.n_frames = s->t;
  gp.g2_partial = g2 ? s->d_g2tile : nullptr;
  gp.store = store ? 1 : 0;
  if (!s->d_wave) XG_CUDA(c, dalloc(&s->d_wave, 1));
  gp.wave_ctr = s->d_wave;
  s->raw_stored = store;
  if (!store)  // a valid (never written) map over the frames buffer
    return make_map_out32(c, &omap, s->d_x, 32, 32);
  return make_map_out32(c, &omap, s->d_gram, 256, (int64_t)L->rings * slab_elems(s) / 256);
}

int xg_ttc_raw(xg_series* s, uint32_t flags) {
  if (!s) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (s->t < 2) return fail(c, XG_ERR_CONTRACT, "ttc_raw: need at least 2 frames");
  if (s->x_row0 != 0 || s->t > s->xmax)
    return fail(c, XG_ERR_CONTRACT, "ttc_raw: the raw TTC needs every frame resident "
                                    "(series loaded in chunks; use the compressed path)");
  const xg_layout* L = s->L;
  if (flags & XG_STRICT) {
    // reference semantics: first zero-norm frame raises (linalg.cpp:446-449)
    std::vector<int64_t> fz(L->rings);
    XG_CUDA(c, cudaMemcpyAsync(fz.data(), s->d_first_zero, fz.size() * 8,
                               cudaMemcpyDeviceToHost, c->stream));
    XG_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int32_t r = 0; r < L->rings; ++r)
      if (fz[r] != kNoZero) {
        c->payload = fz[r];
        c->payload_ring = r;
        return fail(c, XG_ERR_NORMALIZATION, "row_normalize: frame %lld of ring %d has zero norm",
                    (long long)fz[r], r);
      }
  }
  const bool g2 = !(flags & XG_NO_G2);
  GramParams gp;
  CUtensorMap map, omap;
  int rc = raw_gram_setup(s, g2, !(flags & XG_NO_STORE), gp, map, omap);
  if (rc) return rc;
  XG_CUDA(c, launch_gram_any(s, 0, map, omap, gp));
  c->launches++;
  if (g2) {
    rc = fold_g2(s, s->d_g2, s->d_g2cnt);
    if (rc) return rc;
  }
  s->have_raw = true;
  s->raw_g2 = g2;
  return XG_OK;
}

// load_frames + ttc_raw for frames in HOST memory (pinned for full overlap):
// the frames cross PCIe in chunks on a copy stream while the compute stream
// ingests each arrived chunk and runs the pair tiles whose columns it
// completes (a tile of column block J needs frames < 256 (J+1) only), so
// K1 and K2 hide behind the transfer.  Same results as the two calls.
int xg_series_ttc_raw_host(xg_series* s, const uint8_t* frames, int64_t n, uint32_t flags) {
  if (!s || !frames) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (n < 1 || n > s->xmax)
    return fail(c, XG_ERR_SHAPE, "load_frames: %lld frames, capacity %lld", (long long)n,
                (long long)s->xmax);
  if (n < 2) return fail(c, XG_ERR_CONTRACT, "ttc_raw: need at least 2 frames");
  s->x_row0 = 0;
  if (flags & XG_STRICT) {  // strict needs every frame before the Gram
    int rc = xg_series_load_frames(s, frames, n, 0);
    return rc ? rc : xg_ttc_raw(s, flags);
  }
  if (!c->copy_stream) XG_CUDA(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (int rc0 = ensure_raster(s)) return rc0;
  // ~8 chunks of whole 256-frame column blocks
  const int64_t nbj = (n + 255) / 256;
  const int64_t jb_per = std::max<int64_t>(1, (nbj + 7) / 8);
  const int64_t nchunks = (nbj + jb_per - 1) / jb_per;
  while ((int64_t)c->events.size() < nchunks + 1) {
    cudaEvent_t ev;
    XG_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->events.push_back(ev);
  }
  int rc = reset_stats(s, n);
  if (rc) return rc;
  s->t = n;
  invalidate_results(s);
  const bool g2 = !(flags & XG_NO_G2);
  GramParams gp;
  CUtensorMap map, omap;
  rc = raw_gram_setup(s, g2, !(flags & XG_NO_STORE), gp, map, omap);
  if (rc) return rc;
  // the staging raster may still be read by earlier work on the compute stream
  XG_CUDA(c, cudaEventRecord(c->events[nchunks], c->stream));
  XG_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->events[nchunks], 0));
  for (int64_t k = 0; k < nchunks; ++k) {
    const int64_t jb0 = k * jb_per, jb1 = std::min(nbj, jb0 + jb_per);
    const int64_t t0 = jb0 * 256, t1 = std::min(n, jb1 * 256);
    XG_CUDA(c, cudaMemcpyAsync(s->d_raster + t0 * L->pixels, frames + t0 * L->pixels,
                               (size_t)(t1 - t0) * L->pixels, cudaMemcpyHostToDevice,
                               c->copy_stream));
    XG_CUDA(c, cudaEventRecord(c->events[k], c->copy_stream));
    XG_CUDA(c, cudaStreamWaitEvent(c->stream, c->events[k], 0));
    rc = ingest_range(s, s->d_raster + t0 * L->pixels, t0, t1 - t0);
    if (rc) return rc;
    const int32_t o0 = s->tiles2_joff[jb0], o1 = s->tiles2_joff[jb1];
    XG_CUDA(c, launch_gram_any(s, 0, map, omap, gp, s->d_tiles2_j + o0, o1 - o0));
    c->launches++;
  }
  if (g2) {
    rc = fold_g2(s, s->d_g2, s->d_g2cnt);
    if (rc) return rc;
  }
  s->have_raw = true;
  s->raw_g2 = g2;
  return XG_OK;
}

int xg_series_ttc_raw_events_host(xg_series* s, const int64_t* frame_off, const int32_t* pix,
                                  const uint8_t* val, int64_t n, uint32_t flags) {
  if (!s || !frame_off) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (n < 2) return fail(c, XG_ERR_CONTRACT, "ttc_raw: need at least 2 frames");
  if (flags & XG_STRICT) {  // strict needs every frame before the Gram
    int rc = xg_series_load_events(s, frame_off, pix, val, n, 0);
    return rc ? rc : xg_ttc_raw(s, flags);
  }
  int rc = events_prepare(s, n);
  if (rc) return rc;
  rc = events_stage(s, frame_off, pix, val, n);
  if (rc) return rc;
  if (!c->copy_stream) XG_CUDA(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  const int64_t nbj = (n + 255) / 256;
  const int64_t jb_per = std::max<int64_t>(1, (nbj + 7) / 8);
  const int64_t nchunks = (nbj + jb_per - 1) / jb_per;
  while ((int64_t)c->events.size() < nchunks + 1) {
    cudaEvent_t ev;
    XG_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->events.push_back(ev);
  }
  s->x_row0 = 0;
  rc = reset_stats(s, n);
  if (rc) return rc;
  s->t = n;
  invalidate_results(s);
  rc = events_clear(s, n);
  if (rc) return rc;
  const bool g2 = !(flags & XG_NO_G2);
  GramParams gp;
  CUtensorMap map, omap;
  rc = raw_gram_setup(s, g2, !(flags & XG_NO_STORE), gp, map, omap);
  if (rc) return rc;
  // the staging lists may still be read by earlier work on the compute stream
  XG_CUDA(c, cudaEventRecord(c->events[nchunks], c->stream));
  XG_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->events[nchunks], 0));
  XG_CUDA(c, cudaMemcpyAsync(s->d_evoff, frame_off, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice,
                             c->copy_stream));
  for (int64_t k = 0; k < nchunks; ++k) {
    const int64_t jb0 = k * jb_per, jb1 = std::min(nbj, jb0 + jb_per);
    const int64_t t0 = jb0 * 256, t1 = std::min(n, jb1 * 256);
    const int64_t e0 = frame_off[t0], e1 = frame_off[t1];
    if (e1 > e0) {
      XG_CUDA(c, cudaMemcpyAsync(s->d_evpix + e0, pix + e0, (size_t)(e1 - e0) * 4,
                                 cudaMemcpyHostToDevice, c->copy_stream));
      XG_CUDA(c, cudaMemcpyAsync(s->d_evval + e0, val + e0, (size_t)(e1 - e0),
                                 cudaMemcpyHostToDevice, c->copy_stream));
    }
    XG_CUDA(c, cudaEventRecord(c->events[k], c->copy_stream));
    XG_CUDA(c, cudaStreamWaitEvent(c->stream, c->events[k], 0));
    rc = events_ingest(s, s->d_evoff, s->d_evpix, s->d_evval, t0, t1 - t0);
    if (rc) return rc;
    const int32_t o0 = s->tiles2_joff[jb0], o1 = s->tiles2_joff[jb1];
    XG_CUDA(c, launch_gram_any(s, 0, map, omap, gp, s->d_tiles2_j + o0, o1 - o0));
    c->launches++;
  }
  if (g2) {
    rc = fold_g2(s, s->d_g2, s->d_g2cnt);
    if (rc) return rc;
  }
  s->have_raw = true;
  s->raw_g2 = g2;
  return XG_OK;
}

int xg_series_g2(xg_series* s) {
  if (!s) return XG_ERR_INVALID;
  if (!s->have_raw) return fail(s->ctx, XG_ERR_CONTRACT, "g2: no TTC computed yet");
  if (!s->raw_stored) return fail(s->ctx, XG_ERR_CONTRACT, "g2: TTC computed with XG_NO_STORE");
  const int rc = run_g2(s, 0);
  if (!rc) s->raw_g2 = true;
  return rc;
}

// ------------------------------------------------ split rings
// A ring whose pixels are spread over several processes: each holds the
// exact int32 Gram and |x_t|^2 of its share (both sums over pixels,
// linalg.cpp:127-156), exported as the packed upper pair tiles + a norm^2
// column, summed by the caller (integer sum: exact and order-free), and the
// total imported back into one process's series, which then refreshes the
// ring's norms, zero-frame bookkeeping and g2 (standalone pass over the
// stored Gram: the fused epilogue saw only the partial).
int64_t xg_series_partial_elems(const xg_series* s) {
  if (!s || s->t < 1) return -1;
  const int64_t nb = (s->t + 255) / 256;
  return nb * (nb + 1) / 2 * 65536;
}

static int partial_check(xg_series* s, int32_t ring, const char* what) {
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->have_raw || !s->raw_stored)
    return fail(c, XG_ERR_CONTRACT, "%s: needs a stored raw TTC (ttc_raw without XG_NO_STORE)",
                what);
  return XG_OK;
}

int xg_series_export_partial(xg_series* s, int32_t ring, int32_t* gram, int64_t* norm2,
                             int on_device) {
  if (!s || !gram || !norm2) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  int rc = partial_check(s, ring, "export_partial");
  if (rc) return rc;
  // the stored slab already is the exchange format (packed upper pair tiles)
  const int64_t elems = xg_series_partial_elems(s);
  const cudaMemcpyKind dir = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  cudaError_t e = cudaMemcpyAsync(gram, s->d_gram + (int64_t)ring * slab_elems(s),
                                  (size_t)elems * 4, dir, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(norm2, 8, s->d_norm2 + ring, (size_t)s->L->rings * 8, 8, s->t, dir,
                          c->stream);
  if (e == cudaSuccess && !on_device) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "export_partial");
  return on_device ? XG_OK : check_device_error(c);
}

int xg_series_import_partial(xg_series* s, int32_t ring, const int32_t* gram, const int64_t* norm2,
                             int on_device, uint32_t flags) {
  if (!s || !gram || !norm2) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  int rc = partial_check(s, ring, "import_partial");
  if (rc) return rc;
  const int64_t elems = xg_series_partial_elems(s);
  cudaError_t e = cudaMemcpyAsync(s->d_gram + (int64_t)ring * slab_elems(s), gram,
                                  (size_t)elems * 4,
                                  on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                  c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(s->d_norm2 + ring, (size_t)L->rings * 8, norm2, 8, 8, s->t,
                          on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream);
  // the ring's frame statistics are rebuilt from the summed |x|^2
  if (e == cudaSuccess) e = cudaMemsetAsync(s->d_zero + ring, 0, 8, c->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->d_first_zero + ring, 0x7F, 8, c->stream);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(s->d_nz_bits + (int64_t)ring * s->nz_words, 0, (size_t)s->nz_words * 4,
                        c->stream);
  if (e == cudaSuccess) {
    NormParams np;
    np.t0 = 0;
    np.norm2 = s->d_norm2;
    np.n_frames = s->t;
    np.ld = s->tp;
    np.n_rings = L->rings;
    np.norms = s->d_norms;
    np.inv = s->d_inv;
    np.inv2 = s->d_inv2;
    np.zero_count = s->d_zero;
    np.first_zero = s->d_first_zero;
    np.nz_bits = s->d_nz_bits;
    np.nz_words = s->nz_words;
    np.max_norm2 = reinterpret_cast<unsigned long long*>(s->d_max_norm2);
    np.err = c->d_err;  // the summed ring forms a raw Gram: |x|^2 < 2^31 required
    np.ring0 = ring;
    np.ring_count = 1;
    e = launch_norms(np, c->stream);
  }
  if (!on_device && e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "import_partial");
  c->launches++;
  if (flags & XG_STRICT) {
    int64_t fz = 0;
    XG_CUDA(c, cudaMemcpyAsync(&fz, s->d_first_zero + ring, 8, cudaMemcpyDeviceToHost, c->stream));
    XG_CUDA(c, cudaStreamSynchronize(c->stream));
    if (fz != kNoZero) {
      c->payload = fz;
      c->payload_ring = ring;
      return fail(c, XG_ERR_NORMALIZATION, "row_normalize: frame %lld of ring %d has zero norm",
                  (long long)fz, ring);
    }
  }
  if (!(flags & XG_NO_G2)) {
    rc = run_g2(s, 0, ring, 1);
    if (rc) return rc;
  }
  return XG_OK;
}

// Deviation report of the homomorphic path (north star; ttc_rel_error,
// correlate.cpp:87-108): per ring ||C - C~||_F / ||C||_F from the stored TTCs.
int xg_series_rel_error(xg_series* s, double* out) {
  if (!s || !out) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (!s->have_raw || !s->raw_stored)
    return fail(c, XG_ERR_CONTRACT, "rel_error: needs a stored raw TTC (ttc_raw)");
  if (!s->have_cttc || !s->cmp_stored)
    return fail(c, XG_ERR_CONTRACT, "rel_error: needs a stored compressed TTC");
  double2* part = nullptr;
  double* d_out = nullptr;
  XG_CUDA(c, cudaMalloc(&part, (size_t)L->rings * REL_BLOCKS * sizeof(double2)));
  if (cudaError_t e0 = cudaMalloc(&d_out, (size_t)L->rings * 8); e0 != cudaSuccess) {
    cudaFree(part);
    return cuda_fail(c, e0, "rel_error");
  }
  RelErrParams p;
  p.gram = s->d_gram;
  p.cgram = s->d_cgram;
  p.ring_stride = slab_elems(s);
  p.ld = static_cast<int32_t>(s->tp);
  p.nb = ttc_nb(s);
  p.inv = s->d_inv;
  p.inv_ld = s->tp;
  p.n = s->t;
  p.n_rings = L->rings;
  p.partial = part;
  p.out = d_out;
  cudaError_t e = launch_rel_error(p, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, d_out, (size_t)L->rings * 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(part);
  cudaFree(d_out);
  if (e != cudaSuccess) return cuda_fail(c, e, "rel_error");
  c->launches += 2;
  for (int32_t r = 0; r < L->rings; ++r)
    if (out[r] < 0.0) return fail(c, XG_ERR_CONTRACT, "ttc_rel_error: reference TTC is all zero");
  return check_device_error(c);
}

int xg_series_get_ttc(xg_series* s, int32_t ring, int32_t dtype, void* out, int64_t ld,
                      int out_on_device) {
  if (!s || !out) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->have_raw) return fail(c, XG_ERR_CONTRACT, "get_ttc: no TTC computed yet");
  if (!s->raw_stored) return fail(c, XG_ERR_CONTRACT, "get_ttc: computed with XG_NO_STORE");
  if (dtype < 0 || dtype > 2) return fail(c, XG_ERR_CONTRACT, "get_ttc: bad dtype");
  if (ld < s->t) return fail(c, XG_ERR_SHAPE, "get_ttc: ld < n");
  const size_t esz = dtype == 0 ? 8 : 4;
  const size_t bytes = (size_t)s->t * ld * esz;
  void* dst = out;
  void* tmp = nullptr;
  if (!out_on_device) {
    XG_CUDA(c, ctx_scratch(c, bytes, &tmp));
    dst = tmp;
  }
  ExpandParams p;
  p.gram = s->d_gram + (int64_t)ring * slab_elems(s);
  p.cf32 = nullptr;
  p.ring_stride = 0;
  p.ld = static_cast<int32_t>(s->tp);
  p.nb = ttc_nb(s);
  p.inv = s->d_inv + (int64_t)ring * s->tp;
  p.n = s->t;
  p.out = dst;
  p.out_ld = ld;
  p.out_dtype = dtype;
  cudaError_t e = launch_expand(p, 0, c->stream);
  c->launches++;
  if (e == cudaSuccess && tmp) {
    e = cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "get_ttc");
  return check_device_error(c);
}

int xg_series_get_g2(xg_series* s, int32_t ring, double* values, int64_t* counts) {
  if (!s || !values) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->have_raw) return fail(c, XG_ERR_CONTRACT, "get_g2: no TTC computed yet");
  XG_CUDA(c, cudaMemcpyAsync(values, s->d_g2 + (int64_t)ring * s->tp, (size_t)s->t * 8,
                             cudaMemcpyDeviceToHost, c->stream));
  if (counts)
    XG_CUDA(c, cudaMemcpyAsync(counts, s->d_g2cnt + (int64_t)ring * s->tp, (size_t)s->t * 8,
                               cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

// Device pointers of the g2 curves (borrowed; valid until the series is
// recomputed or destroyed): collectives gather them without a host trip.
int xg_series_g2_device(xg_series* s, int32_t which, const double** values,
                        const int64_t** counts, int64_t* ld) {
  if (!s || !values || !counts || !ld) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (which == 0 ? !(s->have_raw && s->raw_g2) : !(s->have_cttc && s->cmp_g2))
    return fail(c, XG_ERR_CONTRACT, "g2_device: no current %s g2", which == 0 ? "raw" : "compressed");
  *values = which == 0 ? s->d_g2 : s->d_cg2;
  *counts = which == 0 ? s->d_g2cnt : s->d_cg2cnt;
  *ld = s->tp;
  return XG_OK;
}

// g2 of every ring in one transfer: values[r * n + d], counts likewise.
int xg_series_get_g2_all(xg_series* s, double* values, int64_t* counts) {
  if (!s || !values) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (!s->have_raw) return fail(c, XG_ERR_CONTRACT, "get_g2: no TTC computed yet");
  const int64_t n = s->t;
  XG_CUDA(c, cudaMemcpy2DAsync(values, (size_t)n * 8, s->d_g2, (size_t)s->tp * 8, (size_t)n * 8,
                               s->L->rings, cudaMemcpyDeviceToHost, c->stream));
  if (counts)
    XG_CUDA(c, cudaMemcpy2DAsync(counts, (size_t)n * 8, s->d_g2cnt, (size_t)s->tp * 8,
                                 (size_t)n * 8, s->L->rings, cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

int xg_synth_speckle(xg_ctx* c, int64_t n_frames, int64_t height, int64_t width,
                     int32_t n_rings, double mu, int32_t gamma_mode, double gamma_a,
                     uint64_t seed, uint8_t* out_device) {
  if (!c || !out_device) return XG_ERR_INVALID;
  if (n_frames < 1 || height < 1 || width < 1 || n_rings < 1 || !(mu >= 0.0))
    return fail(c, XG_ERR_CONTRACT, "synth_speckle: bad arguments");
  auto mix = [](uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
  };
  const uint64_t kStream = 0xD6E8FEB86659FD93ULL;  // CounterRng::substream (rng.cpp:20-22)
  SynthParams p;
  p.t_first = 0;
  p.t_frames = n_frames;
  p.h = height;
  p.w = width;
  p.q = n_rings;
  p.gamma_mode = gamma_mode;
  p.gamma_a = gamma_a;
  p.mu = mu;
  p.s_re = mix(seed ^ (1 * kStream));
  p.s_im = mix(seed ^ (2 * kStream));
  p.s_po = mix(seed ^ (3 * kStream));
  p.carry_re = nullptr;
  p.carry_im = nullptr;
  p.out = out_device;
  p.out_ld = height * width;
  XG_CUDA(c, launch_synth(p, c->stream));
  c->launches++;
  return XG_OK;
}

int xg_series_get_norms(xg_series* s, int32_t ring, double* norms, int64_t* n_zero) {
  if (!s) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (norms)
    XG_CUDA(c, cudaMemcpyAsync(norms, s->d_norms + (int64_t)ring * s->tp, (size_t)s->t * 8,
                               cudaMemcpyDeviceToHost, c->stream));
  if (n_zero)
    XG_CUDA(c, cudaMemcpyAsync(n_zero, s->d_zero + ring, 8, cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

// ------------------------------------------------------------- compressed
int xg_basis_create(xg_ctx* c, const xg_layout* L, int32_t k, int32_t digits, xg_basis** out) {
  if (!c || !L || !out) return XG_ERR_INVALID;
  *out = nullptr;
  if (k < 1) return fail(c, XG_ERR_CONTRACT, "basis: k must be >= 1");
  if (digits < 1 || digits > 3) return fail(c, XG_ERR_CONTRACT, "basis: digits must be 1..3");
  xg_basis* B = new xg_basis();
  B->ctx = c;
  B->L = L;
  B->k = k;
  B->digits = digits;
  // coefficients per N-tile: multiple of 16 with digits*kt <= 256
  const int32_t kmax = (256 / digits) / 16 * 16;
  const int32_t k16 = static_cast<int32_t>(round_up(k, 16));
  B->ntiles_n = (k16 + kmax - 1) / kmax;
  B->kt = static_cast<int32_t>(round_up((k16 + B->ntiles_n - 1) / B->ntiles_n, 16));
  B->vrows = static_cast<int64_t>(B->ntiles_n) * digits * B->kt;
  B->h_vd.assign(static_cast<size_t>(B->vrows * L->ktot), 0);
  B->h_scale.assign(static_cast<size_t>(L->rings) * k, 0.0);
  B->ring_set.assign(L->rings, 0);
  cudaError_t e;
  if ((e = dalloc(&B->d_vd, B->h_vd.size())) != cudaSuccess ||
      (e = dalloc(&B->d_scale, B->h_scale.size())) != cudaSuccess) {
    xg_basis_destroy(B);
    return cuda_fail(c, e, "basis alloc");
  }
  *out = B;
  return XG_OK;
}

void xg_basis_destroy(xg_basis* B) {
  if (!B) return;
  dfree(B->d_vd);
  dfree(B->d_scale);
  dfree(B->d_vmaps);
  delete B;
}

// V (M_q x k, mask order, f64) -> per-column scale and S int8 digits:
// V ~= scale * (d0 + d1/254 + d2/254^2), written at the ring-major columns.
int xg_basis_set_ring(xg_basis* B, int32_t ring, const double* v) {
  if (!B || !v) return XG_ERR_INVALID;
  xg_ctx* c = B->ctx;
  const xg_layout* L = B->L;
  if (ring < 0 || ring >= L->rings) return fail(c, XG_ERR_SHAPE, "basis: ring %d out of range", ring);
  const int64_t m = L->ring_pixels[ring], k = B->k;
  const int64_t* col = L->colpos.data() + L->mask_off[ring];
  for (int64_t j = 0; j < k; ++j) {
    double amax = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double x = v[i * k + j];
      if (!std::isfinite(x)) return fail(c, XG_ERR_CONTRACT, "basis: non-finite entry");
      amax = std::max(amax, std::fabs(x));
    }
    const double scale = amax > 0.0 ? amax / 127.0 : 1.0;
    B->h_scale[(size_t)ring * k + j] = scale;
    const int64_t nt = j / B->kt, jj = j % B->kt;
    for (int64_t i = 0; i < m; ++i) {
      double u = v[i * k + j] / scale;
      for (int s = 0; s < B->digits; ++s) {
        double d = std::nearbyint(u);
        d = std::min(127.0, std::max(-127.0, d));
        const int64_t row = (nt * B->digits + s) * B->kt + jj;
        B->h_vd[(size_t)(ring_base(L, B->vrows, ring) + row * ring_ld(L, ring) +
                         (col[i] - L->koff[ring]))] = static_cast<int8_t>(d);
        u = (u - d) * 254.0;
      }
    }
  }
  B->ring_set[ring] = 1;
  B->dirty = true;
  return XG_OK;
}

// Zero-norm check of XG_STRICT (reference semantics, compress.cpp:48-81 via
// row_normalize): the first zero frame of any ring raises.
static int strict_zero_check(xg_series* s, const char* what) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  std::vector<int64_t> fz(L->rings);
  XG_CUDA(c, cudaMemcpyAsync(fz.data(), s->d_first_zero, fz.size() * 8, cudaMemcpyDeviceToHost,
                             c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  for (int32_t r = 0; r < L->rings; ++r)
    if (fz[r] != kNoZero) {
      c->payload = fz[r];
      c->payload_ring = r;
      return fail(c, XG_ERR_NORMALIZATION, "%s: frame %lld of ring %d has zero norm", what,
                  (long long)fz[r], r);
    }
  return XG_OK;
}

// Digits, scales and the per-ring digit maps of a basis to the device (once
// per change of the basis).
static int basis_upload(xg_basis* B) {
  if (!B->dirty) return XG_OK;
  xg_ctx* c = B->ctx;
  XG_CUDA(c, cudaMemcpy(B->d_vd, B->h_vd.data(), B->h_vd.size(), cudaMemcpyHostToDevice));
  XG_CUDA(c, cudaMemcpy(B->d_scale, B->h_scale.data(), B->h_scale.size() * 8,
                        cudaMemcpyHostToDevice));
  // one box = a CTA's half of the S*kt digit rows of an N-tile
  const int rc = upload_ring_maps(c, B->L, reinterpret_cast<const uint8_t*>(B->d_vd), B->vrows,
                                  B->vrows, static_cast<uint32_t>(B->digits * B->kt / 2),
                                  &B->d_vmaps);
  if (rc) return rc;
  B->dirty = false;
  return XG_OK;
}

// K3 over the n ring-major rows in x, which hold series frames [t0, t0 + n).
static int compress_rows(xg_series* s, xg_basis* B, int64_t t0, int64_t n) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (int rc0 = basis_upload(B)) return rc0;
  const int32_t kp = static_cast<int32_t>(round_up(B->k, 64));
  if (s->ck != B->k || !s->d_y) {
    dfree(s->d_y);
    dfree(s->d_planes);
    XG_CUDA(c, dalloc(&s->d_y, (size_t)L->rings * s->tp * B->k));
    XG_CUDA(c, dalloc(&s->d_planes, (size_t)L->rings * 3 * s->tp * kp));
    XG_CUDA(c, cudaMemsetAsync(s->d_planes, 0, (size_t)L->rings * 3 * s->tp * kp * 2, c->stream));
    s->ck = B->k;
    s->ckp = kp;
  }
  // tiles: (ring, frame block of x, N-tile), cached per (rows, N-tiles)
  const int64_t key = n * 64 + B->ntiles_n;
  if (s->ptiles_key != key) {
    std::vector<TileDesc> tiles;
    const int64_t nbi = (n + 255) / 256;  // 256-frame blocks: one CTA pair each
    for (int32_t r = 0; r < L->rings; ++r)
      for (int64_t ib = 0; ib < nbi; ++ib)
        for (int32_t nt = 0; nt < B->ntiles_n; ++nt)
          tiles.push_back({r, (int32_t)(ib * 256), nt, 0});
    // The persistent kernel deals tile t to pair t mod P.  A tile costs its
    // ring's K (ring widths span 150x at C5), and a ring has fewer tiles than
    // there are pairs, so the dealt sums drift apart: order the tiles by
    // cost (descending, stable) and deal them in a snake (pairs 0..P-1, then
    // P-1..0, ...), which keeps every pair's total within one tile's cost.
    const int64_t P = std::max(1, c->num_sms / 2);
    std::stable_sort(tiles.begin(), tiles.end(), [&](const TileDesc& a, const TileDesc& b) {
      return L->kpad[a.ring] > L->kpad[b.ring];
    });
    for (size_t r0 = 0; r0 < tiles.size(); r0 += 2 * P) {  // reverse every second round
      const size_t a = std::min(tiles.size(), r0 + P), b = std::min(tiles.size(), r0 + 2 * P);
      if (a < b && b - a == (size_t)P) std::reverse(tiles.begin() + a, tiles.begin() + b);
    }
    dfree(s->d_ptiles);
    XG_CUDA(c, dalloc(&s->d_ptiles, tiles.size()));
    XG_CUDA(c, cudaMemcpy(s->d_ptiles, tiles.data(), tiles.size() * sizeof(TileDesc),
                          cudaMemcpyHostToDevice));
    s->n_ptiles = static_cast<int32_t>(tiles.size());
    s->ptiles_key = key;
  }
  CUtensorMap mx, mv, mp;
  int rc = ensure_xmaps(s, n);
  if (!rc) rc = make_map_u8(c, &mx, s->d_x, L->kpad[0], n, L->kpad[0], 128, 128);  // unused
  // bf16 planes: 16 coefficients x 32 frames boxes, stored by the K3 epilogue
  if (!rc)
    rc = make_map_bf16_box(c, &mp, s->d_planes, kp, (int64_t)L->rings * 3 * s->tp, 16, 32,
                           CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!rc)  // unused (per-ring digit maps)
    rc = make_map_u8(c, &mv, B->d_vd, L->kpad[0], B->vrows, L->kpad[0], 128,
                     B->digits * B->kt / 2);
  if (rc) return rc;
  ProjParams p;
  p.tiles = s->d_ptiles;
  p.t0 = t0;
  p.ntiles = s->n_ptiles;
  p.ring_koff = L->d_ring_koff;
  p.ring_nkb = L->d_ring_nkb;
  p.xmaps = s->d_xmaps;
  p.vmaps = B->d_vmaps;
  p.n_digits = B->digits;
  p.kt = B->kt;
  p.k = B->k;
  p.inv = s->d_inv;
  p.inv_ld = s->tp;
  p.n_frames = n;
  p.scale = B->d_scale;
  p.y = s->d_y;
  p.y_ld = s->tp;
  p.planes = s->d_planes;
  p.plane_rows = s->tp;
  p.kp = kp;
  p.err = c->d_err;
  XG_CUDA(c, launch_project(mx, mv, mp, p, c->num_sms, c->stream));
  c->launches++;
  return XG_OK;
}

static int check_basis(xg_series* s, const xg_basis* B) {
  xg_ctx* c = s->ctx;
  if (B->L != s->L) return fail(c, XG_ERR_BINDING, "compress: basis built for another layout");
  for (int32_t r = 0; r < s->L->rings; ++r)
    if (!B->ring_set[r]) return fail(c, XG_ERR_CONTRACT, "compress: basis of ring %d not set", r);
  return XG_OK;
}

// ------------------------------------------------------------ K9 basis on the device
// build_online_from_frames / build_offline (encoder.cpp:13-60 -> gram_svd,
// linalg.cpp:279-439) for every ring of a series at once; see k_basis.cu.
}  // extern "C"
namespace {

struct DevBufs {  // frees every scratch buffer on any return path
  std::vector<void*> p;
  template <class T>
  cudaError_t get(T** out, size_t count) {
    cudaError_t e = dalloc(out, count);
    if (e == cudaSuccess) p.push_back(*out);
    return e;
  }
  ~DevBufs() {
    for (void* q : p) cudaFree(q);
  }
};

// Upper Cholesky G = R^T R of the leading m x m block (G upper, ld m) and the
// transposed inverse: mt[j][i] = (R^-1)[i][j] (lower triangular, ld m).
// Returns the first collapsed column or -1.
int64_t chol_inv_t(const double* g, int64_t m, std::vector<double>& r, std::vector<double>& mt) {
  r.assign(m * m, 0.0);
  for (int64_t j = 0; j < m; ++j) {
    double d = g[j * m + j];
    for (int64_t i = 0; i < j; ++i) d -= r[i * m + j] * r[i * m + j];
    if (!(d > 0.0)) return j;
    const double rjj = std::sqrt(d);
    r[j * m + j] = rjj;
    for (int64_t l = j + 1; l < m; ++l) {
      double v = g[j * m + l];
      for (int64_t i = 0; i < j; ++i) v -= r[i * m + j] * r[i * m + l];
      r[j * m + l] = v / rjj;
    }
  }
  // X = R^-1 (upper) by back substitution, column by column
  std::vector<double> x(m * m, 0.0);
  for (int64_t c = 0; c < m; ++c) {
    for (int64_t i = c; i >= 0; --i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int64_t l = i + 1; l <= c; ++l) v -= r[i * m + l] * x[l * m + c];
      x[i * m + c] = v / r[i * m + i];
    }
  }
  mt.assign(m * m, 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = i; j < m; ++j) mt[j * m + i] = x[i * m + j];
  return -1;
}

template <class F>
void for_rings(int32_t n, F f) {
  const int nt = std::max(1, std::min<int>(n, (int)std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; ++w)
    pool.emplace_back([&, w] {
      for (int32_t r = w; r < n; r += nt) f(r);
    });
  for (auto& t : pool) t.join();
}

// Per-ring inputs of the device basis builder: the training rows X_r (n x
// kpad_r on the device: ring-major u8 frames or f64 rows), the offset of each
// ring's columns in the shared W / Q buffers (ktot columns in all), the W
// column of every mask-order pixel, and 1/|x_t| per frame (host copy).
struct BasisJob {
  int32_t Q = 0;
  int64_t n = 0;
  BasisSParams sp{};  // S source; n, np, a, v are set by basis_run
  bool x_u8 = true;
  std::vector<const void*> x;
  std::vector<int64_t> ldx, kpad, koff, mq;
  std::vector<const int64_t*> col;
  int64_t ktot = 0;
  std::vector<double> inv;
  int64_t inv_ld = 0;
};

// The device Gram-trick SVD (K9) from S onwards, shared by the series
// builder (counts, S from the exact int32 Gram) and the f64-row builders.
int basis_run(xg_ctx* c, const BasisJob& J, int32_t k, double* const* v_out, double* sigma_out,
              int64_t sigma_ld, int64_t* rank_out, xg_basis* B) {
  const int32_t Q = J.Q;
  const int64_t n = J.n;
  cudaStream_t st = c->stream;
  const int np = static_cast<int>(n + (n & 1));
  const int64_t rs = (int64_t)np * np;
  static const bool timing = std::getenv("XG_BASIS_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[basis] %-10s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  DevBufs db;
  double *d_a[2], *d_v[2];
  JacState* d_state;
  for (int b = 0; b < 2; ++b) {
    XG_CUDA(c, db.get(&d_a[b], (size_t)Q * rs));
    XG_CUDA(c, db.get(&d_v[b], (size_t)Q * rs));
  }
  XG_CUDA(c, db.get(&d_state, (size_t)Q));
  BasisSParams sp = J.sp;
  sp.n = static_cast<int32_t>(n);
  sp.np = np;
  sp.a = d_a[0];
  sp.v = d_v[0];
  phase("gram");
  XG_CUDA(c, launch_basis_s(sp, Q, st));
  c->launches++;
  // ---- Jacobi sweeps (sym_eig, linalg.cpp:234-276)
  std::vector<JacState> hs(Q, JacState{1e-15, 1, 0});
  std::vector<int> final_buf(Q, 0);
  int64_t g = 0;
  XG_CUDA(c, cudaMemcpyAsync(d_state, hs.data(), Q * sizeof(JacState), cudaMemcpyHostToDevice, st));
  for (int sweep = 0; sweep < 100; ++sweep) {
    for (int step = 0; step < np - 1; ++step, ++g) {
      JacParams jp{d_a[g % 2], d_a[(g + 1) % 2], d_v[g % 2], d_v[(g + 1) % 2], d_state, np, step};
      XG_CUDA(c, launch_jacobi_step(jp, Q, st));
      c->launches++;
    }
    XG_CUDA(c, cudaMemcpyAsync(hs.data(), d_state, Q * sizeof(JacState), cudaMemcpyDeviceToHost, st));
    XG_CUDA(c, cudaStreamSynchronize(st));
    bool any = false;
    for (int32_t r = 0; r < Q; ++r) {
      if (!hs[r].active) continue;
      final_buf[r] = static_cast<int>(g % 2);
      if (!hs[r].rotated) {
        hs[r].active = 0;
        continue;
      }
      if (sweep >= 40 && sweep % 10 == 0) hs[r].tol *= 100.0;  // stall escape (linalg.cpp:255)
      hs[r].rotated = 0;
      any = true;
    }
    if (!any) break;
    XG_CUDA(c, cudaMemcpyAsync(d_state, hs.data(), Q * sizeof(JacState), cudaMemcpyHostToDevice, st));
  }
  if (timing) fprintf(stderr, "[basis] %lld Jacobi steps (np %d, %d rings)\n", (long long)g, np, Q);
  phase("jacobi");
  // ---- eigenvalues (index order) and the accumulated rotations
  std::vector<const double*> a_ptr(Q);
  for (int32_t r = 0; r < Q; ++r) a_ptr[r] = d_a[final_buf[r]] + r * rs;
  const double** d_aptr;
  double* d_eig;
  XG_CUDA(c, db.get(&d_aptr, (size_t)Q));
  XG_CUDA(c, db.get(&d_eig, (size_t)Q * np));
  XG_CUDA(c, cudaMemcpyAsync(d_aptr, a_ptr.data(), Q * sizeof(double*), cudaMemcpyHostToDevice, st));
  XG_CUDA(c, launch_jacobi_diag(d_aptr, d_eig, np, Q, st));
  c->launches++;
  std::vector<double> eig((size_t)Q * np), hv((size_t)Q * rs);
  XG_CUDA(c, cudaMemcpyAsync(eig.data(), d_eig, eig.size() * 8, cudaMemcpyDeviceToHost, st));
  for (int32_t r = 0; r < Q; ++r)
    XG_CUDA(c, cudaMemcpyAsync(hv.data() + r * rs, d_v[final_buf[r]] + r * rs, rs * 8,
                               cudaMemcpyDeviceToHost, st));
  XG_CUDA(c, cudaStreamSynchronize(st));
  // Bt[j][t] = inv_t U[t][order_j]: eigenvectors in descending eigenvalue
  // order (stable in the index, linalg.cpp:262-266), rows scaled by 1/|x_t|
  std::vector<double> bt((size_t)Q * n * n);
  for_rings(Q, [&](int32_t r) {
    std::vector<int64_t> ord(n);
    for (int64_t i = 0; i < n; ++i) ord[i] = i;
    const double* e = eig.data() + (size_t)r * np;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return e[a] > e[b]; });
    const double* v = hv.data() + r * rs;
    double* o = bt.data() + (size_t)r * n * n;
    for (int64_t j = 0; j < n; ++j) {
      const int sl = index_slot(static_cast<int>(ord[j]), 0, np);
      for (int64_t t = 0; t < n; ++t) o[j * n + t] = J.inv[r * J.inv_ld + t] * v[t * np + sl];
    }
  });
  phase("eig+Bt");
  double *d_bt, *d_w;
  XG_CUDA(c, db.get(&d_bt, bt.size()));
  XG_CUDA(c, db.get(&d_w, (size_t)n * J.ktot));
  XG_CUDA(c, cudaMemcpyAsync(d_bt, bt.data(), bt.size() * 8, cudaMemcpyHostToDevice, st));
  // ---- W_r = Bt_r X_r  (n x kpad_r), X = the ring-major u8 frames or f64 rows
  int64_t kpad_max = 0;
  std::vector<DGemmRing> gr(Q);
  for (int32_t r = 0; r < Q; ++r) {
    kpad_max = std::max(kpad_max, J.kpad[r]);
    gr[r] = DGemmRing{d_bt + (size_t)r * n * n, n, J.x[r], J.ldx[r],
                      d_w + n * J.koff[r], J.kpad[r], (int32_t)n, (int32_t)J.kpad[r], (int32_t)n};
  }
  DGemmRing* d_gr;
  XG_CUDA(c, db.get(&d_gr, (size_t)Q));
  XG_CUDA(c, cudaMemcpyAsync(d_gr, gr.data(), Q * sizeof(DGemmRing), cudaMemcpyHostToDevice, st));
  XG_CUDA(c, launch_dgemm_nn(d_gr, Q, (int)n, (int)kpad_max, J.x_u8, st));
  c->launches++;
  // ---- measured singular values |W_j| (linalg.cpp:312-320)
  double* d_nrm;
  XG_CUDA(c, db.get(&d_nrm, (size_t)Q * n));
  for (int32_t r = 0; r < Q; ++r) gr[r] = DGemmRing{d_w + n * J.koff[r], J.kpad[r], nullptr, 0,
                                                    nullptr, 0, (int32_t)n, (int32_t)J.kpad[r], 0};
  XG_CUDA(c, cudaMemcpyAsync(d_gr, gr.data(), Q * sizeof(DGemmRing), cudaMemcpyHostToDevice, st));
  XG_CUDA(c, launch_row_norm2(d_gr, Q, (int)n, d_nrm, n, st));
  c->launches++;
  std::vector<double> nrm((size_t)Q * n);
  XG_CUDA(c, cudaMemcpyAsync(nrm.data(), d_nrm, nrm.size() * 8, cudaMemcpyDeviceToHost, st));
  XG_CUDA(c, cudaStreamSynchronize(st));
  phase("W+norms");
  std::vector<std::vector<int32_t>> ord2(Q);
  std::vector<int64_t> rank(Q), kk(Q);
  for (int32_t r = 0; r < Q; ++r) {
    double* nr = nrm.data() + (size_t)r * n;
    for (int64_t j = 0; j < n; ++j) nr[j] = std::sqrt(nr[j]);
    auto& o = ord2[r];
    o.resize(n);
    for (int64_t j = 0; j < n; ++j) o[j] = static_cast<int32_t>(j);
    std::stable_sort(o.begin(), o.end(), [&](int32_t a, int32_t b) { return nr[a] > nr[b]; });
    const double smax = nr[o[0]];
    int64_t rr = 0;
    while (rr < n && nr[o[rr]] > 1e-12 * smax) ++rr;
    rank[r] = rank_out[r] = rr;
  }
  for (int32_t r = 0; r < Q; ++r) {
    if (rank[r] == 0) {
      c->payload = 0;
      c->payload_ring = r;
      return fail(c, XG_ERR_RANK, "gram_svd: matrix is numerically zero, no spectrum");
    }
    if (k > rank[r]) {
      c->payload = rank[r];
      c->payload_ring = r;
      return fail(c, XG_ERR_RANK, "requested k = %d exceeds the numerical rank %lld of the "
                  "training rows (ring %d)", k, (long long)rank[r], r);
    }
    // columns that can reach the first k after the final sort (near-ties)
    kk[r] = k == 0 ? rank[r] : std::min<int64_t>(rank[r], k + 8);
  }
  const int64_t kkmax = *std::max_element(kk.begin(), kk.end());
  // ---- Q0 = kept columns of W (norm order) / |W_j|, then 2 x (Gram, Cholesky, Q R^-1)
  std::vector<int32_t> hidx((size_t)Q * kkmax, 0);
  std::vector<double> hsc((size_t)Q * kkmax, 0.0);
  for (int32_t r = 0; r < Q; ++r)
    for (int64_t j = 0; j < kk[r]; ++j) {
      hidx[r * kkmax + j] = ord2[r][j];
      hsc[r * kkmax + j] = 1.0 / nrm[(size_t)r * n + ord2[r][j]];
    }
  int32_t* d_idx;
  double *d_sc, *d_q[2], *d_g, *d_part, *d_mt;
  const int max_chunks = static_cast<int>((kpad_max + SYRK_CHUNK - 1) / SYRK_CHUNK);
  const int64_t part_stride = (int64_t)max_chunks * kkmax * kkmax;
  XG_CUDA(c, db.get(&d_idx, hidx.size()));
  XG_CUDA(c, db.get(&d_sc, hsc.size()));
  XG_CUDA(c, db.get(&d_q[0], (size_t)kkmax * J.ktot));
  XG_CUDA(c, db.get(&d_q[1], (size_t)kkmax * J.ktot));
  XG_CUDA(c, db.get(&d_g, (size_t)Q * kkmax * kkmax));
  XG_CUDA(c, db.get(&d_part, (size_t)Q * part_stride));
  XG_CUDA(c, db.get(&d_mt, (size_t)Q * kkmax * kkmax));
  XG_CUDA(c, cudaMemcpyAsync(d_idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice, st));
  XG_CUDA(c, cudaMemcpyAsync(d_sc, hsc.data(), hsc.size() * 8, cudaMemcpyHostToDevice, st));
  for (int32_t r = 0; r < Q; ++r)
    gr[r] = DGemmRing{d_w + n * J.koff[r], J.kpad[r], nullptr, 0, d_q[0] + kkmax * J.koff[r],
                      J.kpad[r], (int32_t)kk[r], (int32_t)J.kpad[r], 0};
  XG_CUDA(c, cudaMemcpyAsync(d_gr, gr.data(), Q * sizeof(DGemmRing), cudaMemcpyHostToDevice, st));
  XG_CUDA(c, launch_gather_rows(d_gr, d_idx, d_sc, kkmax, Q, (int)kkmax, (int)kpad_max, st));
  c->launches++;
  // r_total = R2 R1 D^-1 (linalg.cpp:352-373), D = diag(1 / |W_j|)
  std::vector<std::vector<double>> rtot(Q);
  for (int32_t r = 0; r < Q; ++r) rtot[r].assign(kk[r] * kk[r], 0.0);
  for (int32_t r = 0; r < Q; ++r)
    for (int64_t j = 0; j < kk[r]; ++j) rtot[r][j * kk[r] + j] = 1.0;
  std::vector<double> hg((size_t)Q * kkmax * kkmax), hmt((size_t)Q * kkmax * kkmax, 0.0);
  for (int pass = 0; pass < 2; ++pass) {
    double* qin = d_q[pass];
    double* qout = d_q[pass ^ 1];
    for (int32_t r = 0; r < Q; ++r)
      gr[r] = DGemmRing{qin + kkmax * J.koff[r], J.kpad[r], nullptr, 0,
                        d_g + (size_t)r * kkmax * kkmax, kk[r], (int32_t)kk[r],
                        (int32_t)J.kpad[r], 0};
    XG_CUDA(c, cudaMemcpyAsync(d_gr, gr.data(), Q * sizeof(DGemmRing), cudaMemcpyHostToDevice, st));
    XG_CUDA(c, launch_dsyrk(d_gr, Q, (int)kkmax, max_chunks, d_part, part_stride, st));
    XG_CUDA(c, launch_dsyrk_sum(d_gr, Q, (int)kkmax, max_chunks, d_part, part_stride, st));
    c->launches += 2;
    XG_CUDA(c, cudaMemcpyAsync(hg.data(), d_g, hg.size() * 8, cudaMemcpyDeviceToHost, st));
    XG_CUDA(c, cudaStreamSynchronize(st));
    std::vector<int64_t> bad(Q, -1);
    for_rings(Q, [&](int32_t r) {
      const int64_t m = kk[r];
      std::vector<double> rf, mt;
      bad[r] = chol_inv_t(hg.data() + (size_t)r * kkmax * kkmax, m, rf, mt);
      if (bad[r] >= 0) return;
      std::copy(mt.begin(), mt.end(), hmt.begin() + (size_t)r * kkmax * kkmax);
      std::vector<double> nt(m * m, 0.0);  // rtot = rf * rtot
      for (int64_t i = 0; i < m; ++i)
        for (int64_t l = i; l < m; ++l) {
          double v = 0.0;
          for (int64_t j = i; j <= l; ++j) v += rf[i * m + j] * rtot[r][j * m + l];
          nt[i * m + l] = v;
        }
      rtot[r].swap(nt);
    });
    for (int32_t r = 0; r < Q; ++r)
      if (bad[r] >= 0) {
        c->payload = bad[r];
        c->payload_ring = r;
        return fail(c, XG_ERR_RANK, "gram_svd: column collapse during orthogonalization");
      }
    XG_CUDA(c, cudaMemcpyAsync(d_mt, hmt.data(), hmt.size() * 8, cudaMemcpyHostToDevice, st));
    for (int32_t r = 0; r < Q; ++r)
      gr[r] = DGemmRing{d_mt + (size_t)r * kkmax * kkmax, kk[r], qin + kkmax * J.koff[r],
                        J.kpad[r], qout + kkmax * J.koff[r], J.kpad[r], (int32_t)kk[r],
                        (int32_t)J.kpad[r], (int32_t)kk[r]};
    XG_CUDA(c, cudaMemcpyAsync(d_gr, gr.data(), Q * sizeof(DGemmRing), cudaMemcpyHostToDevice, st));
    XG_CUDA(c, launch_dgemm_nn(d_gr, Q, (int)kkmax, (int)kpad_max, false, st));
    c->launches++;
  }
  phase("cholqr2");
  // ---- orthonormal columns (d_q[0] after two passes) to the host
  std::vector<double> hq((size_t)kkmax * J.ktot);
  XG_CUDA(c, cudaMemcpyAsync(hq.data(), d_q[0], hq.size() * 8, cudaMemcpyDeviceToHost, st));
  XG_CUDA(c, cudaStreamSynchronize(st));
  std::vector<int> set_rc(Q, XG_OK);
  for_rings(Q, [&](int32_t r) {
    const int64_t m = kk[r], kout = k == 0 ? rank[r] : k, mq = J.mq[r];
    // sigma_j = |a_j|, a = u_kept r_total^T with orthonormal u: the row norms
    // of r_total times |W_j| (linalg.cpp:377-383); near-ties re-sorted (:387-391)
    std::vector<double> sig(m);
    for (int64_t j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int64_t l = j; l < m; ++l) {
        const double v = rtot[r][j * m + l] * nrm[(size_t)r * n + ord2[r][l]];
        acc += v * v;
      }
      sig[j] = std::sqrt(acc);
    }
    std::vector<int64_t> perm(m);
    for (int64_t j = 0; j < m; ++j) perm[j] = j;
    std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return sig[a] > sig[b]; });
    if (sigma_out) {
      double* so = sigma_out + (size_t)r * sigma_ld;
      for (int64_t j = 0; j < n; ++j) so[j] = 0.0;
      for (int64_t j = 0; j < m; ++j) so[j] = sig[perm[j]];
      for (int64_t j = m; j < rank[r]; ++j) so[j] = nrm[(size_t)r * n + ord2[r][j]];
    }
    std::vector<double> vloc;
    double* vo = v_out ? v_out[r] : nullptr;
    if (!vo) {
      if (!B) return;
      vloc.resize(mq * kout);
      vo = vloc.data();
    }
    const int64_t* col = J.col[r];
    const double* qb = hq.data() + kkmax * J.koff[r];
    for (int64_t j = 0; j < kout; ++j) {
      const double* qrow = qb + perm[j] * J.kpad[r];
      // sign: largest-magnitude entry positive, first in mask order (linalg.cpp:421-436)
      int64_t arg = 0;
      double best = -1.0;
      for (int64_t i = 0; i < mq; ++i) {
        const double mag = std::fabs(qrow[col[i] - J.koff[r]]);
        if (mag > best) {
          best = mag;
          arg = i;
        }
      }
      const double sg = qrow[col[arg] - J.koff[r]] < 0.0 ? -1.0 : 1.0;
      for (int64_t i = 0; i < mq; ++i) vo[i * kout + j] = sg * qrow[col[i] - J.koff[r]];
    }
    if (B) set_rc[r] = xg_basis_set_ring(B, r, vo);
  });
  phase("V out");
  for (int32_t r = 0; r < Q; ++r)
    if (set_rc[r]) return set_rc[r];
  return XG_OK;
}


}  // namespace
extern "C" {

int xg_series_build_basis(xg_series* s, int32_t k, double* const* v_out, double* sigma_out,
                          int64_t sigma_ld, int64_t* rank_out, xg_basis* B) {
  if (!s || !rank_out) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  const int32_t Q = L->rings;
  const int64_t n = s->t;
  if (k < 0) return fail(c, XG_ERR_CONTRACT, "build_online_from_frames: k must be >= 1");
  if (n < 2) return fail(c, XG_ERR_CONTRACT, "build_online_from_frames: need at least 2 frames");
  if (n > 2048) return fail(c, XG_ERR_CONTRACT, "build_basis: at most 2048 training frames");
  if (s->x_row0 != 0 || n > s->xmax)
    return fail(c, XG_ERR_CONTRACT, "build_basis: every training frame must be resident");
  if (B && (B->L != L || B->k != k || k == 0))
    return fail(c, XG_ERR_CONTRACT, "build_basis: basis of rank %d does not match k = %d",
                B ? B->k : 0, k);
  if (sigma_out && sigma_ld < n) return fail(c, XG_ERR_SHAPE, "build_basis: sigma_ld < frames");
  int rc = strict_zero_check(s, "row_normalize");  // encoder_from_rows -> row_normalize
  if (rc) return rc;
  if (!(s->have_raw && s->raw_stored)) {
    rc = xg_ttc_raw(s, 0);  // the exact Gram of the training frames (K2)
    if (rc) return rc;
  }
  BasisJob J;
  J.Q = Q;
  J.n = n;
  J.sp = BasisSParams{s->d_gram, static_cast<int32_t>(s->tp), s->d_inv, s->tp, 0, 0, nullptr,
                      nullptr, ttc_nb(s), slab_elems(s), nullptr};
  J.x_u8 = true;
  J.ktot = L->ktot;
  for (int32_t r = 0; r < Q; ++r) {
    J.x.push_back(s->d_x + ring_base(L, s->xmax, r));
    J.ldx.push_back(ring_ld(L, r));
    J.kpad.push_back(L->kpad[r]);
    J.koff.push_back(L->koff[r]);
    J.mq.push_back(L->ring_pixels[r]);
    J.col.push_back(L->colpos.data() + L->mask_off[r]);
  }
  J.inv_ld = s->tp;
  J.inv.resize((size_t)Q * s->tp);
  XG_CUDA(c, cudaMemcpyAsync(J.inv.data(), s->d_inv, J.inv.size() * 8, cudaMemcpyDeviceToHost,
                             c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return basis_run(c, J, k, v_out, sigma_out, sigma_ld, rank_out, B);
}

// build_online_from_frames / build_offline over f64 training rows of any
// values (encoder.cpp:32-60 -> gram_svd, linalg.cpp:184-439), on the device:
// row_normalize and S = Xn Xn^T by the reference-order f64 kernels
// (k_exact.cu, so S carries the reference's bits), then the same Jacobi /
// W / Cholesky-QR pipeline as the count builder.  Rings (x_ring[r]: n x
// m_ring[r], host, row-major) are factorised together; v_ring[r] receives
// m_ring[r] x kk (kk = k, or the ring's numerical rank when k = 0).
// rank_out[r]: the rank, or the first zero-norm row (XG_ERR_NORMALIZATION),
// or the achievable rank (XG_ERR_RANK).
static int basis_f64(int32_t Q, const double* const* x_ring, int64_t n, const int64_t* m_ring,
                     int32_t k, double* const* v_ring, double* sigma_out, int64_t* rank_out) {
  if (Q < 1 || !x_ring || !m_ring || !rank_out || n < 2 || k < 0) return XG_ERR_CONTRACT;
  if (n > 2048) return XG_ERR_CONTRACT;  // the device Jacobi's training-row limit
  for (int32_t r = 0; r < Q; ++r)
    if (!x_ring[r] || m_ring[r] < 1) return XG_ERR_CONTRACT;
  xg_ctx cx;
  xg_ctx* c = &cx;
  if (cudaGetDevice(&c->device) != cudaSuccess) return XG_ERR_CUDA;
  cudaStream_t st = nullptr;
  BasisJob J;
  J.Q = Q;
  J.n = n;
  J.x_u8 = false;
  for (int32_t r = 0; r < Q; ++r) {
    J.koff.push_back(J.ktot);
    J.kpad.push_back(m_ring[r]);
    J.ldx.push_back(m_ring[r]);
    J.mq.push_back(m_ring[r]);
    J.ktot += m_ring[r];
  }
  std::vector<int64_t> colv(J.ktot);
  std::iota(colv.begin(), colv.end(), int64_t{0});
  DevBufs db;
  double *d_x, *d_xn, *d_norm, *d_s;
  unsigned long long* d_bad;
  XG_CUDA(c, db.get(&d_x, (size_t)n * J.ktot));
  XG_CUDA(c, db.get(&d_xn, (size_t)n * J.ktot));
  XG_CUDA(c, db.get(&d_norm, (size_t)Q * n));
  XG_CUDA(c, db.get(&d_s, (size_t)Q * n * n));
  XG_CUDA(c, db.get(&d_bad, (size_t)Q));
  XG_CUDA(c, cudaMemsetAsync(d_bad, 0xff, Q * sizeof(unsigned long long), st));
  for (int32_t r = 0; r < Q; ++r) {
    double* xr = d_x + n * J.koff[r];
    XG_CUDA(c, cudaMemcpyAsync(xr, x_ring[r], (size_t)n * m_ring[r] * 8, cudaMemcpyHostToDevice, st));
    XG_CUDA(c, launch_exact_rownorm(xr, n, m_ring[r], d_xn + n * J.koff[r], d_norm + r * n,
                                    d_bad + r, st));
    XG_CUDA(c, launch_exact_gram(d_xn + n * J.koff[r], n, m_ring[r], d_s + (size_t)r * n * n, st));
    J.x.push_back(xr);
    J.col.push_back(colv.data() + J.koff[r]);
  }
  std::vector<unsigned long long> bad(Q);
  J.inv.resize((size_t)Q * n);
  J.inv_ld = n;
  XG_CUDA(c, cudaMemcpyAsync(bad.data(), d_bad, Q * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st));
  XG_CUDA(c, cudaMemcpyAsync(J.inv.data(), d_norm, J.inv.size() * 8, cudaMemcpyDeviceToHost, st));
  XG_CUDA(c, cudaStreamSynchronize(st));
  for (int32_t r = 0; r < Q; ++r)
    if (bad[r] != ~0ull) {  // row_normalize (linalg.cpp:441-456): first zero row
      rank_out[r] = static_cast<int64_t>(bad[r]);
      return XG_ERR_NORMALIZATION;
    }
  for (double& v : J.inv) v = 1.0 / v;
  J.sp = BasisSParams{nullptr, 0, nullptr, 0, 0, 0, nullptr, nullptr, 0, 0, d_s};
  return basis_run(c, J, k, v_ring, sigma_out, n, rank_out, nullptr);
}

int xg_build_basis(const double* x, int64_t n, int64_t m, int32_t k, double* v_out,
                   double* sigma_out, int64_t* rank_out) {
  if (!x || !rank_out || n < 2 || m < 1 || k < 0) return XG_ERR_CONTRACT;
  return basis_f64(1, &x, n, &m, k, &v_out, sigma_out, rank_out);
}

int xg_build_basis_batch(int32_t n_rings, const double* const* x_ring, int64_t n,
                         const int64_t* m_ring, int32_t k, double* const* v_ring,
                         int32_t /*threads: one device pass over all rings*/, int64_t* rank_out) {
  if (n_rings < 1 || !v_ring) return XG_ERR_CONTRACT;
  return basis_f64(n_rings, x_ring, n, m_ring, k, v_ring, nullptr, rank_out);
}

int xg_compress(xg_series* s, const xg_basis* Bc, uint32_t flags) {
  if (!s || !Bc) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  xg_basis* B = const_cast<xg_basis*>(Bc);
  if (s->t < 1) return fail(c, XG_ERR_CONTRACT, "compress: no frames loaded");
  if (s->x_row0 != 0 || s->t > s->xmax)
    return fail(c, XG_ERR_CONTRACT, "compress: series loaded in chunks; compress each chunk");
  int rc = check_basis(s, B);
  if (rc) return rc;
  if ((flags & XG_STRICT) && (rc = strict_zero_check(s, "compress_series"))) return rc;
  rc = compress_rows(s, B, 0, s->t);
  if (rc) return rc;
  s->have_y = true;
  s->have_cttc = false;
  return XG_OK;
}

// One chunk of a series larger than the ring-major buffer: frames [t, t + n)
// (t = frames so far) are ingested into x, their norms land at series rows
// t.., and K3 writes their coefficients/planes at rows t..; the frames are not
// kept.  Chunk 0 resets the series.  Only the compressed path follows.
int xg_series_compress_chunk(xg_series* s, const xg_basis* Bc, const uint8_t* frames, int64_t n,
                             int on_device, uint32_t flags) {
  if (!s || !Bc || !frames) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  xg_basis* B = const_cast<xg_basis*>(Bc);
  int rc = check_basis(s, B);
  if (rc) return rc;
  const int64_t t0 = (flags & XG_CHUNK_FIRST) ? 0 : s->t;
  if (n < 1 || n > s->xmax)
    return fail(c, XG_ERR_SHAPE, "compress_chunk: %lld frames, buffer %lld", (long long)n,
                (long long)s->xmax);
  if (t0 + n > s->tmax)
    return fail(c, XG_ERR_SHAPE, "compress_chunk: %lld frames exceed capacity %lld",
                (long long)(t0 + n), (long long)s->tmax);
  const uint8_t* src = frames;
  if (!on_device) {
    if (int rc0 = ensure_raster(s)) return rc0;
    XG_CUDA(c, cudaMemcpyAsync(s->d_raster, frames, (size_t)n * L->pixels,
                               cudaMemcpyHostToDevice, c->stream));
    src = s->d_raster;
  }
  if (t0 == 0) {
    rc = reset_stats(s, s->tmax);
    if (rc) return rc;
    invalidate_results(s);
  }
  // a chunk grows the series past any raw TTC and replaces the compressed one
  s->have_raw = false;
  s->raw_stored = false;
  s->raw_g2 = false;
  s->have_cttc = false;
  s->cmp_stored = false;
  s->cmp_g2 = false;
  s->x_row0 = t0;
  rc = ingest_range(s, src, t0, n);
  if (rc) return rc;
  if ((flags & XG_STRICT) && (rc = strict_zero_check(s, "compress_series"))) return rc;
  rc = compress_rows(s, B, t0, n);
  if (rc) return rc;
  s->t = t0 + n;
  s->have_y = true;
  s->have_cttc = false;
  return XG_OK;
}

int xg_ttc_compressed(xg_series* s, uint32_t flags) {
  if (!s) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (!s->have_y) return fail(c, XG_ERR_CONTRACT, "ttc_compressed: compress first");
  if (s->t < 2) return fail(c, XG_ERR_CONTRACT, "ttc_compressed: need at least 2 frames");
  const bool store = !(flags & XG_NO_STORE);
  if (!s->d_cg2) {
    XG_CUDA(c, dalloc(&s->d_cg2, (size_t)L->rings * s->tp));
    XG_CUDA(c, dalloc(&s->d_cg2cnt, (size_t)L->rings * s->tp));
  }
  if (flags & XG_G2_SPECTRAL) {
    // g2 only, in the Fourier domain (k_spectral.cu): no C~ tile at all
    if (store || (flags & XG_NO_G2))
      return fail(c, XG_ERR_CONTRACT, "ttc_compressed: XG_G2_SPECTRAL computes g2 only "
                                      "(needs XG_NO_STORE, not XG_NO_G2)");
    const size_t need = spectral_scratch_bytes(L->rings, s->t, s->ck);
    if (need > s->spec_cap) {
      dfree(s->d_spec);
      s->spec_cap = 0;
      XG_CUDA(c, cudaMalloc(&s->d_spec, need));
      s->spec_cap = need;
    }
    SpecParams sp{};
    sp.y = s->d_y;
    sp.y_ld = s->tp;
    sp.k = s->ck;
    sp.n = s->t;
    sp.n_rings = L->rings;
    sp.nz_bits = s->d_nz_bits;
    sp.nz_words = s->nz_words;
    sp.zero_count = s->d_zero;
    sp.g2 = s->d_cg2;
    sp.counts = s->d_cg2cnt;
    sp.g2_ld = s->tp;
    const cudaError_t e = launch_spectral_g2(sp, s->d_spec, c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "spectral g2");
    c->launches += 4;
    s->cmp_stored = false;
    s->have_cttc = true;
    s->cmp_g2 = true;
    return check_device_error(c);
  }
  if (store && !s->d_cgram) XG_CUDA(c, dalloc(&s->d_cgram, (size_t)L->rings * slab_elems(s)));
  int rc = build_tiles(s);
  if (rc) return rc;
  CUtensorMap my;
  rc = make_map_bf16(c, &my, s->d_planes, s->ckp, (int64_t)L->rings * 3 * s->tp);
  if (rc) return rc;
  GramParams gp;
  gp.tiles = s->d_tiles;
  gp.ntiles = s->ntiles;
  gp.ring_koff = L->d_ring_koff;
  gp.ring_nkb = L->d_ring_nkb;
  gp.gram = reinterpret_cast<uint32_t*>(s->d_cgram);
  gp.ring_stride = slab_elems(s);
  gp.ld = static_cast<int32_t>(s->tp);
  gp.nb = ttc_nb(s);
  gp.err = c->d_err;
  gp.max_norm2 = reinterpret_cast<const unsigned long long*>(s->d_max_norm2);
  const bool g2 = !(flags & XG_NO_G2);
  gp.inv = s->d_inv;
  gp.inv2 = s->d_inv2;
  gp.inv_ld = s->tp;
  gp.n_frames = s->t;
  gp.g2_partial = g2 ? s->d_g2tile : nullptr;
  if (flags & XG_CMP_BF16) {  // single bf16 product: hi x hi
    gp.n_pairs = 1;
    gp.pairs = 0x0;
  } else {  // (0,0) (0,1) (1,0) (1,1) (0,2) (2,0): ~24-bit products, f32 accumulate;
    // ascending highest plane (k_gram2.cu: each product waits only for its planes)
    const int pa[6] = {0, 0, 1, 1, 0, 2}, pb[6] = {0, 1, 0, 1, 2, 0};
    gp.n_pairs = 6;
    gp.pairs = 0;
    for (int i = 0; i < 6; ++i) gp.pairs |= (pa[i] | (pb[i] << 2)) << (4 * i);
  }
  gp.kb_per_plane = s->ckp / 64;
  gp.plane_rows = static_cast<int32_t>(s->tp);
  gp.store = store ? 1 : 0;
  s->cmp_stored = store;
  CUtensorMap omap;
  rc = store ? make_map_out32(c, &omap, s->d_cgram, 256, (int64_t)L->rings * slab_elems(s) / 256)
             : make_map_out32(c, &omap, s->d_x, 32, 32);
  if (rc) return rc;
  XG_CUDA(c, launch_gram_any(s, 1, my, omap, gp));
  c->launches++;
  if (g2) {
    rc = fold_g2(s, s->d_cg2, s->d_cg2cnt, true);
    if (rc) return rc;
  }
  s->have_cttc = true;
  s->cmp_g2 = g2;
  return XG_OK;
}

// ------------------------------------------------ analysis consumers (8(f) 4)
int xg_series_ttc_background(xg_series* s, int32_t which, int64_t exclusion, double* out) {
  if (!s || !out) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (which == 0 ? !(s->have_raw && s->raw_stored) : !(s->have_cttc && s->cmp_stored))
    return fail(c, XG_ERR_CONTRACT, "ttc_background: needs a stored %s TTC",
                which == 0 ? "raw" : "compressed");
  if (exclusion < 0 || s->t <= 2 * exclusion)
    return fail(c, XG_ERR_CONTRACT,
                "ttc_background: exclusion band of %lld covers the whole %lld-frame TTC",
                (long long)exclusion, (long long)s->t);
  double2* part = nullptr;
  double* d_buf = nullptr;
  XG_CUDA(c, cudaMalloc(&part, (size_t)L->rings * BG_BLOCKS * sizeof(double2)));
  if (cudaError_t e0 = cudaMalloc(&d_buf, (size_t)L->rings * 8 * 3); e0 != cudaSuccess) {
    cudaFree(part);
    return cuda_fail(c, e0, "ttc_background");
  }
  BgParams p;
  p.gram = which == 0 ? s->d_gram : nullptr;
  p.cgram = which == 0 ? nullptr : s->d_cgram;
  p.ring_stride = slab_elems(s);
  p.nb = ttc_nb(s);
  p.ld = static_cast<int32_t>(s->tp);
  p.inv = s->d_inv;
  p.inv_ld = s->tp;
  p.n = s->t;
  p.excl = exclusion;
  p.n_rings = L->rings;
  p.partial = part;
  p.mean = d_buf;
  p.count = reinterpret_cast<int64_t*>(d_buf + L->rings);
  p.out = d_buf + 2 * L->rings;
  cudaError_t e = launch_ttc_background(p, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, p.out, (size_t)L->rings * 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(part);
  cudaFree(d_buf);
  if (e != cudaSuccess) return cuda_fail(c, e, "ttc_background");
  c->launches += 4;
  for (int32_t r = 0; r < L->rings; ++r)
    if (out[r] < 0.0) {
      c->payload_ring = r;
      return fail(c, XG_ERR_CONTRACT, "ttc_background: no entries outside the band (ring %d)", r);
    }
  return check_device_error(c);
}

int xg_series_fit_kww(xg_series* s, int32_t which, double frame_period, double min_lag,
                      double max_lag, double* out, int32_t* status) {
  if (!s || !out || !status) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (which == 0 ? !(s->have_raw && s->raw_g2) : !(s->have_cttc && s->cmp_g2))
    return fail(c, XG_ERR_CONTRACT, "fit_kww: no %s g2 computed", which == 0 ? "raw" : "compressed");
  if (!(frame_period > 0.0) || !std::isfinite(frame_period))
    return fail(c, XG_ERR_CONTRACT, "fit_kww: frame_period must be positive and finite");
  if (!(min_lag <= max_lag)) return fail(c, XG_ERR_CONTRACT, "fit_kww: window is empty (min > max)");
  double* d_out = nullptr;
  XG_CUDA(c, cudaMalloc(&d_out, (size_t)L->rings * (4 * 8 + 4)));
  KwwParams p;
  p.g2 = which == 0 ? s->d_g2 : s->d_cg2;
  p.g2_ld = s->tp;
  p.n = s->t;
  p.period = frame_period;
  p.min_lag = min_lag;
  p.max_lag = max_lag;
  p.n_rings = L->rings;
  p.out = d_out;
  p.status = reinterpret_cast<int32_t*>(d_out + 4 * L->rings);
  cudaError_t e = launch_fit_kww(p, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, d_out, (size_t)L->rings * 32, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(status, p.status, (size_t)L->rings * 4, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d_out);
  if (e != cudaSuccess) return cuda_fail(c, e, "fit_kww");
  c->launches++;
  return check_device_error(c);
}

int xg_series_get_coeffs(xg_series* s, int32_t ring, double* y, double* norms) {
  if (!s) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->have_y) return fail(c, XG_ERR_CONTRACT, "get_coeffs: compress first");
  if (y)
    XG_CUDA(c, cudaMemcpyAsync(y, s->d_y + (int64_t)ring * s->tp * s->ck,
                               (size_t)s->t * s->ck * 8, cudaMemcpyDeviceToHost, c->stream));
  if (norms)
    XG_CUDA(c, cudaMemcpyAsync(norms, s->d_norms + (int64_t)ring * s->tp, (size_t)s->t * 8,
                               cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

int xg_series_get_cttc(xg_series* s, int32_t ring, int32_t dtype, void* out, int64_t ld,
                       int out_on_device) {
  if (!s || !out) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->have_cttc) return fail(c, XG_ERR_CONTRACT, "get_cttc: no compressed TTC yet");
  if (!s->cmp_stored) return fail(c, XG_ERR_CONTRACT, "get_cttc: computed with XG_NO_STORE");
  if (dtype != XG_F64 && dtype != XG_F32) return fail(c, XG_ERR_CONTRACT, "get_cttc: bad dtype");
  if (ld < s->t) return fail(c, XG_ERR_SHAPE, "get_cttc: ld < n");
  const size_t bytes = (size_t)s->t * ld * (dtype == XG_F64 ? 8 : 4);
  void* dst = out;
  void* tmp = nullptr;
  if (!out_on_device) {
    XG_CUDA(c, ctx_scratch(c, bytes, &tmp));
    dst = tmp;
  }
  ExpandParams p;
  p.gram = nullptr;
  p.cf32 = s->d_cgram + (int64_t)ring * slab_elems(s);
  p.nb = ttc_nb(s);
  p.ring_stride = 0;
  p.ld = static_cast<int32_t>(s->tp);
  p.inv = nullptr;
  p.n = s->t;
  p.out = dst;
  p.out_ld = ld;
  p.out_dtype = dtype;
  cudaError_t e = launch_expand(p, 1, c->stream);
  c->launches++;
  if (e == cudaSuccess && tmp) {
    e = cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "get_cttc");
  return check_device_error(c);
}

int xg_series_get_cg2(xg_series* s, int32_t ring, double* values, int64_t* counts) {
  if (!s || !values) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->have_cttc) return fail(c, XG_ERR_CONTRACT, "get_cg2: no compressed TTC yet");
  XG_CUDA(c, cudaMemcpyAsync(values, s->d_cg2 + (int64_t)ring * s->tp, (size_t)s->t * 8,
                             cudaMemcpyDeviceToHost, c->stream));
  if (counts)
    XG_CUDA(c, cudaMemcpyAsync(counts, s->d_cg2cnt + (int64_t)ring * s->tp, (size_t)s->t * 8,
                               cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

// --------------------------------------------------------------- streaming
}  // extern "C"

struct xg_stream {
  xg_ctx* ctx = nullptr;
  const xg_layout* L = nullptr;
  const xg_basis* B = nullptr;
  uint32_t flags = 0;
  int64_t tmax = 0, t = 0, tp = 0;
  int64_t max_kpad = 0;
  // raw + compressed: the compressed column runs on a side stream, forked
  // after the ingest and joined at the end of the push
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint8_t* d_frame = nullptr;
  uint8_t* d_x = nullptr;
  int64_t *d_norm2 = nullptr, *d_zero = nullptr, *d_first_zero = nullptr;
  double *d_norms = nullptr, *d_inv = nullptr;
  uint32_t* d_nz_bits = nullptr;
  double *d_g2sum = nullptr, *d_cg2sum = nullptr, *d_g2out = nullptr;
  int64_t *d_g2cnt = nullptr, *d_cg2cnt = nullptr;
  int32_t* d_gcol = nullptr;
  float* d_ccol = nullptr;
  int8_t* d_vdt = nullptr;
  int32_t vdt_ld = 0;
  double* d_y = nullptr;
  float* d_yf = nullptr;
  uint8_t* d_hist = nullptr;  // sparse mode: pixel-major history [ktot][hp]
  int32_t* d_colpix = nullptr;  // [ktot] detector pixel of each column (-1 = padding)
  int32_t* d_blk_ring = nullptr;  // [ktot/128] ring of each 128-column block
  int32_t* d_pixcol = nullptr;  // sparse mode: [pixels] ring << 22 | column (-1: no ring)
  int32_t* d_pacc = nullptr;    // with a basis: [ring][768] projection digit sums
  int64_t hp = 0;
  int32_t* d_nz_col = nullptr;
  uint8_t* d_nz_val = nullptr;
  int32_t* d_nz_n = nullptr;     // [3][ring]: counts of push t at t % 3
  // batched photon-event ingest (xg_stream_push_batch): nonzero lists and
  // counts of up to kIngestBatch frames, slot = frame index in the batch
  int32_t* d_nzb_col = nullptr;
  uint8_t* d_nzb_val = nullptr;
  int32_t* d_nzb_n = nullptr;
  // batches ingest on their own stream into two halves of the slots, so
  // batch b + 1's ingest runs beside batch b's columns
  cudaStream_t ing = nullptr;
  cudaEvent_t ev_ing[2] = {nullptr, nullptr}, ev_col[2] = {nullptr, nullptr}, ev_main = nullptr;
  bool col_recorded[2] = {false, false};
  int64_t nbatch = 0;
  // batched columns: per-frame scratch columns [ring][kIngestBatch][tp] and
  // per-frame projection digit sums [kIngestBatch][ring][768]
  int32_t* d_gscr = nullptr;
  float* d_cscr = nullptr;
  int32_t* d_paccb = nullptr;
  bool scr_ready = false;
  // photon-event history of a sparse raw stream (batched columns): blocks
  // of ev_tb frames sealed from the dense history into kEvL1 level-0 slots
  // (k_stream_seal), every kEvL1 consecutive blocks merged into one level-1
  // segment (k_stream_merge); allocated at the first seal.  ev_tb = 0: dense
  // history only (XG_STREAM_EVENT_FRAMES=0, or no memory for the pools).
  int32_t ev_tb = 0;
  int32_t ev_sealed = 0;   // blocks sealed
  int32_t ev_merged = 0;   // level-1 segments
  int64_t ev_cap0 = 0, ev_cap1 = 0;
  uint32_t *d_ev0 = nullptr, *d_ev1 = nullptr;
  int2 *d_evidx0 = nullptr, *d_evidx1 = nullptr;
  unsigned long long *d_ev_cursor0 = nullptr, *d_ev_cursor1 = nullptr;
  int32_t *d_ev_dense0 = nullptr, *d_ev_dense1 = nullptr;
  unsigned int* d_done = nullptr;  // sparse ingest's CTA counters, one per batch frame
};

extern "C" {

int xg_stream_create(xg_ctx* c, const xg_layout* L, const xg_basis* B, int64_t max_frames,
                     uint32_t flags, xg_stream** out) {
  if (!c || !L || !out) return XG_ERR_INVALID;
  *out = nullptr;
  if (max_frames < 1) return fail(c, XG_ERR_CONTRACT, "stream: max_frames must be >= 1");
  if (B && B->L != L) return fail(c, XG_ERR_BINDING, "stream: basis built for another layout");
  if (B && B->digits * B->k > 768)
    return fail(c, XG_ERR_CONTRACT, "stream: digits x k = %d exceeds 768 (k <= 256 at 3 digits)",
                B->digits * B->k);
  if (B)
    for (int32_t r = 0; r < L->rings; ++r)
      if (!B->ring_set[r]) return fail(c, XG_ERR_CONTRACT, "stream: basis of ring %d not set", r);
  xg_stream* s = new xg_stream();
  s->ctx = c;
  s->L = L;
  s->B = B;
  s->flags = flags;
  s->tmax = max_frames;
  s->tp = round_up(max_frames, 32);
  for (int32_t r = 0; r < L->rings; ++r) s->max_kpad = std::max(s->max_kpad, L->kpad[r]);
  const int64_t Q = L->rings;
  cudaError_t e = cudaSuccess;
  const bool store = (flags & XG_STREAM_STORE_TTC) != 0;
  if ((e = dalloc(&s->d_frame, (size_t)L->pixels)) != cudaSuccess ||
      // the ring-major u8 history (dense K5); sparse mode keeps hist instead
      (e = dalloc(&s->d_x, (flags & XG_STREAM_SPARSE) ? 1 : (size_t)max_frames * L->ktot)) !=
          cudaSuccess ||
      (e = dalloc(&s->d_norm2, (size_t)max_frames * Q)) != cudaSuccess ||
      (e = dalloc(&s->d_zero, (size_t)Q)) != cudaSuccess ||
      (e = dalloc(&s->d_first_zero, (size_t)Q)) != cudaSuccess ||
      (e = dalloc(&s->d_norms, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_inv, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_nz_bits, (size_t)Q * (s->tp / 32))) != cudaSuccess ||
      (e = dalloc(&s->d_g2sum, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_g2cnt, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_cg2sum, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_cg2cnt, (size_t)Q * s->tp)) != cudaSuccess ||
      (e = dalloc(&s->d_g2out, (size_t)s->tp)) != cudaSuccess ||
      (store && (e = dalloc(&s->d_gcol, (size_t)Q * s->tp * s->tp)) != cudaSuccess) ||
      (store && B && (e = dalloc(&s->d_ccol, (size_t)Q * s->tp * s->tp)) != cudaSuccess)) {
    xg_stream_destroy(s);
    return cuda_fail(c, e, "stream alloc");
  }
  if (flags & XG_STREAM_SPARSE) {
    s->hp = round_up(max_frames, 128);  // whole 32-frame lane loads stay inside a row
    if ((e = dalloc(&s->d_hist, (size_t)L->ktot * s->hp)) != cudaSuccess) {
      xg_stream_destroy(s);
      return cuda_fail(c, e, "stream sparse history alloc");
    }
    cudaMemsetAsync(s->d_hist, 0, (size_t)L->ktot * s->hp, c->stream);
    if (!(flags & XG_STREAM_NO_RAW)) {
      const char* ev = getenv("XG_STREAM_EVENT_FRAMES");
      const int tb = ev ? atoi(ev) : 1024;
      s->ev_tb = (tb >= 128 && tb <= 1024 && tb % 128 == 0) ? tb : 0;
    }
    // packed (ring << 22 | column) of every pixel, -1 outside the rings
    std::vector<int32_t> pc(static_cast<size_t>(L->pixels), -1);
    if (L->ktot >= (1 << 22) || L->rings > 512) {
      xg_stream_destroy(s);
      return fail(c, XG_ERR_CONTRACT, "sparse stream: at most 2^22 columns and 512 rings");
    }
    for (int32_t r = 0; r < L->rings; ++r)
      for (int64_t col = L->koff[r]; col < L->koff[r] + L->kpad[r]; ++col)
        if (L->colpix[col] >= 0) pc[L->colpix[col]] = (r << 22) | static_cast<int32_t>(col);
    if ((e = dalloc(&s->d_done, 16)) != cudaSuccess ||  // one per batch frame
        (e = cudaMemset(s->d_done, 0, 16 * sizeof(unsigned int))) != cudaSuccess ||
        (e = dalloc(&s->d_pixcol, pc.size())) != cudaSuccess ||
        (e = cudaMemcpy(s->d_pixcol, pc.data(), pc.size() * 4, cudaMemcpyHostToDevice)) !=
            cudaSuccess) {
      xg_stream_destroy(s);
      return cuda_fail(c, e, "stream sparse pixel table");
    }
  }
  if ((flags & XG_STREAM_SPARSE) || B) {
    // the new frame's nonzeros per ring (sparse raw column, sparse projection)
    // nonzero lists double-buffered and counters triple-buffered by push, so
    // push t + 1's ingest may run beside push t's column kernel (PDL)
    if ((e = dalloc(&s->d_nz_col, (size_t)2 * L->ktot)) != cudaSuccess ||
        (e = dalloc(&s->d_nz_val, (size_t)2 * L->ktot)) != cudaSuccess ||
        (e = dalloc(&s->d_nz_n, (size_t)3 * Q)) != cudaSuccess ||
        (B && (e = dalloc(&s->d_pacc, (size_t)Q * 768)) != cudaSuccess)) {
      xg_stream_destroy(s);
      return cuda_fail(c, e, "stream nonzero lists alloc");
    }
    cudaMemsetAsync(s->d_nz_n, 0, (size_t)3 * Q * 4, c->stream);
    if (B) cudaMemsetAsync(s->d_pacc, 0, (size_t)Q * 768 * 4, c->stream);
  }
  {
    // column -> pixel and 128-column block -> ring tables for the one-frame ingest
    std::vector<int32_t> br(static_cast<size_t>(L->ktot / 128));
    for (int32_t r = 0; r < L->rings; ++r)
      for (int64_t b = L->koff[r] / 128; b < (L->koff[r] + L->kpad[r]) / 128; ++b) br[b] = r;
    if ((e = dalloc(&s->d_colpix, (size_t)L->ktot)) != cudaSuccess ||
        (e = dalloc(&s->d_blk_ring, br.size())) != cudaSuccess ||
        (e = cudaMemcpy(s->d_colpix, L->colpix.data(), (size_t)L->ktot * 4,
                        cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_blk_ring, br.data(), br.size() * 4, cudaMemcpyHostToDevice)) !=
            cudaSuccess) {
      xg_stream_destroy(s);
      return cuda_fail(c, e, "stream ingest tables");
    }
  }
  if (!(flags & XG_STREAM_SPARSE)) cudaMemsetAsync(s->d_x, 0, (size_t)max_frames * L->ktot, c->stream);
  cudaMemsetAsync(s->d_norm2, 0, (size_t)max_frames * Q * 8, c->stream);
  cudaMemsetAsync(s->d_zero, 0, (size_t)Q * 8, c->stream);
  cudaMemsetAsync(s->d_first_zero, 0x7F, (size_t)Q * 8, c->stream);
  cudaMemsetAsync(s->d_nz_bits, 0, (size_t)Q * (s->tp / 32) * 4, c->stream);
  cudaMemsetAsync(s->d_g2sum, 0, (size_t)Q * s->tp * 8, c->stream);
  cudaMemsetAsync(s->d_g2cnt, 0, (size_t)Q * s->tp * 8, c->stream);
  cudaMemsetAsync(s->d_cg2sum, 0, (size_t)Q * s->tp * 8, c->stream);
  cudaMemsetAsync(s->d_cg2cnt, 0, (size_t)Q * s->tp * 8, c->stream);
  if (B) {
    // pixel-major copy of the basis digits: [ktot][digits * k], index s*k + j
    xg_basis* b = const_cast<xg_basis*>(B);
    s->vdt_ld = static_cast<int32_t>(round_up(b->digits * b->k, 16));  // 16-byte rows, zero pad
    std::vector<int8_t> vdt((size_t)L->ktot * s->vdt_ld, 0);
    for (int64_t row = 0; row < b->vrows; ++row) {
      const int64_t nt = row / (b->digits * b->kt), rem = row % (b->digits * b->kt);
      const int64_t dig = rem / b->kt, j = nt * b->kt + rem % b->kt;
      if (j >= b->k) continue;
      for (int32_t q = 0; q < L->rings; ++q) {  // ring-blocked digits
        const int8_t* src = b->h_vd.data() + ring_base(L, b->vrows, q) + row * ring_ld(L, q);
        for (int64_t cc = 0; cc < L->kpad[q]; ++cc)
          if (src[cc])
            vdt[(size_t)(L->koff[q] + cc) * s->vdt_ld + dig * b->k + j] = src[cc];
      }
    }
    if ((e = dalloc(&s->d_vdt, vdt.size())) != cudaSuccess ||
        (e = dalloc(&s->d_y, (size_t)Q * s->tp * b->k)) != cudaSuccess ||
        (e = dalloc(&s->d_yf, (size_t)Q * s->tp * ((b->k + 3) / 4 * 4))) != cudaSuccess ||
        (e = cudaMemcpy(s->d_vdt, vdt.data(), vdt.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
      xg_stream_destroy(s);
      return cuda_fail(c, e, "stream basis");
    }
    cudaMemsetAsync(s->d_yf, 0, (size_t)Q * s->tp * ((b->k + 3) / 4 * 4) * 4, c->stream);
    if (int rc0 = basis_upload(b)) {
      xg_stream_destroy(s);
      return rc0;
    }
  }
  *out = s;
  return XG_OK;
}

void xg_stream_destroy(xg_stream* s) {
  if (!s) return;
  if (s->side) {
    cudaStreamSynchronize(s->side);
    cudaStreamDestroy(s->side);
  }
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  dfree(s->d_frame);
  dfree(s->d_x);
  dfree(s->d_norm2);
  dfree(s->d_zero);
  dfree(s->d_first_zero);
  dfree(s->d_norms);
  dfree(s->d_inv);
  dfree(s->d_nz_bits);
  dfree(s->d_g2sum);
  dfree(s->d_g2cnt);
  dfree(s->d_cg2sum);
  dfree(s->d_cg2cnt);
  dfree(s->d_g2out);
  dfree(s->d_gcol);
  dfree(s->d_ccol);
  dfree(s->d_vdt);
  dfree(s->d_y);
  dfree(s->d_yf);
  dfree(s->d_hist);
  dfree(s->d_colpix);
  dfree(s->d_blk_ring);
  dfree(s->d_pixcol);
  dfree(s->d_done);
  dfree(s->d_pacc);
  dfree(s->d_nz_col);
  dfree(s->d_nz_val);
  dfree(s->d_nz_n);
  if (s->ing) {
    cudaStreamSynchronize(s->ing);
    cudaStreamDestroy(s->ing);
  }
  for (int h = 0; h < 2; ++h) {
    if (s->ev_ing[h]) cudaEventDestroy(s->ev_ing[h]);
    if (s->ev_col[h]) cudaEventDestroy(s->ev_col[h]);
  }
  if (s->ev_main) cudaEventDestroy(s->ev_main);
  dfree(s->d_nzb_col);
  dfree(s->d_nzb_val);
  dfree(s->d_nzb_n);
  dfree(s->d_gscr);
  dfree(s->d_cscr);
  dfree(s->d_paccb);
  dfree(s->d_ev0);
  dfree(s->d_evidx0);
  dfree(s->d_ev_cursor0);
  dfree(s->d_ev_dense0);
  dfree(s->d_ev1);
  dfree(s->d_evidx1);
  dfree(s->d_ev_cursor1);
  dfree(s->d_ev_dense1);
  delete s;
}

int64_t xg_stream_frames(const xg_stream* s) { return s ? s->t : -1; }

// The stream's column-kernel parameters for frame s->t (the per-push nonzero
// list / counter slots and the frame pointer are set by the caller).
static StreamParams column_params(const xg_stream* s) {
  const xg_layout* L = s->L;
  StreamParams sp{};
  sp.x = s->d_x;
  sp.ktot = L->ktot;
  sp.t = s->t;
  sp.ring_koff = L->d_ring_koff;
  sp.ring_nkb = L->d_ring_nkb;
  sp.inv = s->d_inv;
  sp.inv_ld = s->tp;
  sp.g2sum = s->d_g2sum;
  sp.g2cnt = s->d_g2cnt;
  sp.cg2sum = s->d_cg2sum;
  sp.cg2cnt = s->d_cg2cnt;
  sp.g2_ld = s->tp;
  sp.gcol = s->d_gcol;
  sp.ccol = s->d_ccol;
  sp.col_ring_stride = s->tp * s->tp;
  sp.col_ld = s->tp;
  sp.vdt = s->d_vdt;
  sp.vdt_ld = s->vdt_ld;
  sp.n_digits = s->B ? s->B->digits : 0;
  sp.k = s->B ? s->B->k : 0;
  sp.scale = s->B ? s->B->d_scale : nullptr;
  sp.y = s->d_y;
  sp.yf = s->d_yf;
  sp.kq = s->B ? (s->B->k + 3) / 4 * 4 : 0;
  sp.y_ld = s->tp;
  sp.hist = s->d_hist;
  sp.hp = s->hp;
  sp.pacc = s->d_pacc;
  sp.pixcol = s->d_pixcol;
  sp.pixels = L->pixels;
  sp.colpix = s->d_colpix;
  sp.blk_ring = s->d_blk_ring;
  sp.n_rings = L->rings;
  sp.norm2 = reinterpret_cast<unsigned long long*>(s->d_norm2);
  sp.norms_w = s->d_norms;
  sp.inv_w = s->d_inv;
  sp.zero_count = s->d_zero;
  sp.first_zero = s->d_first_zero;
  sp.nz_bits = s->d_nz_bits;
  sp.nz_words = static_cast<int32_t>(s->tp / 32);
  sp.err = s->ctx->d_err;
  sp.ovf_check = (s->flags & XG_STREAM_NO_RAW) ? 0 : 1;
  sp.done = s->d_done;
  return sp;
}

constexpr int kIngestBatchMax = 16;  // frames per push_many batch (kIngestBatch below)

// One push.  slot >= 0: photon-event batch member whose ingest already ran
// (xg_stream_push_batch), its nonzero lists in batch slot `slot`.
static int push_one(xg_stream* s, const uint8_t* frame, int on_device, int slot) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (s->t >= s->tmax) return fail(c, XG_ERR_SHAPE, "stream: capacity %lld reached", (long long)s->tmax);
  // a device frame is read in place when 16-byte aligned (stream-ordered:
  // the caller keeps it valid until the push's work has run)
  const uint8_t* d_frame = s->d_frame;
  if (on_device && (reinterpret_cast<uintptr_t>(frame) & 15u) == 0)
    d_frame = frame;
  else
    XG_CUDA(c, cudaMemcpyAsync(s->d_frame, frame, (size_t)L->pixels,
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               c->stream));
  StreamParams sp = column_params(s);
  sp.nz_col = s->d_nz_col ? s->d_nz_col + (s->t & 1) * L->ktot : nullptr;
  sp.nz_val = s->d_nz_val ? s->d_nz_val + (s->t & 1) * L->ktot : nullptr;
  sp.nz_n = s->d_nz_n ? s->d_nz_n + (s->t % 3) * L->rings : nullptr;
  sp.nz_next = s->d_nz_n ? s->d_nz_n + ((s->t + 1) % 3) * L->rings : nullptr;
  sp.nz_bstride = 0;
  if (slot >= 0) {
    sp.nz_col = s->d_nzb_col + slot * L->ktot;
    sp.nz_val = s->d_nzb_val + slot * L->ktot;
    sp.nz_n = s->d_nzb_n + slot * L->rings;
    sp.nz_next = nullptr;
  }
  sp.frame = d_frame;
  sp.norm2_next = s->t + 1 < s->tmax
                      ? reinterpret_cast<unsigned long long*>(s->d_norm2 + (s->t + 1) * L->rings)
                      : nullptr;
  const bool sparse = (s->flags & XG_STREAM_SPARSE) != 0;
  // raw sparse pushes chain ingest -> [compressed column ->] raw column ->
  // next ingest with programmatic dependent launches on one stream (no launch
  // gaps, no events; k_stream.cu); a staging copy in between takes the
  // ordinary stream order
  const bool pdl = sparse && !(s->flags & XG_STREAM_NO_RAW) && d_frame == frame;
  sp.pdl_wait_end = (pdl && s->B) ? 1 : 0;
  // raw batch members after the first: K5s follows K5s (see k_stream_sparse)
  sp.pdl_wait_fin = (pdl && !s->B && slot > 0) ? 1 : 0;
  if (slot >= 0)
    ;  // ingested with its batch
  else if (sparse)  // its last CTA also finishes the frame's norms
    XG_CUDA(c, launch_stream_ingest_sparse(sp, c->stream, pdl && s->t > 0));
  else
    XG_CUDA(c, launch_stream_ingest(sp, c->stream));
  NormParams np;
  np.t0 = s->t;
  np.norm2 = s->d_norm2;
  np.n_frames = 1;
  np.ld = s->tp;
  np.n_rings = L->rings;
  np.norms = s->d_norms;
  np.inv = s->d_inv;
  np.inv2 = nullptr;
  np.zero_count = s->d_zero;
  np.first_zero = s->d_first_zero;
  np.nz_bits = s->d_nz_bits;
  np.nz_words = static_cast<int32_t>(s->tp / 32);
  np.max_norm2 = nullptr;
  np.err = (s->flags & XG_STREAM_NO_RAW) ? nullptr : c->d_err;  // int32 columns formed
  if (!sparse) XG_CUDA(c, launch_norms(np, c->stream));
  c->launches += slot >= 0 ? 0 : sparse ? 1 : 2;
  // single pushes read the dense pixel-major history (PDL-chained, 0.66 of
  // HBM at depth 8192); a per-frame walk of the event segments measured
  // slower (57 vs 40 us per push: too few CTAs per frame, partial columns)
  const bool raw = !(s->flags & XG_STREAM_NO_RAW);
  const bool fork = raw && s->B && !pdl;  // compressed column on the side stream, overlapped
  if (fork) {
    if (!s->side) {
      XG_CUDA(c, cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
      XG_CUDA(c, cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
      XG_CUDA(c, cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    }
    XG_CUDA(c, cudaEventRecord(s->ev_fork, c->stream));
    XG_CUDA(c, cudaStreamWaitEvent(s->side, s->ev_fork, 0));
  }
  if (s->B) {
    sp.scr_nb = 1;  // one frame: K6 adds its column to the lag sums itself
    XG_CUDA(c, launch_stream_cmp(sp, L->rings, fork ? s->side : c->stream, pdl));
    c->launches += 3;
  }
  if (raw) {
    if (s->flags & XG_STREAM_SPARSE)
      XG_CUDA(c, launch_stream_sparse(sp, L->rings, c->stream, pdl));
    else
      XG_CUDA(c, launch_stream_raw(sp, L->rings, s->max_kpad, c->stream));
    c->launches++;
  }
  if (fork) {
    XG_CUDA(c, cudaEventRecord(s->ev_join, s->side));
    XG_CUDA(c, cudaStreamWaitEvent(c->stream, s->ev_join, 0));
  }
  s->t++;
  return XG_OK;
}

int xg_stream_push(xg_stream* s, const uint8_t* frame, int on_device) {
  if (!s || !frame) return XG_ERR_INVALID;
  return push_one(s, frame, on_device, -1);
}

// n consecutive frames (n x pixels, raster order) in one call: the same as n
// pushes, without the per-frame host round trip of the caller.  Photon-event
// streams fed device frames ingest kIngestBatch frames per launch (one
// latency-bound ingest of ~10 us amortised over the batch instead of paid in
// front of every column), then form the batch's columns together
// (launch_stream_batch): the raw columns of all its frames in one grid, the
// compressed columns with every history row read once for the whole batch,
// and the lag sums folded in frame order -- the raw results bitwise those of
// n pushes, C~ to fp32 rounding (K6 on tensor cores vs the pushes' K6b).
// XG_STREAM_BATCH_COLUMNS=0 runs each frame's columns as in a push instead.
constexpr int kIngestBatch = kIngestBatchMax;
constexpr int kEvL1 = 8;  // level-0 blocks per level-1 event segment

static void free_event_pools(xg_stream* s) {
  dfree(s->d_ev0);
  dfree(s->d_evidx0);
  dfree(s->d_ev_cursor0);
  dfree(s->d_ev_dense0);
  dfree(s->d_ev1);
  dfree(s->d_evidx1);
  dfree(s->d_ev_cursor1);
  dfree(s->d_ev_dense1);
  s->d_ev0 = s->d_ev1 = nullptr;
  s->d_evidx0 = s->d_evidx1 = nullptr;
  s->d_ev_cursor0 = s->d_ev_cursor1 = nullptr;
  s->d_ev_dense0 = s->d_ev_dense1 = nullptr;
}

// Seal the blocks of ev_tb frames that precede the next push (s->t) into the
// level-0 slots, merging every kEvL1 of them into a level-1 segment.  Event
// pools are sized for 1/8 occupancy (ev_cap0 = ktot tb / 8 events per
// block); a block with more events stays dense (k_stream_seal's flag).
static int seal_event_blocks(xg_stream* s) {
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  const int tb = s->ev_tb;
  const int64_t nseg_max = s->tmax / (int64_t{tb} * kEvL1);
  auto sealable = [&] {
    return int64_t{s->ev_sealed + 1} * tb <= s->t && s->ev_sealed - s->ev_merged * kEvL1 < kEvL1;
  };
  if (!sealable()) return XG_OK;
  if (!s->d_ev0) {
    s->ev_cap0 = (L->ktot * tb / 8 + 3) / 4 * 4;  // 16-byte aligned slots (K5e reads uint4)
    s->ev_cap1 = s->ev_cap0 * kEvL1;
    const int64_t n1 = std::max<int64_t>(nseg_max, 1);
    cudaError_t e = dalloc(&s->d_ev0, (size_t)(s->ev_cap0 * kEvL1));
    if (e == cudaSuccess) e = dalloc(&s->d_evidx0, (size_t)(L->ktot * kEvL1));
    if (e == cudaSuccess) e = dalloc(&s->d_ev_cursor0, (size_t)kEvL1);
    if (e == cudaSuccess) e = dalloc(&s->d_ev_dense0, (size_t)kEvL1);
    if (e == cudaSuccess && nseg_max) e = dalloc(&s->d_ev1, (size_t)(s->ev_cap1 * n1));
    if (e == cudaSuccess) e = dalloc(&s->d_evidx1, (size_t)(L->ktot * n1));
    if (e == cudaSuccess) e = dalloc(&s->d_ev_cursor1, (size_t)n1);
    if (e == cudaSuccess) e = dalloc(&s->d_ev_dense1, (size_t)n1);
    if (e != cudaSuccess) {  // no room: keep the dense history
      cudaGetLastError();
      free_event_pools(s);
      s->ev_tb = 0;
      return XG_OK;
    }
    XG_CUDA(c, cudaMemsetAsync(s->d_ev_cursor1, 0, n1 * sizeof(unsigned long long), c->stream));
    XG_CUDA(c, cudaMemsetAsync(s->d_ev_dense1, 0, n1 * sizeof(int32_t), c->stream));
  }
  while (sealable()) {
    const int slot = s->ev_sealed % kEvL1;
    XG_CUDA(c, cudaMemsetAsync(s->d_ev_cursor0 + slot, 0, sizeof(unsigned long long), c->stream));
    XG_CUDA(c, cudaMemsetAsync(s->d_ev_dense0 + slot, 0, sizeof(int32_t), c->stream));
    SealParams sl;
    sl.hist = s->d_hist;
    sl.hp = s->hp;
    sl.ktot = L->ktot;
    sl.block = s->ev_sealed;
    sl.slot = slot;
    sl.tb = tb;
    sl.cap = s->ev_cap0;
    sl.ev = s->d_ev0;
    sl.evidx = s->d_evidx0;
    sl.cursor = s->d_ev_cursor0;
    sl.dense = s->d_ev_dense0;
    XG_CUDA(c, launch_stream_seal(sl, c->stream));
    c->launches++;
    s->ev_sealed++;
    if (s->ev_sealed % kEvL1 == 0 && s->ev_merged < nseg_max) {
      MergeParams mp;
      mp.ev0 = s->d_ev0;
      mp.evidx0 = s->d_evidx0;
      mp.dense0 = s->d_ev_dense0;
      mp.cap0 = s->ev_cap0;
      mp.tb = tb;
      mp.nf = kEvL1;
      mp.ktot = L->ktot;
      mp.seg = s->ev_merged;
      mp.cap1 = s->ev_cap1;
      mp.ev1 = s->d_ev1;
      mp.evidx1 = s->d_evidx1;
      mp.cursor1 = s->d_ev_cursor1;
      mp.dense1 = s->d_ev_dense1;
      XG_CUDA(c, launch_stream_merge(mp, c->stream));
      c->launches++;
      s->ev_merged++;
    }
  }
  return XG_OK;
}

// The sealed event segments of a photon-event stream for the raw column
// kernels: level 0 = merged 8192-frame segments, level 1 = the blocks not yet
// merged (in their slots); frames from s_begin on are read densely.
static void event_params(const xg_stream* s, StreamParams& bp) {
  const int l0 = s->ev_sealed - s->ev_merged * kEvL1;  // level-0 blocks not merged
  bp.ev[0] = s->d_ev1;
  bp.evidx[0] = s->d_evidx1;
  bp.ev_dense[0] = s->d_ev_dense1;
  bp.ev_cap[0] = s->ev_cap1;
  bp.ev_tb[0] = s->ev_tb * kEvL1;
  bp.ev_n[0] = s->ev_merged;
  bp.ev_first[0] = 0;
  bp.ev_ring[0] = 0;
  bp.ev[1] = s->d_ev0;
  bp.evidx[1] = s->d_evidx0;
  bp.ev_dense[1] = s->d_ev_dense0;
  bp.ev_cap[1] = s->ev_cap0;
  bp.ev_tb[1] = s->ev_tb;
  bp.ev_n[1] = l0;
  bp.ev_first[1] = s->ev_merged * kEvL1;
  bp.ev_ring[1] = kEvL1;
  bp.s_begin = int64_t{s->ev_sealed} * s->ev_tb;
}

static bool batch_columns_enabled() {
  static const bool on = [] {
    const char* e = getenv("XG_STREAM_BATCH_COLUMNS");
    return !(e && e[0] == '0');
  }();
  return on;
}
int xg_stream_push_batch(xg_stream* s, const uint8_t* frames, int64_t n, int on_device) {
  if (!s || !frames) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  const xg_layout* L = s->L;
  if (n < 0) return fail(c, XG_ERR_SHAPE, "stream: negative frame count");
  if (s->t + n > s->tmax)
    return fail(c, XG_ERR_SHAPE, "stream: capacity %lld reached", (long long)s->tmax);
  const bool batched = (s->flags & XG_STREAM_SPARSE) && on_device && n > 1 &&
                       (reinterpret_cast<uintptr_t>(frames) & 15u) == 0 && (L->pixels & 15) == 0;
  if (!batched) {
    for (int64_t i = 0; i < n; ++i) {
      const int rc = push_one(s, frames + i * L->pixels, on_device, -1);
      if (rc) return rc;
    }
    return XG_OK;
  }
  // ingest of batch b + 1 beside batch b's columns: a clear gain with one
  // column chain (raw-only or compressed-only: 24.9 -> 22.4 / 21.4 -> 20.7
  // us per frame at C3 depth 19k); with both chains already running side by
  // side it only competes with them (36.7 -> 37.7 us; 37.8 with the ingest
  // on a low-priority stream), so it stays in line
#ifndef XG_ING_OVERLAP_BOTH
#define XG_ING_OVERLAP_BOTH 0
#endif
  const bool both_chains = !(s->flags & XG_STREAM_NO_RAW) && s->B;
  const bool overlap = batch_columns_enabled() && (XG_ING_OVERLAP_BOTH || !both_chains);
  if (!s->d_nzb_col) {  // two halves of kIngestBatch slots
    XG_CUDA(c, dalloc(&s->d_nzb_col, (size_t)2 * kIngestBatch * L->ktot));
    XG_CUDA(c, dalloc(&s->d_nzb_val, (size_t)2 * kIngestBatch * L->ktot));
    XG_CUDA(c, dalloc(&s->d_nzb_n, (size_t)2 * kIngestBatch * L->rings));
  }
  if (overlap) {
    if (!s->ing) {
      XG_CUDA(c, cudaStreamCreateWithFlags(&s->ing, cudaStreamNonBlocking));
      for (int h = 0; h < 2; ++h) {
        XG_CUDA(c, cudaEventCreateWithFlags(&s->ev_ing[h], cudaEventDisableTiming));
        XG_CUDA(c, cudaEventCreateWithFlags(&s->ev_col[h], cudaEventDisableTiming));
      }
      XG_CUDA(c, cudaEventCreateWithFlags(&s->ev_main, cudaEventDisableTiming));
    }
    // earlier work on the main stream (single pushes, readbacks) first
    XG_CUDA(c, cudaEventRecord(s->ev_main, c->stream));
    XG_CUDA(c, cudaStreamWaitEvent(s->ing, s->ev_main, 0));
  }
  for (int64_t i0 = 0; i0 < n; i0 += kIngestBatch) {
    const int nb = static_cast<int>(std::min<int64_t>(kIngestBatch, n - i0));
    const int half = overlap ? static_cast<int>(s->nbatch & 1) : 0;
    int32_t* nzb_col = s->d_nzb_col + (int64_t)half * kIngestBatch * L->ktot;
    uint8_t* nzb_val = s->d_nzb_val + (int64_t)half * kIngestBatch * L->ktot;
    int32_t* nzb_n = s->d_nzb_n + (int64_t)half * kIngestBatch * L->rings;
    cudaStream_t ist = overlap ? s->ing : c->stream;
    StreamParams sp{};
    sp.t = s->t;
    sp.frame = frames + i0 * L->pixels;
    sp.pixels = L->pixels;
    sp.pixcol = s->d_pixcol;
    sp.n_rings = L->rings;
    sp.ring_koff = L->d_ring_koff;
    sp.nz_col = nzb_col;
    sp.nz_val = nzb_val;
    sp.nz_n = nzb_n;
    sp.nz_bstride = L->ktot;
    sp.nz_next = nullptr;
    sp.norm2 = reinterpret_cast<unsigned long long*>(s->d_norm2);
    sp.norm2_next = nullptr;  // rows are zero from creation and written once
    sp.hist = s->d_hist;
    sp.hp = s->hp;
    sp.norms_w = s->d_norms;
    sp.inv_w = s->d_inv;
    sp.inv_ld = s->tp;
    sp.zero_count = s->d_zero;
    sp.first_zero = s->d_first_zero;
    sp.nz_bits = s->d_nz_bits;
    sp.nz_words = static_cast<int32_t>(s->tp / 32);
    sp.err = c->d_err;
    sp.ovf_check = (s->flags & XG_STREAM_NO_RAW) ? 0 : 1;
    sp.done = s->d_done;
    // this half's slots are free once the columns of the batch before the
    // previous one have run (same stream without the overlap)
    if (overlap && s->col_recorded[half]) XG_CUDA(c, cudaStreamWaitEvent(ist, s->ev_col[half], 0));
    XG_CUDA(c, cudaMemsetAsync(nzb_n, 0, (size_t)nb * L->rings * sizeof(int32_t), ist));
    XG_CUDA(c, launch_stream_ingest_sparse(sp, ist, false, nb));
    c->launches++;
    if (overlap) {
      XG_CUDA(c, cudaEventRecord(s->ev_ing[half], ist));
      XG_CUDA(c, cudaStreamWaitEvent(c->stream, s->ev_ing[half], 0));
    }
    const bool raw = !(s->flags & XG_STREAM_NO_RAW);
    if (batch_columns_enabled()) {
      if (!s->scr_ready) {
        const size_t cols = (size_t)L->rings * kIngestBatch * s->tp;
        if (raw) XG_CUDA(c, dalloc(&s->d_gscr, cols));
        if (s->B) {
          if (!s->d_cscr) XG_CUDA(c, dalloc(&s->d_cscr, cols));
          XG_CUDA(c, dalloc(&s->d_paccb, (size_t)kIngestBatch * L->rings * 768));
          XG_CUDA(c, cudaMemsetAsync(s->d_paccb, 0,
                                     (size_t)kIngestBatch * L->rings * 768 * sizeof(int32_t),
                                     c->stream));
        }
        s->scr_ready = true;
      }
      // seal every event block whose frames all precede this batch (while a
      // level-0 slot is free), merging each run of kEvL1 blocks into a
      // level-1 segment
      if (raw && s->ev_tb) {
        const int rc = seal_event_blocks(s);
        if (rc) return rc;
      }
      StreamParams bp = column_params(s);
      if (raw && s->ev_tb && s->ev_sealed) event_params(s, bp);
      bp.nz_col = nzb_col;
      bp.nz_val = nzb_val;
      bp.nz_n = nzb_n;
      bp.nz_bstride = L->ktot;
      bp.pacc = s->d_paccb;
      bp.pacc_bstride = (int64_t)L->rings * 768;
      bp.gscr = raw ? s->d_gscr : nullptr;
      bp.cscr = s->d_cscr;
      bp.scr_ld = s->tp;
      bp.scr_nb = nb;
      if (raw && s->B) {
        // the compressed columns (issue-bound) on the side stream beside the
        // raw columns (latency-bound event walks): both read only this
        // batch's ingest and write disjoint sums
        if (!s->side) {
          XG_CUDA(c, cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
          XG_CUDA(c, cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
          XG_CUDA(c, cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
        }
        XG_CUDA(c, cudaEventRecord(s->ev_fork, c->stream));
        XG_CUDA(c, cudaStreamWaitEvent(s->side, s->ev_fork, 0));
        XG_CUDA(c, launch_stream_batch(bp, L->rings, false, true, s->side));
        XG_CUDA(c, launch_stream_batch(bp, L->rings, true, false, c->stream));
        XG_CUDA(c, cudaEventRecord(s->ev_join, s->side));
        XG_CUDA(c, cudaStreamWaitEvent(c->stream, s->ev_join, 0));
      } else {
        XG_CUDA(c, launch_stream_batch(bp, L->rings, raw, s->B != nullptr, c->stream));
      }
      c->launches += (raw ? 2 + (bp.ev_n[0] > 0) + (bp.ev_n[1] > 0) : 0) + (s->B ? 4 : 0);
      if (overlap) {  // this half's slots are read: the ingest two batches on may reuse them
        XG_CUDA(c, cudaEventRecord(s->ev_col[half], c->stream));
        s->col_recorded[half] = true;
        s->nbatch++;
      }
      s->t += nb;
      continue;
    }
    for (int j = 0; j < nb; ++j) {
      const int rc = push_one(s, frames + (i0 + j) * L->pixels, on_device, j);
      if (rc) return rc;
    }
  }
  // the single-push counters expect push t's slot zeroed by push t - 1
  XG_CUDA(c, cudaMemsetAsync(s->d_nz_n, 0, (size_t)3 * L->rings * sizeof(int32_t), c->stream));
  return XG_OK;
}

// which: 0 raw, 1 compressed
int xg_stream_get_g2(xg_stream* s, int32_t ring, int32_t which, double* values, int64_t* counts) {
  if (!s || !values) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (which == 1 && !s->B) return fail(c, XG_ERR_CONTRACT, "stream has no basis");
  if (s->t < 1) return fail(c, XG_ERR_CONTRACT, "stream is empty");
  const double* sum = (which ? s->d_cg2sum : s->d_g2sum) + (int64_t)ring * s->tp;
  const int64_t* cnt = (which ? s->d_cg2cnt : s->d_g2cnt) + (int64_t)ring * s->tp;
  XG_CUDA(c, launch_g2_div(sum, cnt, s->d_g2out, s->t, c->stream));
  c->launches++;
  XG_CUDA(c, cudaMemcpyAsync(values, s->d_g2out, (size_t)s->t * 8, cudaMemcpyDeviceToHost,
                             c->stream));
  if (counts)
    XG_CUDA(c, cudaMemcpyAsync(counts, cnt, (size_t)s->t * 8, cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

int xg_stream_get_coeffs(xg_stream* s, int32_t ring, double* y, double* norms) {
  if (!s) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (y) {
    if (!s->B) return fail(c, XG_ERR_CONTRACT, "stream has no basis");
    XG_CUDA(c, cudaMemcpyAsync(y, s->d_y + (int64_t)ring * s->tp * s->B->k,
                               (size_t)s->t * s->B->k * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (norms)
    XG_CUDA(c, cudaMemcpyAsync(norms, s->d_norms + (int64_t)ring * s->tp, (size_t)s->t * 8,
                               cudaMemcpyDeviceToHost, c->stream));
  XG_CUDA(c, cudaStreamSynchronize(c->stream));
  return check_device_error(c);
}

// ------------------------------------------------ formats
// rows [t0, t1) of one ring (coefficients [ring][tp][k], norms [ring][tp])
// to an XCMP store through the host writer (xg_io.cpp)
static int write_xcmp_rows(xg_ctx* c, const double* d_y, const double* d_norms, int64_t tp,
                           int64_t k, int32_t ring, int64_t t0, int64_t t1, const char* path,
                           uint64_t hash, int32_t append) {
  const int64_t n = t1 - t0;
  std::vector<double> y((size_t)std::max<int64_t>(n, 0) * k), nr((size_t)std::max<int64_t>(n, 0));
  if (n > 0) {
    XG_CUDA(c, cudaMemcpyAsync(y.data(), d_y + ((int64_t)ring * tp + t0) * k, (size_t)n * k * 8,
                               cudaMemcpyDeviceToHost, c->stream));
    XG_CUDA(c, cudaMemcpyAsync(nr.data(), d_norms + (int64_t)ring * tp + t0, (size_t)n * 8,
                               cudaMemcpyDeviceToHost, c->stream));
    XG_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  // Device rows come from the 3-digit int8 basis (|dV| <= 3e-8 max|V|): a
  // row of a frame inside the basis span may land a few 1e-9 above unit norm,
  // which the reference's append (model.cpp:184-193) would reject on read.
  // Such rows are rescaled to unit norm (the projection of a unit row has
  // norm <= 1 exactly); anything further above 1 is a real contract error.
  for (int64_t i = 0; i < n; ++i) {
    double* row = y.data() + (size_t)i * k;
    double sq = 0.0;
    for (int64_t j = 0; j < k; ++j) sq += row[j] * row[j];
    if (sq > (1.0 + 1e-10) * (1.0 + 1e-10) && sq <= (1.0 + 1e-6) * (1.0 + 1e-6)) {
      const double inv = 1.0 / std::sqrt(sq);
      for (int64_t j = 0; j < k; ++j) row[j] *= inv;
    }
  }
  const int rc = xg_io_write_xcmp(path, k, hash, n, nr.data(), y.data(), append);
  if (rc == XG_OK) return check_device_error(c);
  if (rc == XG_ERR_NORMALIZATION) {
    c->payload = t0 + xg_io_last_payload();
    c->payload_ring = ring;
    return fail(c, rc, "write_xcmp: frame %lld of ring %d has zero norm", (long long)c->payload, ring);
  }
  if (rc == XG_ERR_FORMAT) c->payload = xg_io_last_payload();
  return fail(c, rc, "%s", xg_io_last_error());
}

int xg_series_write_xcmp(xg_series* s, int32_t ring, const char* path, uint64_t hash,
                         int32_t append) {
  if (!s || !path) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->have_y) return fail(c, XG_ERR_CONTRACT, "write_xcmp: compress first");
  return write_xcmp_rows(c, s->d_y, s->d_norms, s->tp, s->ck, ring, 0, s->t, path, hash, append);
}

int xg_stream_append_xcmp(xg_stream* s, int32_t ring, const char* path, uint64_t hash,
                          int64_t from_frame) {
  if (!s || !path) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (!s->B) return fail(c, XG_ERR_CONTRACT, "stream has no basis");
  if (from_frame < 0 || from_frame > s->t)
    return fail(c, XG_ERR_SHAPE, "append_xcmp: from_frame %lld outside [0, %lld]",
                (long long)from_frame, (long long)s->t);
  return write_xcmp_rows(c, s->d_y, s->d_norms, s->tp, s->B->k, ring, from_frame, s->t, path, hash, 1);
}

// TTC tile sink: "XTTC", u32 version 1, u32 dtype (0 f64 C, 1 f32 C~, 2 i32
// exact Gram), u64 n, then the upper triangle row after row (row i: columns
// i .. n-1), little-endian; size 20 + n (n + 1) / 2 * elem.  Streamed from
// the stored tiles in blocks of 256 rows (CSV export, io.cpp:465-478, does
// not scale to C4/C5 TTCs).
int xg_series_write_ttc(xg_series* s, int32_t ring, int32_t which, int32_t dtype,
                        const char* path) {
  if (!s || !path) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if (which == 0 ? !(s->have_raw && s->raw_stored) : !(s->have_cttc && s->cmp_stored))
    return fail(c, XG_ERR_CONTRACT, "write_ttc: needs a stored %s TTC", which == 0 ? "raw" : "compressed");
  if (which == 0 ? (dtype != XG_F64 && dtype != XG_I32_GRAM) : dtype != XG_F32)
    return fail(c, XG_ERR_CONTRACT, "write_ttc: dtype %d not available for this TTC", dtype);
  const int64_t n = s->t;
  const int elem = dtype == XG_F64 ? 8 : 4;
  const uint32_t code = dtype == XG_F64 ? 0u : dtype == XG_F32 ? 1u : 2u;
  FILE* f = fopen(path, "wb");
  if (!f) return fail(c, XG_ERR_FORMAT, "cannot create TTC file %s", path);
  struct Closer {
    FILE* f;
    ~Closer() {
      if (f) fclose(f);
    }
  } closer{f};
  uint8_t head[20];
  std::memcpy(head, "XTTC", 4);
  const uint32_t ver = 1;
  const uint64_t nn = static_cast<uint64_t>(n);
  for (int i = 0; i < 4; ++i) head[4 + i] = static_cast<uint8_t>(ver >> (8 * i));
  for (int i = 0; i < 4; ++i) head[8 + i] = static_cast<uint8_t>(code >> (8 * i));
  for (int i = 0; i < 8; ++i) head[12 + i] = static_cast<uint8_t>(nn >> (8 * i));
  if (fwrite(head, 1, 20, f) != 20) return fail(c, XG_ERR_FORMAT, "failed writing TTC file %s", path);
  constexpr int64_t RB = 256;
  const size_t cap = static_cast<size_t>(RB) * n * elem;
  void* d_stage = nullptr;
  XG_CUDA(c, cudaMalloc(&d_stage, cap));
  std::vector<uint8_t> h(cap);
  ExpandParams p;
  p.gram = which == 0 ? s->d_gram + (int64_t)ring * slab_elems(s) : nullptr;
  p.cf32 = which == 0 ? nullptr : s->d_cgram + (int64_t)ring * slab_elems(s);
  p.nb = ttc_nb(s);
  p.ring_stride = 0;
  p.ld = static_cast<int32_t>(s->tp);
  p.inv = s->d_inv + (int64_t)ring * s->tp;
  p.n = n;
  p.out = d_stage;
  p.out_ld = 0;
  p.out_dtype = dtype;
  int rc = XG_OK;
  for (int64_t r0 = 0; r0 < n && rc == XG_OK; r0 += RB) {
    const int64_t rows = std::min(RB, n - r0);
    const int64_t cnt = rows * n - ((r0 + rows) * (r0 + rows - 1) / 2 - r0 * (r0 - 1) / 2);
    cudaError_t e = launch_pack_upper(p, which, r0, rows, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h.data(), d_stage, (size_t)cnt * elem, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      rc = cuda_fail(c, e, "write_ttc");
      break;
    }
    c->launches++;
    if (fwrite(h.data(), 1, (size_t)cnt * elem, f) != (size_t)cnt * elem)
      rc = fail(c, XG_ERR_FORMAT, "failed writing TTC file %s", path);
  }
  cudaFree(d_stage);
  if (rc) return rc;
  closer.f = nullptr;
  if (fclose(f) != 0) return fail(c, XG_ERR_FORMAT, "failed writing TTC file %s", path);
  return check_device_error(c);
}

int xg_series_load_xfsr(xg_series* s, const char* path, double* period) {
  if (!s || !path) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  int64_t n = 0, m = 0;
  double per = 0.0;
  int rc = xg_io_read_xfsr_u8(path, nullptr, 0, &n, &m, &per);
  if (rc == XG_OK) {
    if (m != s->L->pixels)
      return fail(c, XG_ERR_SHAPE, "load_xfsr: file frames have %lld pixels, layout %lld",
                  (long long)m, (long long)s->L->pixels);
    if (n > s->xmax)
      return fail(c, XG_ERR_SHAPE, "load_xfsr: %lld frames, capacity %lld", (long long)n,
                  (long long)s->xmax);
    std::vector<uint8_t> buf((size_t)n * m);
    rc = xg_io_read_xfsr_u8(path, buf.data(), (int64_t)buf.size(), &n, &m, &per);
    if (rc == XG_OK) {
      if (period) *period = per;
      return xg_series_load_frames(s, buf.data(), n, 0);
    }
  }
  if (rc == XG_ERR_FORMAT || rc == XG_ERR_CONTRACT) c->payload = xg_io_last_payload();
  return fail(c, rc, "%s", xg_io_last_error());
}

// Full n x n TTC of a ring from the stored columns (XG_STREAM_STORE_TTC).
int xg_stream_get_ttc(xg_stream* s, int32_t ring, int32_t which, int32_t dtype, void* out,
                      int64_t ld) {
  if (!s || !out) return XG_ERR_INVALID;
  xg_ctx* c = s->ctx;
  if (ring < 0 || ring >= s->L->rings) return fail(c, XG_ERR_SHAPE, "ring %d out of range", ring);
  if ((which == 0 && !s->d_gcol) || (which == 1 && !s->d_ccol))
    return fail(c, XG_ERR_CONTRACT, "stream was created without XG_STREAM_STORE_TTC");
  if (ld < s->t) return fail(c, XG_ERR_SHAPE, "get_ttc: ld < n");
  if (which == 1 && dtype == XG_I32_GRAM) return fail(c, XG_ERR_CONTRACT, "bad dtype");
  const size_t bytes = (size_t)s->t * ld * (dtype == XG_F64 ? 8 : 4);
  void* tmp = nullptr;
  XG_CUDA(c, ctx_scratch(c, bytes, &tmp));
  ExpandParams p;
  p.gram = which == 0 ? s->d_gcol + (int64_t)ring * s->tp * s->tp : nullptr;
  p.cf32 = which == 1 ? s->d_ccol + (int64_t)ring * s->tp * s->tp : nullptr;
  p.ring_stride = 0;
  p.ld = static_cast<int32_t>(s->tp);
  p.inv = s->d_inv + (int64_t)ring * s->tp;
  p.n = s->t;
  p.out = tmp;
  p.out_ld = ld;
  p.out_dtype = dtype;
  cudaError_t e = launch_expand(p, which, c->stream);
  c->launches++;
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "stream get_ttc");
  return check_device_error(c);
}

}  // extern "C"
