/*
 * xpcs_b200.h -- C ABI of the B200-native XPCS correlation hot path.
 *
 * This is the drop-in boundary for the reference's operator API
 * (namespace xpcs, /root/reference/proj/include/xpcsvd/{correlate,compress,
 * model}.hpp).  The reference has no FFI of its own; its C++ API is bound
 * one-to-one by the C++ facade in include/xpcs_b200.hpp (and by
 * paper_2407_20356_b200/_abi.py through ctypes), see INTEGRATION.md.
 *
 * Conventions
 *   - plain pointers + sizes, no exceptions cross this boundary;
 *   - every entry returns an xg_status; on error xg_last_error() gives the
 *     message, xg_last_error_payload() the frame index (NormalizationError
 *     frame_index, errors.hpp:36-45) / achievable rank (RankError);
 *   - the caller owns host buffers, the library owns device buffers behind
 *     the opaque handles; `*_on_device` flags say whether a pointer is a
 *     device pointer (0 = host);
 *   - a context is bound to one device and one CUDA stream and is not
 *     re-entrant (single writer, like CompressedSeries, model.hpp:85-122).
 *   - matrices are row-major; TTC values are returned as the reference's
 *     f64 (or f32 / exact int32 Gram on request).
 */
#ifndef XPCS_B200_H_
#define XPCS_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define XG_API __attribute__((visibility("default")))
#else
#define XG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: one per xpcs::Error subclass (errors.hpp:11-74). */
typedef enum xg_status {
  XG_OK = 0,
  XG_ERR_SHAPE = 1,          /* xpcs::ShapeError */
  XG_ERR_CONTRACT = 2,       /* xpcs::ContractError */
  XG_ERR_MASK = 3,           /* xpcs::MaskError */
  XG_ERR_NORMALIZATION = 4,  /* xpcs::NormalizationError (payload = frame) */
  XG_ERR_RANK = 5,           /* xpcs::RankError (payload = achievable rank) */
  XG_ERR_BINDING = 6,        /* xpcs::BindingError */
  XG_ERR_FORMAT = 7,         /* xpcs::FormatError */
  XG_ERR_CUDA = 100,         /* CUDA runtime / launch failure */
  XG_ERR_DEVICE = 101,       /* no sm_100 device, or kernel self-check failed */
  XG_ERR_INVALID = 102       /* bad handle / null pointer */
} xg_status;

/* Output element types for TTC readback. */
typedef enum xg_dtype { XG_F64 = 0, XG_F32 = 1, XG_I32_GRAM = 2 } xg_dtype;

/* Flags */
#define XG_STRICT 0x1u      /* zero-norm frame -> XG_ERR_NORMALIZATION (reference
                              behaviour, linalg.cpp:446-449); default flags the
                              frame and excludes it from g2 instead */
#define XG_NO_G2 0x2u       /* skip the g2 reduction */
#define XG_CMP_BF16 0x4u    /* compressed Gram from the bf16 coefficients only
                              (one product; ~1e-2 relative) instead of the
                              bf16x3 split (6 products; ~1e-6 relative) */
#define XG_CHUNK_FIRST 0x10u /* xg_series_compress_chunk: first chunk of a series */
#define XG_G2_SPECTRAL 0x20u /* xg_ttc_compressed: g2 only, from the coefficient series'
                              autocorrelations by FFT (no C~ tile is formed; f64) */
#define XG_NO_STORE 0x8u    /* g2 only: the TTC tiles never leave the chip (no
                              Q x T x T buffer is allocated or written; TTC
                              readback then fails) -- series whose TTC outgrows
                              HBM */

typedef struct xg_ctx xg_ctx;
typedef struct xg_layout xg_layout;
typedef struct xg_series xg_series;
typedef struct xg_basis xg_basis;
typedef struct xg_stream xg_stream;

/* ---- library / context ------------------------------------------------ */
XG_API int xg_version(void);
/* device: CUDA ordinal; stream: a cudaStream_t (NULL = library-owned). */
XG_API int xg_ctx_create(int device, void* stream, xg_ctx** out);
XG_API void xg_ctx_destroy(xg_ctx* ctx);
XG_API const char* xg_last_error(const xg_ctx* ctx);
XG_API int64_t xg_last_error_payload(const xg_ctx* ctx, int32_t* ring);
XG_API int xg_synchronize(xg_ctx* ctx);
/* Number of kernels this library launched on ctx since creation. */
XG_API int64_t xg_kernel_launches(const xg_ctx* ctx);

/* ---- q-ring layout ----------------------------------------------------
 * A set of PixelMask (model.hpp:16-24, model.cpp:10-26): ring r selects
 * mask_indices[mask_offsets[r] .. mask_offsets[r+1]), strictly ascending and
 * < full_pixels.  Replaces the per-ring apply_mask column gather
 * (model.cpp:42-59) by one device permutation into a ring-major, zero-padded
 * u8 layout. */
XG_API int xg_layout_create(xg_ctx* ctx, int64_t full_pixels, int32_t n_rings,
                     const int64_t* mask_offsets, const int64_t* mask_indices,
                     xg_layout** out);
/* The same for a height x width row-major detector (full_pixels = height *
 * width): on a detector wider than 512 pixels the ingest reads 32-row x
 * 512-column blocks instead of 16384-pixel raster strips, so each band holds
 * longer pieces of every annulus (the ring-major column order differs;
 * every result is the same). */
XG_API int xg_layout_create_2d(xg_ctx* ctx, int64_t height, int64_t width, int32_t n_rings,
                               const int64_t* mask_offsets, const int64_t* mask_indices,
                               xg_layout** out);
XG_API void xg_layout_destroy(xg_layout* layout);
XG_API int64_t xg_layout_ring_pixels(const xg_layout* layout, int32_t ring);

/* ---- batch series (FrameSeries + TTC per ring) ------------------------ */
XG_API int xg_series_create(xg_ctx* ctx, const xg_layout* layout, int64_t max_frames,
                     xg_series** out);
/* A series of up to max_frames whose ring-major frame buffer holds only
 * x_frames (<= max_frames): for series larger than HBM, frames are fed in
 * chunks through xg_series_compress_chunk (compressed path only). */
XG_API int xg_series_create2(xg_ctx* ctx, const xg_layout* layout, int64_t max_frames,
                             int64_t x_frames, xg_series** out);
XG_API void xg_series_destroy(xg_series* s);
/* frames: n_frames x full_pixels u8 photon counts (raster order).  Ingest:
 * [H2D] + ring permutation + per-(frame, ring) statistics. */
XG_API int xg_series_load_frames(xg_series* s, const uint8_t* frames, int64_t n_frames,
                          int frames_on_device);
/* Photon-event frames (what event-mode photon-counting detectors emit, and
 * ~1/4 of the raster's PCIe bytes at 0.05 photons/pixel): frame f's events
 * are pix[frame_off[f] .. frame_off[f+1]) (raster pixel indices, unique
 * within a frame) with counts val[...] (>= 1); every other pixel is 0.
 * Loads the same series as xg_series_load_frames of the dense frames (Gram,
 * norms, g2 bitwise identical): the ring-major rows are cleared and the
 * events scattered into them, |x|^2 summed per (frame, ring).  Pixels
 * outside every ring are ignored; an index outside [0, full_pixels) is an
 * XG_ERR_SHAPE at the next synchronising call.  Buffers on the host (copied
 * H2D: 8 (n + 1) + 5 nnz bytes) or, with on_device, in device memory.
 * Replaces the frame-by-frame raster fill in front of
 * FrameSeries::push_back (model.cpp:28-40). */
XG_API int xg_series_load_events(xg_series* s, const int64_t* frame_off, const int32_t* pix,
                                 const uint8_t* val, int64_t n_frames, int on_device);
/* Raw two-time correlation of every ring (ttc_raw, correlate.cpp:19-25):
 * exact u8 x u8 -> int32 Gram on tcgen05 tensor cores, f64 normalisation and
 * g2 (g2_from_ttc, correlate.cpp:67-85) on the device.  Asynchronous: a
 * contract violation found on the device (a frame with |x|^2 >= 2^31, which
 * the int32 Gram cannot hold) is returned as XG_ERR_CONTRACT by the next
 * synchronising call (any readback, xg_synchronize).  XG_STRICT checks the
 * zero-frame rule (NormalizationError) before launching. */
XG_API int xg_ttc_raw(xg_series* s, uint32_t flags);
/* xg_series_load_frames + xg_ttc_raw for frames in host memory (pinned for
 * full overlap): chunked H2D on a second stream overlapped with ingest and
 * the Gram tiles each arrived chunk completes.  Same results. */
XG_API int xg_series_ttc_raw_host(xg_series* s, const uint8_t* frames, int64_t n_frames,
                                  uint32_t flags);
/* xg_series_load_events + xg_ttc_raw for event lists in host memory (pinned
 * for full overlap): the frames' events cross PCIe in chunks of whole
 * 256-frame column blocks on a second stream, each chunk scattered and its
 * Gram tiles run as it lands.  Same results. */
XG_API int xg_series_ttc_raw_events_host(xg_series* s, const int64_t* frame_off,
                                         const int32_t* pix, const uint8_t* val, int64_t n_frames,
                                         uint32_t flags);
/* g2 of every ring from the current raw TTC (run separately after
 * xg_ttc_raw(..., XG_NO_G2)). */
XG_API int xg_series_g2(xg_series* s);
/* Split rings across processes (multi-GPU).  The Gram and the
 * frame norms^2 of a ring are sums over its pixels (gram, linalg.cpp:127-156),
 * so a ring whose pixels are divided among processes is exact after an
 * integer sum of the per-process partials.  Each process runs xg_ttc_raw on
 * its share (stored, not XG_NO_STORE); xg_series_export_partial writes the
 * share's exact Gram as the packed upper 256 x 256 pair tiles (I <= J in
 * (I, J) row-major order, xg_series_partial_elems() int32 values) and its
 * |x_t|^2 column (n_frames int64); the caller sums them (e.g. NCCL int32 /
 * int64 sum, or send + add); xg_series_import_partial writes the total back
 * into one process's series and refreshes the ring's norms, zero-frame
 * bookkeeping and (unless XG_NO_G2) g2.  XG_STRICT raises the reference's
 * NormalizationError for a zero frame of the summed ring; a summed |x|^2 >=
 * 2^31 is reported as XG_ERR_CONTRACT by the next synchronising call.
 * on_device: the buffers are device (1) or host (0) memory. */
XG_API int64_t xg_series_partial_elems(const xg_series* s);
XG_API int xg_series_export_partial(xg_series* s, int32_t ring, int32_t* gram, int64_t* norm2,
                                    int on_device);
XG_API int xg_series_import_partial(xg_series* s, int32_t ring, const int32_t* gram,
                                    const int64_t* norm2, int on_device, uint32_t flags);
/* Readback.  dtype XG_F64/XG_F32: C = G_ij / (|x_i| |x_j|) (full symmetric
 * n x n, ld elements per row); XG_I32_GRAM: the exact integer Gram. */
XG_API int xg_series_get_ttc(xg_series* s, int32_t ring, int32_t dtype, void* out, int64_t ld,
                      int out_on_device);
/* g2 values (n), counts (n; N-d, or fewer when frames were flagged), lags in
 * frames (multiply by frame_period for seconds). */
XG_API int xg_series_get_g2(xg_series* s, int32_t ring, double* values, int64_t* counts);
/* Device pointers of every ring's g2 values / pair counts (which: 0 raw, 1
 * compressed), [ring][ld] with n_frames valid per ring; borrowed, valid until
 * the series is recomputed or destroyed (collectives gather g2 without a
 * host round trip). */
XG_API int xg_series_g2_device(xg_series* s, int32_t which, const double** values,
                               const int64_t** counts, int64_t* ld);
/* g2 and pair counts of every ring in one transfer: [ring][n_frames] each */
XG_API int xg_series_get_g2_all(xg_series* s, double* values, int64_t* counts);
/* Deviation of the homomorphic path per ring (ttc_rel_error, correlate.cpp:
 * 87-108): ||C - C~||_F / ||C||_F over the full symmetric matrices, from the
 * stored raw TTC and compressed TTC (both computed, not XG_NO_STORE). */
XG_API int xg_series_rel_error(xg_series* s, double* out_per_ring);
/* f64 frame norms |x_t| of ring (n) and the count of zero-norm frames. */
XG_API int xg_series_get_norms(xg_series* s, int32_t ring, double* norms, int64_t* n_zero);
/* Analysis consumers on the device (which: 0 raw, 1
 * compressed).  ttc_background (analysis.cpp:202-235): per ring, the
 * standard deviation of the stored TTC entries with lag > exclusion (two
 * passes: mean, then squared deviations; pairs with a flagged zero-norm frame
 * left out, as in g2).  fit_kww (analysis.cpp:77-172): per ring, the KWW fit
 * g2 = B + C exp(-2 lag / t0) of the device g2 curve over lags
 * [min_lag, max_lag] (lags d * frame_period), the reference's initialisation
 * and damped Gauss-Newton; out[ring * 4 + {0..3}] = B, C, t0, residual rms;
 * status[ring] = 0 ok, 1 FitDegenerateError, 2 FitError (out = the last
 * accepted iterate), 3 ContractError (fewer than 5 points / non-finite). */
/* On-disk formats next to the device buffers (the
 * reference's io.cpp).  XCMP store (io.cpp:319-441): xg_series_write_xcmp
 * writes one ring's compressed rows (norm + k f64 coefficients per frame),
 * or with append != 0 extends an existing store like CompressedFileAppender
 * (k mismatch -> XG_ERR_SHAPE, encoder hash -> XG_ERR_BINDING, corrupt
 * file -> XG_ERR_FORMAT with the byte offset); xg_stream_append_xcmp appends
 * the stream's rows [from_frame, t).  A flagged zero-norm frame cannot be
 * stored (XG_ERR_NORMALIZATION, payload = frame).  XFSR frames (io.cpp:150-
 * 225): dtype 0 u16 / 1 f32 / 2 f64 as the reference, dtype 3 = u8 photon
 * counts (new); xg_series_load_xfsr reads any of them into the series
 * (values must be integer counts in [0, 255]).  Host-only helpers report
 * through xg_io_last_error / xg_io_last_payload. */
/* Device coefficient rows a few 1e-9 above unit norm (the 3-digit int8 basis
 * of a frame inside the basis span) are rescaled to unit norm before writing,
 * so the reference reader's append() (model.cpp:184-193) accepts the store;
 * rows further above 1, non-finite rows (and, in xg_io_write_xcmp, any row
 * above 1 + 1e-10) are XG_ERR_CONTRACT. */
XG_API int xg_series_write_xcmp(xg_series* s, int32_t ring, const char* path,
                                uint64_t encoder_hash, int32_t append);
XG_API int xg_stream_append_xcmp(xg_stream* s, int32_t ring, const char* path,
                                 uint64_t encoder_hash, int64_t from_frame);
XG_API int xg_series_load_xfsr(xg_series* s, const char* path, double* frame_period);
/* TTC tile sink (new format; CSV export, io.cpp:465-478, does not scale to
 * C4/C5): "XTTC", u32 1, u32 dtype (0 f64 C, 1 f32 C~, 2 i32 exact Gram),
 * u64 n, then the upper triangle row after row (row i: columns i..n-1),
 * streamed from the stored tiles; which 0 raw (XG_F64 or XG_I32_GRAM),
 * 1 compressed (XG_F32). */
XG_API int xg_series_write_ttc(xg_series* s, int32_t ring, int32_t which, int32_t dtype,
                               const char* path);
XG_API const char* xg_io_last_error(void);
XG_API int64_t xg_io_last_payload(void);
XG_API int xg_io_write_xcmp(const char* path, int64_t k, uint64_t encoder_hash, int64_t n,
                            const double* norms, const double* coeffs, int32_t append);
XG_API int xg_io_write_xfsr_u8(const char* path, const uint8_t* frames, int64_t n, int64_t m,
                               double frame_period);
XG_API int xg_io_read_xfsr_u8(const char* path, uint8_t* out, int64_t out_cap, int64_t* n,
                              int64_t* m, double* frame_period);
/* XENC encoder file (io.cpp:273-321): a device-built basis (V per ring,
 * mask order) saved for / read from the reference.  read: v == null returns
 * the header only (mode, m, k, spectrum_len). */
XG_API int xg_io_write_xenc(const char* path, int32_t mode, int64_t m, int64_t k,
                            const double* spectrum, int64_t spectrum_len, const double* v);
XG_API int xg_io_read_xenc(const char* path, int32_t* mode, int64_t* m, int64_t* k,
                           int64_t* spectrum_len, double* spectrum, double* v);
XG_API int xg_series_ttc_background(xg_series* s, int32_t which, int64_t exclusion,
                                    double* out_per_ring);
XG_API int xg_series_fit_kww(xg_series* s, int32_t which, double frame_period, double min_lag,
                             double max_lag, double* out, int32_t* status);
XG_API int64_t xg_series_frames(const xg_series* s);

/* ---- rank-k compression and the homomorphic TTC -----------------------
 * Basis: one EncodingMatrix V_q (M_q x k, orthonormal columns, mask row
 * order; model.hpp:53-67) per ring, stored on the device as `digits` signed
 * int8 planes per column (V ~= s (d0 + d1/254 + d2/254^2); 3 digits keep
 * ~3e-8 of max|V|, 2 digits ~8e-6).  xg_compress = compress_series
 * (compress.cpp:48-81): Y_q = (X_q/|x|) V_q on tcgen05 int8 tensor cores,
 * exact integer accumulation, f64 combination.  xg_ttc_compressed =
 * ttc_compressed (correlate.cpp:27-35): C~_q = Y_q Y_q^T on tcgen05 bf16 tensor
 * cores (bf16x3 split, or XG_CMP_BF16) + fused g2. */
/* Basis construction from f64 training rows of any values (host buffers in,
 * computed on the CURRENT CUDA device by K9; untimed setup).  The reference's
 * encoder_from_rows (encoder.cpp:13-28): row_normalize and S = Xn Xn^T in the
 * reference's f64 order (k_exact.cu) -> parallel-order Jacobi (linalg.cpp:
 * 234-276) -> measured sigma, rank at 1e-12 sigma_max -> 2x Cholesky-QR ->
 * largest entry positive -> first k right vectors.  k = 0 keeps the full
 * numerical rank (build_offline).  2 <= n <= 2048 rows.  Returns XG_ERR_RANK
 * with the achievable rank in *rank_out when k exceeds it,
 * XG_ERR_NORMALIZATION with the zero frame in *rank_out, XG_ERR_CUDA without
 * a device.  Photon-count series use xg_series_build_basis (exact Gram). */
XG_API int xg_build_basis(const double* x, int64_t n, int64_t m, int32_t k, double* v_out,
                          double* sigma_out, int64_t* rank_out);
/* content_hash_u64 (model.cpp:99-114): 64-bit FNV-1a over "XENC", the mode
 * byte (0 offline, 1 online-related, 2 online-unrelated), n_pixels, k and the
 * f64 bits of V (m x k row-major), little-endian.  The store binding id. */
XG_API uint64_t xg_content_hash(const double* v, int64_t m, int64_t k, int32_t mode);
/* Every ring at once (x_ring[r]: n x m_ring[r]); threads is ignored (one
 * device pass). */
XG_API int xg_build_basis_batch(int32_t n_rings, const double* const* x_ring, int64_t n,
                                const int64_t* m_ring, int32_t k, double* const* v_ring,
                                int32_t threads, int64_t* rank_out);
XG_API int xg_basis_create(xg_ctx* ctx, const xg_layout* layout, int32_t k, int32_t digits,
                           xg_basis** out);
XG_API void xg_basis_destroy(xg_basis* basis);
XG_API int xg_basis_set_ring(xg_basis* basis, int32_t ring, const double* v);
/* The same basis built ON THE DEVICE for every ring of a series, whose
 * loaded frames are the training rows (replaces encoder_from_rows ->
 * gram_svd, encoder.cpp:13-28 / linalg.cpp:279-439, per ring; T <= 2048):
 * exact int32 Gram (K2) -> S = G/(|x_i||x_j|) -> parallel-order Jacobi ->
 * W = Xn^T U (f64 GEMM) -> measured sigma, rank at 1e-12 sigma_max ->
 * 2x Cholesky-QR (the k x k factor on the host) -> sign convention.
 * k = 0: full numerical rank per ring (build_offline).  Outputs (each
 * optional): v_out[ring] = m_ring x k_ring f64 in mask order (k_ring = k, or
 * the ring's rank when k = 0); sigma_out[ring * sigma_ld + j] the spectrum;
 * rank_out[ring] (required); basis (k > 0) gets every ring (set_ring).
 * XG_ERR_RANK: k exceeds a ring's rank (payload = rank, ring);
 * XG_ERR_NORMALIZATION: a zero training frame (payload = frame, ring). */
XG_API int xg_series_build_basis(xg_series* s, int32_t k, double* const* v_out, double* sigma_out,
                                 int64_t sigma_ld, int64_t* rank_out, xg_basis* basis);
XG_API int xg_compress(xg_series* s, const xg_basis* basis, uint32_t flags);
/* Append n frames (u8 raster) to a chunked series and compress them:
 * series rows [t, t + n) get norms, coefficients and bf16 planes; the frames
 * themselves are not kept.  XG_CHUNK_FIRST starts a new series. */
XG_API int xg_series_compress_chunk(xg_series* s, const xg_basis* basis, const uint8_t* frames,
                                    int64_t n_frames, int frames_on_device, uint32_t flags);
XG_API int xg_ttc_compressed(xg_series* s, uint32_t flags);
/* coefficients (n x k, f64) and norms (n) of one ring */
XG_API int xg_series_get_coeffs(xg_series* s, int32_t ring, double* y, double* norms);
XG_API int xg_series_get_cttc(xg_series* s, int32_t ring, int32_t dtype, void* out, int64_t ld,
                              int out_on_device);
XG_API int xg_series_get_cg2(xg_series* s, int32_t ring, double* values, int64_t* counts);

/* ---- streaming (kHz) mode ---------------------------------------------
 * Frames arrive one at a time; each push correlates the new frame against
 * every previous frame of every ring: the exact raw column G(s,t) (u8 dp4a)
 * and, with a basis, the projected coefficients y_t (compress_frame,
 * compress.cpp:34-46; bitwise equal to the batch xg_compress rows) and the
 * compressed column y_s . y_t (ttc_extend, correlate.cpp:37-65).  g2 sums
 * are accumulated per lag as frames arrive.  Single writer. */
#define XG_STREAM_STORE_TTC 0x1u  /* keep every column (Q x T x T) for readback */
#define XG_STREAM_NO_RAW 0x2u     /* compressed only */
#define XG_STREAM_SPARSE 0x4u     /* raw columns from the new frame's nonzeros (pixel-major
                                     history): nnz*t bytes per frame instead of M*t */
XG_API int xg_stream_create(xg_ctx* ctx, const xg_layout* layout, const xg_basis* basis,
                            int64_t max_frames, uint32_t flags, xg_stream** out);
XG_API void xg_stream_destroy(xg_stream* s);
XG_API int xg_stream_push(xg_stream* s, const uint8_t* frame, int on_device);
/* n consecutive frames (n x full_pixels, raster order) pushed in one call. */
XG_API int xg_stream_push_batch(xg_stream* s, const uint8_t* frames, int64_t n, int on_device);
XG_API int64_t xg_stream_frames(const xg_stream* s);
/* which: 0 raw, 1 compressed */
XG_API int xg_stream_get_g2(xg_stream* s, int32_t ring, int32_t which, double* values,
                            int64_t* counts);
XG_API int xg_stream_get_coeffs(xg_stream* s, int32_t ring, double* y, double* norms);
XG_API int xg_stream_get_ttc(xg_stream* s, int32_t ring, int32_t which, int32_t dtype, void* out,
                             int64_t ld);

/* ---- reference-facing f64 entries (one per xpcs:: function) -----------
 * Same arguments as the reference (row-major f64 host buffers, N frames x M
 * pixels / K coefficients), same validation and errors, and the reference's
 * exact floating-point operation order executed on the current CUDA device
 * (no FMA contraction), so the outputs are the reference's bits:
 *   xg_f64_ttc_raw          <- xpcs::ttc_raw          correlate.cpp:19-25
 *   xg_f64_ttc_compressed   <- xpcs::ttc_compressed   correlate.cpp:27-35
 *   xg_f64_ttc_extend       <- xpcs::ttc_extend       correlate.cpp:37-65
 *   xg_f64_g2_from_ttc      <- xpcs::g2_from_ttc      correlate.cpp:67-85
 *   xg_f64_ttc_rel_error    <- xpcs::ttc_rel_error    correlate.cpp:87-108
 *   xg_f64_compress_series  <- xpcs::compress_series  compress.cpp:48-81
 *   xg_f64_compress_frame   <- xpcs::compress_frame   compress.cpp:34-46
 * Errors: xg_f64_last_error() / xg_f64_last_payload() (thread-local). */
XG_API const char* xg_f64_last_error(void);
XG_API int64_t xg_f64_last_payload(void);
XG_API int xg_f64_ttc_raw(const double* x, int64_t n, int64_t m, double* out);
XG_API int xg_f64_ttc_compressed(const double* y, int64_t n, int64_t k, double* out,
                                 int* lossless);
XG_API int xg_f64_ttc_extend(const double* g, int64_t n, const double* y, int64_t k,
                             const double* row, double* out, int* lossless);
XG_API int xg_f64_g2_from_ttc(const double* g, int64_t n, double period, double* lags,
                              double* values, int64_t* counts);
XG_API int xg_f64_compress_series(const double* x, int64_t n, int64_t m, const double* v,
                                  int64_t k, double* coeffs, double* norms);
/* The same over integer photon counts packed to u8 by the caller (1 B per
 * pixel over PCIe, widened to f64 on the device): results bitwise those of
 * xg_f64_compress_series on the same values. */
XG_API int xg_f64_compress_series_u8(const uint8_t* x, int64_t n, int64_t m, const double* v,
                                     int64_t k, double* coeffs, double* norms);
XG_API int xg_f64_compress_frame(const double* frame, int64_t m, const double* v, int64_t k,
                                 double* coeffs, double* norm);
XG_API int xg_f64_ttc_rel_error(const double* a, const double* b, int64_t count, double* out);

/* ---- synthetic source (benchmark input; not on the correlation path) ---
 * Seeded speckle counts: complex AR(1) field per pixel with
 * rho = exp(-Gamma) (gamma_mode 0: Gamma = a r^2, 1: a 10^(3q/(Q-1))), Poisson
 * counts of mean mu |f|^2 clipped to 255, CounterRng (rng.cpp:12-44)
 * substreams 1/2/3.  Writes n_frames x (height*width) u8 to device memory. */
XG_API int xg_synth_speckle(xg_ctx* ctx, int64_t n_frames, int64_t height, int64_t width,
                            int32_t n_rings, double mu, int32_t gamma_mode, double gamma_a,
                            uint64_t seed, uint8_t* out_device);

#ifdef __cplusplus
}
#endif

#endif /* XPCS_B200_H_ */
