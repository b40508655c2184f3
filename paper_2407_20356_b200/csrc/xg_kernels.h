// xg_kernels.h -- device-kernel launch interface shared by the host runtime
// (xg_api.cu) and the kernel translation units.  Internal; not installed.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace xg {

// Stored TTC (int32 Gram / f32 C~) of a series, one slab per ring: the upper
// 256 x 256 pair tiles (I <= J) packed in (I, J) row-major tile order, each
// tile row-major -- half the memory of a full T x T square, and the same
// bytes as the split-ring exchange format.  nb = tiles per row (ceil(T/256)).
// nb <= 0 selects a plain row-major square with leading dimension ld (the
// streaming columns).  Requires a <= b (every reader takes the upper triangle).
#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t ttc_off(int64_t a, int64_t b, int64_t ld, int32_t nb) {
  if (nb <= 0) return a * ld + b;
  const int64_t I = a >> 8, J = b >> 8;
  return ((I * nb - (I * (I - 1)) / 2 + (J - I)) << 16) + ((a & 255) << 8) + (b & 255);
}
inline int64_t ttc_slab(int64_t nb) { return nb * (nb + 1) / 2 * 65536; }


// ---------------------------------------------------------------- K1 ingest
// A detector band (8192 pixels) is staged in shared memory as 512-byte pieces
// at a 528-byte pitch (+16 zero bytes that padding entries point to).
constexpr int INGEST_PIECE = 512;
constexpr int INGEST_PITCH = 528;
#ifndef XG_INGEST_CONSUMERS
#define XG_INGEST_CONSUMERS 8
#endif
constexpr int INGEST_CONSUMERS = XG_INGEST_CONSUMERS;  // consumer warps per K1 CTA
__host__ __device__ constexpr int ingest_band_stride(int band) {
  return ((band + INGEST_PIECE - 1) / INGEST_PIECE) * INGEST_PITCH + 16;
}
__host__ __device__ constexpr int ingest_smem_offset(int e) {  // band byte -> smem byte
  return e + (INGEST_PITCH - INGEST_PIECE) * (e / INGEST_PIECE);
}
// 2D bands (xg_layout_create_2d on a detector wider than a piece): kBandH
// rows x kBandW columns, one piece per row.
constexpr int kBandW = INGEST_PIECE;
constexpr int kBandH = 16384 / INGEST_PIECE;


// The pixels of one ring inside one band form a "segment" of the ring-major
// row: first every source word whose 4 pixels all belong to the ring (copied
// as a word), then the remaining pixels packed 4 per group (gathered byte by
// byte, zero padded).  A "piece" is the part of a segment one consumer warp
// handles; pieces are balanced across the band's 8 consumer warps.
struct Piece {
  int32_t ring;
  int32_t dst;       // first output byte column (multiple of 4)
  int32_t n_word;    // whole-word groups
  int32_t word_off;  // into the band's word table (u16 smem word index each)
  int32_t n_byte;    // byte-gathered groups (after the word groups)
  int32_t byte_off;  // into the band's byte table (4 u16 smem byte offsets each)
  int32_t koff;      // the ring's first ring-major column (ring-blocked x, below)
  int32_t kpad;      // the ring's padded width (its row stride in x)
};

// Ring-major frames x: on a layout with long rows ring-BLOCKED -- ring q owns
// x + xmax koff_q .. + xmax (koff_q + kpad_q), a [xmax frames][kpad_q] matrix
// -- so a TMA box of 128 frames spans 128 kpad_q bytes instead of 128 ktot
// (C5: 3 MB instead of 400 MB of address space: K3 at C5 geometry ran at
// half its per-byte speed with the interleaved rows); else interleaved
// [frame][ktot] rows.  Pieces carry the addressing (Piece::koff / kpad).
struct IngestParams {
  const uint8_t* raster;     // n_frames x pixels (device)
  uint8_t* x;                // ring-blocked (above), xmax frames per ring block
  int64_t pixels;
  int64_t ktot;
  int32_t band;              // pixels per band
  int32_t n_bands;
  int32_t n_rings;
  const int32_t* band_piece; // [n_bands][9]: piece range of each consumer warp
  const Piece* pieces;
  const int32_t* band_word;  // n_bands + 1 ranges of `words`
  const uint16_t* words;
  const int32_t* band_byte;  // n_bands + 1 ranges of `bytes` (in groups)
  const uint16_t* bytes;     // 4 per group
  int32_t max_words;         // largest band word table
  int32_t max_bytes;         // largest band byte table (groups)
  int32_t max_band_pieces;
  int64_t t0;                // first frame index written (statistics row)
  int64_t x_row0;            // frame index of row 0 of x (chunked series; else 0)
  int64_t n_frames;
  int32_t frames_per_cta;
  unsigned long long* norm2;  // [frame][ring] |x|^2, accumulated per piece (rows pre-zeroed)
  int64_t xmax;               // frames per ring block of x
  int32_t blocked;            // x ring-blocked (else interleaved [frame][ktot] rows)
  int32_t width = 0;          // > 0: 2D bands of kBandH x kBandW over a height x width
  int32_t height = 0;         //      detector; band b = block (b / blocks_x, b % blocks_x)
  int32_t blocks_x = 0;
};
cudaError_t launch_ingest(const IngestParams& p, cudaStream_t s);

// K1e: photon-event frames (CSR by frame) scattered into cleared ring-major
// rows; |x|^2 per (frame, ring) summed in shared memory, one row per CTA.
struct EventIngestParams {
  const int64_t* frame_off;  // [t0 + n_frames + 1] (event indices into pix / val)
  int64_t t0;                // first frame of this launch
  const int32_t* pix;        // raster pixel index per event
  const uint8_t* val;        // count per event
  int64_t n_frames;
  int64_t pixels;
  const int32_t* pixcol;     // [pixels] ring << 22 | column (-1: no ring)
  const int32_t* ring_koff;
  const int32_t* ring_nkb;
  int32_t n_rings;
  uint8_t* x;
  int64_t xmax, ktot;
  int32_t blocked;
  unsigned long long* norm2; // [frame][ring], written (not accumulated)
  int* err;                  // bit 3: pixel index out of range
};
cudaError_t launch_ingest_events(const EventIngestParams& p, cudaStream_t s);

// --------------------------------------------------------- per-ring norms
// norms[r][t] = sqrt(norm2[t][r]), inv = 1/norms (0 for zero frames);
// counts zero frames per ring and flags int32-Gram overflow (norm2 >= 2^31).
struct NormParams {
  int64_t t0;                // first frame processed (streaming: the new frame)
  const int64_t* norm2;      // [frame][ring] |x|^2 (exact, from K1)
  int64_t n_frames;
  int64_t ld;                // frame stride of norms/inv (>= n_frames)
  int32_t n_rings;
  double* norms;             // [ring][ld]
  double* inv;               // [ring][ld]
  float2* inv2;              // [ring][ld] (hi, lo) float split of inv (or null)
  int64_t* zero_count;       // [ring]
  int64_t* first_zero;       // [ring] smallest zero-norm frame (sentinel if none)
  uint32_t* nz_bits;         // [ring][nz_words] nonzero-frame bitmask (pre-zeroed)
  int32_t nz_words;
  unsigned long long* max_norm2;  // running max of |x|^2 (or null)
  int* err;                  // bit 2: overflow (null: not checked here)
  int32_t ring0 = 0;         // first ring processed (split-ring import: one ring)
  int32_t ring_count = -1;   // rings processed (-1: all n_rings)
};
cudaError_t launch_norms(const NormParams& p, cudaStream_t s);

// ------------------------------------------------------------ K2 raw Gram
struct TileDesc {
  int32_t ring;
  int32_t i0;
  int32_t j0;
  int32_t pad;
};
struct GramParams {
  const TileDesc* tiles;
  int32_t ntiles;
  const int32_t* ring_koff;  // byte column of each ring in the ring-major row
  const int32_t* ring_nkb;   // 128-byte K blocks per ring
  const CUtensorMap* xmaps;  // raw mode: per-ring TMA maps of the ring blocks of x (global)
  uint32_t* gram;            // [ring][ld][ld] exact int32 Gram / f32 C~ (upper tiles)
  int64_t ring_stride;
  int32_t ld;
  int32_t nb = 0;            // packed-tile row length ceil(T/256) of the stored TTC
  int* err;                  // bit 0: pipeline timeout
  // fused g2 (null g2_partial = off): per tile, the sums over each tile
  // diagonal (j - i + 127 in [0, 383)) of C(i,j) = G_ij inv_i inv_j, j >= i
  const double* inv;         // [ring][inv_ld]
  const float2* inv2;        // [ring][inv_ld] (hi, lo) float split of inv
  int64_t inv_ld;
  int64_t n_frames;
  float2* g2_partial;        // [ntiles][384] (hi, lo) double-float diagonal sums
  int32_t store;             // 0: g2 only, the TTC tiles are not written
  // compressed mode (launch_gram2_cmp): K blocks run over precision pairs
  // (plane_a, plane_b) packed 4 bits each in `pairs`, kb_per_plane 64-element
  // blocks per plane; plane rows of ring r, plane s start at (3r+s)*plane_rows
  int32_t n_pairs;
  int32_t pairs;
  int32_t kb_per_plane;
  int32_t plane_rows;
  // pair kernel (k_gram2): 256 x 256 tiles, pad = 1-CTA half-tile index of
  // the upper half; 128-row / 256-col block counts of the 1-CTA enumeration
  int32_t g2_nbi, g2_nbj;
  // max |x_t|^2 over the series (K1b): G_ij <= it, so < 2^23 lets the fused g2
  // run in FP32 double-float arithmetic with exact float Gram values
  const unsigned long long* max_norm2;
  // wave gate (K2): pair p takes tiles p, p + P, p + 2P, ... (P pairs); before
  // starting its wave w the leader waits until every pair has started wave
  // w - gate_lag (wave_ctr counts started tiles, zero at launch), so no pair
  // drifts more than gate_lag waves ahead and the tiles in flight stay inside
  // the L2-resident super-tile (null: ungated)
  unsigned int* wave_ctr = nullptr;
  int32_t gate_lag = 2;
};
size_t gram2_smem_bytes(int mode);
cudaError_t launch_gram2_u8(const CUtensorMap& tmX, const CUtensorMap& tmOut, const GramParams& p,
                            int num_sms, cudaStream_t stream);
cudaError_t launch_gram2_cmp(const CUtensorMap& tmY, const CUtensorMap& tmOut, const GramParams& p,
                             int num_sms, cudaStream_t stream);

// Fold the per-tile diagonal sums of K2 into g2[ring][d] (fixed order) and
// count the valid (t, t+d) pairs from the nonzero-frame bitmask.
struct G2FoldParams {
  const float2* g2_partial;  // [ntiles][384] (hi, lo); K4: [ntiles][384] float
  int32_t single;            // 1: fp32 partials (K4)
  double* runs;              // [ring][2 nbj][384] per-delta run sums (k_g2_runs)
  int32_t tiles_per_ring;
  int32_t nbi, nbj;
  int64_t n_frames;
  int32_t n_rings;
  const uint32_t* nz_bits;   // [ring][nz_words] bit t = frame t has nonzero norm
  int32_t nz_words;
  const int64_t* zero_count; // [ring] zero-norm frames (0: every count is T - d)
  double* g2;                // [ring][g2_ld]
  int64_t* counts;
  int64_t g2_ld;
};
cudaError_t launch_g2_fold(const G2FoldParams& p, cudaStream_t s);

// ------------------------------------------------------ K3 projection
#ifdef __CUDACC__
// y = scale / |x| * (a0 + a1/254 + a2/254^2) with every rounding explicit, so
// the batch (K3) and streaming (K5) projections agree bitwise.
__device__ __forceinline__ double combine_digits(int32_t a0, int32_t a1, int32_t a2, int n_digits,
                                                 double scale, double inv) {
  double s = static_cast<double>(a0);
  if (n_digits > 1) s = __dadd_rn(s, __dmul_rn(static_cast<double>(a1), 1.0 / 254.0));
  if (n_digits > 2) s = __dadd_rn(s, __dmul_rn(static_cast<double>(a2), 1.0 / 64516.0));
  return __dmul_rn(__dmul_rn(scale, inv), s);
}
#endif

struct ProjParams {
  const TileDesc* tiles;     // (ring, i0 = first frame of x, j0 = N-tile index)
  int64_t t0;                // series frame index of x row 0 (chunked compress; else 0)
  int32_t ntiles;
  const int32_t* ring_koff;
  const int32_t* ring_nkb;
  const CUtensorMap* xmaps;  // per-ring TMA maps of the ring blocks of x (global)
  const CUtensorMap* vmaps;  // per-ring TMA maps of the ring blocks of the basis digits
  int32_t n_digits;          // S in {1, 2, 3}
  int32_t kt;                // coefficients per N-tile (multiple of 16, S*kt <= 256)
  int32_t k;                 // rank
  const double* inv;         // [ring][inv_ld] 1/|x_t|
  int64_t inv_ld;
  int64_t n_frames;
  const double* scale;       // [ring][k] digit scale of each basis column
  double* y;                 // [ring][y_ld][k] coefficients (f64)
  int64_t y_ld;
  __nv_bfloat16* planes;     // [(ring*3 + s) * plane_rows + t][kp] bf16 split of y (or null)
  int64_t plane_rows;
  int32_t kp;                // plane row length (multiple of 64)
  int* err;
};
size_t project_smem_bytes(int nt_rows);
cudaError_t launch_project(const CUtensorMap& tmX, const CUtensorMap& tmV, const CUtensorMap& tmP,
                           const ProjParams& p, int num_sms, cudaStream_t stream);

// ------------------------------------------------------ K5/K6 streaming
struct StreamParams {
  const uint8_t* x;          // ring-major history [t][ktot]
  int64_t ktot;
  int64_t t;                 // index of the new frame
  const int32_t* ring_koff;
  const int32_t* ring_nkb;
  const double* inv;         // [ring][inv_ld]
  int64_t inv_ld;
  double* g2sum;             // [ring][g2_ld] running sums over lag (raw)
  int64_t* g2cnt;
  double* cg2sum;            // compressed
  int64_t* cg2cnt;
  int64_t g2_ld;
  int32_t* gcol;             // optional: exact Gram G(s,t) at [ring][s][t]
  float* ccol;               // optional: C~(s,t)
  int64_t col_ring_stride, col_ld;
  // compressed
  const int8_t* vdt;         // pixel-major basis digits [ktot][vdt_ld], index s*k + j
  int32_t vdt_ld;
  int32_t n_digits;
  int32_t k;
  const double* scale;       // [ring][k]
  double* y;                 // [ring][y_ld][k]
  float* yf;                 // [ring][y_ld][kq] fp32 copy: the compressed column's history
  int32_t kq;                // k rounded up to 4 (zero pad)
  int64_t y_ld;
  // sparse raw mode: pixel-major history hist[c][hp] (u8, column c of the
  // ring-major layout, frame s) and the new frame's nonzeros per ring
  uint8_t* hist;
  int64_t hp;                // frames per pixel row (multiple of 16)
  int32_t* nz_col;           // [ktot]: ring r's nonzero columns at [koff_r, ...)
  uint8_t* nz_val;           // [ktot]
  int32_t* nz_n;             // [ring] counts of this push (zero on entry)
  int32_t* nz_next;          // [ring] counts of the next push: zeroed by the ingest
  int32_t* pacc;             // [ring][768] projection digit sums (zero on entry)
  // one-frame ingest
  const uint8_t* frame;      // raster of the new frame
  const int32_t* colpix;     // [ktot] detector pixel of each column (-1 = padding)
  const int32_t* blk_ring;   // [ktot / 128] ring of each 128-column block
  const int32_t* pixcol;     // [pixels] ring << 22 | ring-major column (-1: no ring)
  int64_t pixels;
  int32_t n_rings;
  unsigned long long* norm2; // [frame][ring] (row t zero on entry)
  unsigned long long* norm2_next;  // row t + 1, zeroed by the ingest (or null)
  // sparse ingest: its last CTA finishes frame t's norms (k_norms' work)
  double* norms_w;           // [ring][inv_ld]
  double* inv_w;             // [ring][inv_ld]
  int64_t* zero_count;       // [ring]
  int64_t* first_zero;       // [ring]
  uint32_t* nz_bits;         // [ring][nz_words]
  int32_t nz_words;
  int* err;
  int32_t ovf_check;         // raw columns formed: |x|^2 >= 2^31 sets err bit 2
  int32_t pdl_wait_end;      // K5s in a compressed PDL chain: wait at the end (k_stream.cu)
  int32_t pdl_wait_fin;      // K5s after K5s in a batch: wait before the finishing step
  unsigned int* done;        // CTA counter (zero on entry, reset by the last CTA)
  // batched sparse ingest (grid.y = frames t .. t + gridDim.y - 1): frame f
  // at frame + f * pixels, its nonzero lists at nz_col/nz_val + f * nz_bstride
  // and counts at nz_n + f * n_rings (zeroed before the launch)
  int64_t nz_bstride;
  // batched columns (push_batch, grid.z = frames t .. t + nb - 1): the column
  // kernels write their entries to per-frame scratch columns
  // [ring][scr_nb][scr_ld] (raw: int32 Gram, compressed: fp32 C~) and
  // k_stream_fold adds them to the lag sums in ascending frame order.
  int32_t* gscr;
  float* cscr;
  int64_t scr_ld;
  int32_t scr_nb;            // frames of the batch
  int64_t pacc_bstride;      // proj_acc/proj_fin: frame f's digit sums at pacc + f * pacc_bstride
  // photon-event history (batched raw columns): frames [0, s_begin) are
  // sealed event segments -- per segment and pixel column an (offset, count)
  // entry into the segment's event list (s_local << 8 | count, ascending s),
  // or the segment's dense flag when its events did not fit -- and K5s
  // covers only [s_begin, t].  One launch_stream_batch call covers up to two
  // segment levels: ev_n[l] segments of ev_tb[l] frames, the first being
  // segment ev_first[l] of its level, stored in slot (index % ev_ring[l]).
  int64_t s_begin;
  const uint32_t* ev[2];
  const int2* evidx[2];
  const int32_t* ev_dense[2];
  int64_t ev_cap[2];         // events per segment
  int32_t ev_tb[2];          // frames per segment (multiple of 128)
  int32_t ev_n[2];
  int32_t ev_first[2];
  int32_t ev_ring[2];        // 0: slot = index
};

// Seal block `block` of a photon-event history (frames [block tb, + tb)):
// pixel-major events from the dense history into slot `slot` (its list at
// ev + slot cap, entries at evidx + slot ktot, cursor/dense[slot] zero on
// entry); a block whose events do not fit is flagged dense.
struct SealParams {
  const uint8_t* hist;
  int64_t hp;
  int64_t ktot;
  int32_t block;
  int32_t slot;
  int32_t tb;
  int64_t cap;
  uint32_t* ev;
  int2* evidx;
  unsigned long long* cursor;
  int32_t* dense;
};
cudaError_t launch_stream_seal(const SealParams& p, cudaStream_t s);
// Merge the nf sealed blocks in slots 0 .. nf - 1 (consecutive, ascending)
// into segment `seg` of nf * tb frames: each pixel's lists concatenated with
// the block offset added to s_local; any dense block makes the segment dense.
struct MergeParams {
  const uint32_t* ev0;
  const int2* evidx0;
  const int32_t* dense0;
  int64_t cap0;
  int32_t tb;
  int32_t nf;
  int64_t ktot;
  int32_t seg;
  int64_t cap1;
  uint32_t* ev1;
  int2* evidx1;
  unsigned long long* cursor1;  // [seg], zero on entry
  int32_t* dense1;              // [seg], zero on entry
};
cudaError_t launch_stream_merge(const MergeParams& p, cudaStream_t s);
// One-frame ingest for the streaming path: ring-major row t of the history,
// |x_t|^2 per ring, and in sparse mode the frame's nonzeros per ring plus
// their scatter into the pixel-major history.
cudaError_t launch_stream_ingest(const StreamParams& p, cudaStream_t s);
// Sparse mode: the same from the raster in pixel order (no ring-major row):
// only the frame's nonzero pixels touch the tables.
cudaError_t launch_stream_ingest_sparse(const StreamParams& p, cudaStream_t s, bool pdl,
                                        int32_t n_frames = 1);
// Sparse raw streaming (photon-event data): the new column costs nnz * t
// bytes instead of M * t; results equal the dense kernel's bitwise.
cudaError_t launch_stream_sparse(const StreamParams& p, int32_t n_rings, cudaStream_t s, bool pdl);
cudaError_t launch_stream_raw(const StreamParams& p, int32_t n_rings, int64_t max_kpad,
                              cudaStream_t s);
cudaError_t launch_stream_cmp(const StreamParams& p, int32_t n_rings, cudaStream_t s, bool pdl);
// Batched columns of frames t .. t + nb - 1 (p.scr_nb = nb, ingested): the
// photon-event raw columns (K5s, grid.z = frame), the projections (K6a, one
// launch each for the batch) and the compressed columns (K6c: every history
// row loaded once for all nb new rows), each to its scratch columns, then
// the in-order lag-sum fold.  Results equal nb single pushes bitwise.
cudaError_t launch_stream_batch(const StreamParams& p, int32_t n_rings, bool raw, bool cmp,
                                cudaStream_t s);
cudaError_t launch_g2_div(const double* sum, const int64_t* cnt, double* out, int64_t n,
                          cudaStream_t s);

// ------------------------------------------- K9 reference-order f64 replicas
cudaError_t launch_exact_widen_u8(const uint8_t* x, int64_t count, double* out, cudaStream_t s);
cudaError_t launch_exact_rownorm(const double* x, int64_t n, int64_t m, double* xn, double* norms,
                                 unsigned long long* bad, cudaStream_t s);
cudaError_t launch_exact_gram(const double* x, int64_t n, int64_t m, double* g, cudaStream_t s);
cudaError_t launch_exact_extend(const double* g, int64_t n, const double* y, int64_t k,
                                const double* row, double* out, cudaStream_t s);
cudaError_t launch_exact_g2(const double* g, int64_t n, double period, double* lags,
                            double* values, int64_t* counts, cudaStream_t s);
cudaError_t launch_exact_project(const double* xn, int64_t n, int64_t m, const double* v,
                                 int64_t k, double* coeffs, cudaStream_t s);
cudaError_t launch_exact_relerr(const double* a, const double* b, int64_t count, double* out,
                                cudaStream_t s);

// --------------------------------------------------------------- K7 g2
// g2[r][d] = sum_{t} G(t,t+d) inv_t inv_{t+d} / count, ascending t within
// segments of `seg` frames, segments combined in ascending order.
struct G2Params {
  const int32_t* gram;       // int32 Gram source (mode 0) ...
  const float* cf32;         // ... or an already normalised f32 C (mode 1)
  int64_t ring_stride;
  int32_t ld;
  int32_t nb = 0;            // > 0: packed upper pair tiles (ttc_off), else ld-square
  const double* inv;         // [ring][inv_ld] (mode 0)
  int64_t inv_ld;
  int64_t n_frames;
  int32_t n_rings;
  int32_t seg;
  int32_t n_seg;
  double* partial;           // [ring][n_seg][n_frames]
  int64_t* pcount;           // [ring][n_seg][n_frames]
  double* g2;                // [ring][g2_ld]
  int64_t* counts;           // [ring][g2_ld]
  int64_t g2_ld;
};
cudaError_t launch_g2(const G2Params& p, int mode, cudaStream_t s);


// ---------------------------------------------------- TTC readback expand
struct ExpandParams {
  const int32_t* gram;       // mode int: exact Gram, normalised with inv
  const float* cf32;         // mode f32 source (already normalised)
  int64_t ring_stride;
  int32_t ld;
  int32_t nb = 0;            // > 0: packed upper pair tiles (ttc_off), else ld-square
  const double* inv;         // [n] for this ring
  int64_t n;
  void* out;
  int64_t out_ld;
  int32_t out_dtype;         // 0 f64, 1 f32, 2 i32 (raw Gram)
};
cudaError_t launch_expand(const ExpandParams& p, int src_mode, cudaStream_t s);
// rows [row0, row0 + rows) of the upper triangle, packed (row i: columns i..n-1)
cudaError_t launch_pack_upper(const ExpandParams& p, int src_mode, int64_t row0, int64_t rows,
                              cudaStream_t s);

// ttc_rel_error (correlate.cpp:87-108) of every ring between the stored raw
// TTC (exact Gram * 1/|x_i| 1/|x_j|) and the stored compressed C~, over the
// full symmetric matrices; fixed-order reductions (deterministic).
struct RelErrParams {
  const int32_t* gram;       // [ring][ld][ld] upper tiles
  const float* cgram;        // [ring][ld][ld] upper tiles
  int64_t ring_stride;
  int32_t ld;
  int32_t nb = 0;            // > 0: packed upper pair tiles (ttc_off), else ld-square
  const double* inv;         // [ring][inv_ld]
  int64_t inv_ld;
  int64_t n;
  int32_t n_rings;
  double2* partial;          // [ring][REL_BLOCKS] (num, den)
  double* out;               // [ring]
};
constexpr int REL_BLOCKS = 64;
cudaError_t launch_rel_error(const RelErrParams& p, cudaStream_t s);

// ---------------------------------------------------------- analysis (8(f) 4)
// ttc_background (analysis.cpp:202-235) of every ring's stored TTC: two
// deterministic passes (mean, then squared deviations) over the upper tiles.
struct BgParams {
  const int32_t* gram;       // raw: exact Gram [ring][ld][ld] (cgram == null)
  const float* cgram;        // compressed C~ (or null)
  int64_t ring_stride;
  int32_t ld;
  int32_t nb = 0;            // > 0: packed upper pair tiles (ttc_off), else ld-square
  const double* inv;         // [ring][inv_ld]
  int64_t inv_ld;
  int64_t n;
  int64_t excl;              // exclusion band (lags <= excl left out)
  int32_t n_rings;
  double2* partial;          // [ring][BG_BLOCKS] (sum, count)
  double* mean;              // [ring]
  int64_t* count;            // [ring] entries outside the band (upper triangle)
  double* out;               // [ring] sigma (-1: none)
};
constexpr int BG_BLOCKS = 64;
cudaError_t launch_ttc_background(const BgParams& p, cudaStream_t s);

// fit_kww (analysis.cpp:77-172) of every ring's g2 curve, one warp per ring.
struct KwwParams {
  const double* g2;          // [ring][g2_ld]
  int64_t g2_ld;
  int64_t n;                 // curve points (lags d * period, d < n)
  double period, min_lag, max_lag;
  int32_t n_rings;
  double* out;               // [ring][4] B, C, t0, residual rms
  int32_t* status;           // [ring] 0 ok, 1 FitDegenerate, 2 FitError, 3 Contract
};
cudaError_t launch_fit_kww(const KwwParams& p, cudaStream_t s);

// ---------------------------------------------------------- spectral g2 (compressed, g2 only)
// g2 of C~ = Y Y^T from the coefficient series' autocorrelations by FFT
// (k_spectral.cu): no T x T tile is formed.
constexpr int SPEC_B = 4096;  // frames per time block
constexpr int SPEC_L = 8192;  // FFT length (2 B: linear correlation)
struct SpecParams {
  const double* y;           // [ring][y_ld][k] coefficients (f64)
  int64_t y_ld;
  int32_t k;
  int64_t n;
  int32_t n_rings;
  const uint32_t* nz_bits;   // [ring][nz_words]
  int32_t nz_words;
  const int64_t* zero_count; // [ring]
  double* g2;                // [ring][g2_ld]
  int64_t* counts;
  int64_t g2_ld;
  // set by the launcher inside the scratch buffer
  int32_t nb, nm, npairs;
  const double2* tw;
  double2* spec;
  double* corr;
};
size_t spectral_scratch_bytes(int n_rings, int64_t n, int k);
cudaError_t launch_spectral_g2(SpecParams p, void* scratch, cudaStream_t s);

// ---------------------------------------------------------- K8 synthetic
struct SynthParams {
  int64_t t_first;           // global index of the first frame generated
  int64_t t_frames;          // frames in this chunk
  int64_t h, w;
  int32_t q;
  int32_t gamma_mode;        // 0: Gamma = a r^2 ; 1: Gamma = a 10^(3q/(Q-1))
  double gamma_a;
  double mu;
  uint64_t s_re, s_im, s_po; // CounterRng substreams 1, 2, 3 of the seed
  double* carry_re;          // per-pixel field carried across chunks (or null)
  double* carry_im;
  uint8_t* out;              // t_frames x out_ld
  int64_t out_ld;
};
cudaError_t launch_synth(const SynthParams& p, cudaStream_t s);

// ---------------------------------------------------------- K9 basis (gram_svd on the device)
// Gram-trick SVD of every ring's training frames (linalg.cpp:279-439):
// S = G_q / (|x_i||x_j|) from the exact int32 Gram, parallel-order Jacobi on
// S, W = Xn^T U (f64 GEMM over the ring-major u8 frames), column norms,
// Cholesky-QR x2 (the host factors the k x k Gram), K9.
// Circle-method pairing of step s over np indices (np even, R = np - 1 fixed
// point).  Pair 0 = (R, s); pair k >= 1 = (s + k, s - k) mod R.  Within a pair
// the smaller original index takes the even slot (p < q, as the reference).
__host__ __device__ inline int slot_index(int slot, int s, int np) {
  const int R = np - 1, k = slot >> 1;
  int x, y;
  if (k == 0) {
    x = R;
    y = s;
  } else {
    x = (s + k) % R;
    y = (s - k + R) % R;
  }
  const int lo = (x < y ? x : y), hi = (x < y ? y : x);
  return (slot & 1) ? hi : lo;
}

__host__ __device__ inline int index_slot(int i, int s, int np) {
  const int R = np - 1, half = np >> 1;
  int k, partner;
  if (i == R) {
    k = 0;
    partner = s;
  } else {
    const int d = (i - s + R) % R;
    if (d == 0) {
      k = 0;
      partner = R;
    } else if (d <= half - 1) {
      k = d;
      partner = (s - d + R) % R;
    } else {
      k = R - d;
      partner = (s + k) % R;
    }
  }
  return 2 * k + (i > partner ? 1 : 0);
}

struct JacState {
  double tol;                // reference threshold, x100 per 10 sweeps after 40
  int32_t active;            // 0 once a whole sweep rotated nothing
  int32_t rotated;           // set by the step kernels of the current sweep
};
struct JacParams {
  const double* a_in;        // [ring][np][np] slot layout of this step
  double* a_out;             // [ring][np][np] slot layout of the next step
  const double* v_in;        // [ring][np][np] rows: coordinates, cols: slots
  double* v_out;
  JacState* state;           // [ring]
  int32_t np;                // padded (even) order
  int32_t step;              // 0 .. np-2 within the sweep
};
cudaError_t launch_jacobi_step(const JacParams& p, int n_rings, cudaStream_t s);

struct BasisSParams {
  const int32_t* gram;       // stored Gram, ring slabs of ring_stride elements (ttc_off)
  int32_t ld;
  const double* inv;         // [ring][inv_ld]
  int64_t inv_ld;
  int32_t n, np;
  double* a;                 // [ring][np][np] slot layout of step 0
  double* v;                 // [ring][np][np] identity in slot layout
  int32_t nb;                // packed-tile row length (ttc_off)
  int64_t ring_stride;       // elements per ring slab
  const double* s64;         // non-null: S given in f64, [ring][n][n] (gram/inv unused)
};
cudaError_t launch_basis_s(const BasisSParams& p, int n_rings, cudaStream_t s);
// diag of the converged A (slot layout of step 0) -> eig [ring][np]
cudaError_t launch_jacobi_diag(const double* const* a_ring, double* eig, int np, int n_rings,
                               cudaStream_t s);

// One ring's operands of the f64 GEMMs: C[M x N] = A[M x K] * B[K x N]
// (B u8 or f64, row-major), or the Gram C[M x M] = A A^T split over K.
struct DGemmRing {
  const double* a;  int64_t lda;
  const void* b;    int64_t ldb;
  double* c;        int64_t ldc;
  int32_t m, n, k;
};
cudaError_t launch_dgemm_nn(const DGemmRing* d_rings, int n_rings, int max_m, int max_n,
                            bool b_u8, cudaStream_t s);
constexpr int SYRK_CHUNK = 2048;
// partial [ring][chunk][m][m] (ring stride part_stride), then a fixed-order sum
cudaError_t launch_dsyrk(const DGemmRing* d_rings, int n_rings, int max_m, int max_chunks,
                         double* partial, int64_t part_stride, cudaStream_t s);
cudaError_t launch_dsyrk_sum(const DGemmRing* d_rings, int n_rings, int max_m, int max_chunks,
                             const double* partial, int64_t part_stride, cudaStream_t s);
// row norms^2 of C rows [0, m) over n columns (fixed-order tree)
cudaError_t launch_row_norm2(const DGemmRing* d_rings, int n_rings, int max_m, double* out,
                             int64_t out_ld, cudaStream_t s);
// dst row j = src row idx[j] * scale[j]  (idx/scale [ring][ld_idx])
cudaError_t launch_gather_rows(const DGemmRing* d_rings, const int32_t* idx, const double* scale,
                               int64_t ld_idx, int n_rings, int max_m, int max_n, cudaStream_t s);

}  // namespace xg
