// k_stream.cu -- K5/K6: streaming incremental update, one frame at a time.
//
// The reference's streaming step is ttc_extend (src/correlate.cpp:37-65) on
// compressed rows after compress_frame (src/compress.cpp:34-46): an O(n^2)
// copy plus n dots per frame.  Here the history stays resident in HBM and
// each new frame t only produces its column, for every q-ring at once:
//
//   K5 raw:   G(s,t) = sum_p x_s[p] x_t[p] for s <= t over the ring-major
//             u8 history (exact, dp4a int32), C = G inv_s inv_t, and
//             g2sum[d = t-s] += C -- lags accumulate in ascending t exactly
//             like g2_from_ttc's sequential sum (correlate.cpp:67-85).
//             HBM-bound: t * M bytes per frame, 128-bit coalesced loads.
//   K5s sparse raw (XG_STREAM_SPARSE): the same column from the new frame's
//             nonzeros over a pixel-major history: nnz * t bytes per frame.
//   K6a proj: y_t = (x_t/|x_t|) V from the NONZERO pixels of the new frame
//             only (the reference's project_row skips zeros too,
//             compress.cpp:17) against a pixel-major copy of the int8 basis
//             digits; the f64 combination is the same expression as the
//             batch projection (k_project.cu), so streamed coefficients equal
//             batch coefficients bitwise.
//   K6b cmp:  C~(s,t) = y_s . y_t over an fp32 copy of the coefficient
//             history (C~ is fp32-accurate by contract), g2 accumulated like
//             K5 in f64.  HBM-bound: t * Q * k * 4 B.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

constexpr int SR_THREADS = 256;
constexpr int SR_ROWS = 64;  // history rows per CTA (8 per warp)

__device__ __forceinline__ unsigned dp16(uint4 a, uint4 b, unsigned acc) {
  acc = __dp4a(a.x, b.x, acc);
  acc = __dp4a(a.y, b.y, acc);
  acc = __dp4a(a.z, b.z, acc);
  return __dp4a(a.w, b.w, acc);
}

// K5: grid (ceil((t+1)/SR_ROWS), rings).  dp4a on u8 operands: the u32 words
// are treated as unsigned bytes by __dp4a(unsigned, unsigned, unsigned).
__global__ void __launch_bounds__(SR_THREADS) k_stream_raw(StreamParams p) {
  extern __shared__ uint4 xt[];  // the new frame's ring columns
  const int r = blockIdx.y;
  const int64_t koff = p.ring_koff[r];
  const int nvec = p.ring_nkb[r] * 8;  // 16-byte vectors of the padded ring
  const uint4* src = reinterpret_cast<const uint4*>(p.x + p.t * p.ktot + koff);
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) xt[i] = src[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double inv_t = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  const int64_t s_begin = static_cast<int64_t>(blockIdx.x) * SR_ROWS;
  for (int64_t s = s_begin + warp; s < s_begin + SR_ROWS && s <= p.t; s += SR_THREADS / 32) {
    const uint4* row = reinterpret_cast<const uint4*>(p.x + s * p.ktot + koff);
    unsigned acc = 0;
    int i = lane;
    for (; i + 96 < nvec; i += 128) {  // 4 independent 16-byte loads in flight
      const uint4 a0 = __ldcs(row + i), a1 = __ldcs(row + i + 32);
      const uint4 a2 = __ldcs(row + i + 64), a3 = __ldcs(row + i + 96);
      acc = dp16(a0, xt[i], acc);
      acc = dp16(a1, xt[i + 32], acc);
      acc = dp16(a2, xt[i + 64], acc);
      acc = dp16(a3, xt[i + 96], acc);
    }
    for (; i < nvec; i += 32) acc = dp16(__ldcs(row + i), xt[i], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const double inv_s = p.inv[static_cast<int64_t>(r) * p.inv_ld + s];
      const int64_t d = p.t - s;
      const int64_t gi = static_cast<int64_t>(r) * p.g2_ld + d;
      p.g2sum[gi] += static_cast<double>(static_cast<int>(acc)) * (inv_s * inv_t);
      p.g2cnt[gi] += (inv_s != 0.0 && inv_t != 0.0) ? 1 : 0;
      if (p.gcol) p.gcol[static_cast<int64_t>(r) * p.col_ring_stride + s * p.col_ld + p.t] =
          static_cast<int>(acc);
    }
  }
}

// K6a: grid (rings, PZ).  A CTA takes a slice of the ring's nonzero pixels
// (compacted by the one-frame ingest -- the reference's project_row skips
// zeros too, compress.cpp:17) and accumulates x * digit for every (digit,
// coefficient) pair from the pixel-major int8 digits; slices meet in pacc
// (integer atomics: exact, order-free).
// Programmatic dependent launch (PDL) chains the kernels of a photon-event
// push on ONE stream (no launch gaps, no events).  Each kernel waits
// (griddepcontrol.wait) for its predecessor where it reads its output and
// then lets its successor be scheduled (launch_dependents):
//   ingest(t) -> [proj_acc -> proj_fin -> cmp](t) -> K5s(t) -> ingest(t+1)
// K5s(t) needs only ingest(t) (complete, transitively, once cmp(t) got past
// its wait), so it skips the start wait and overlaps cmp(t); it waits at its
// END instead, so a completed K5s(t) implies a completed cmp(t).  ingest(t+1)
// touches only push t+1's buffers (hist column t+1, nonzero lists of parity
// (t+1) & 1, counters (t+1) % 3), runs beside the previous push's tail and
// waits for its predecessor before it exits: completion stays transitive.
// Without the launch attribute these instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int PZ = 8;
#ifndef XG_PZ_BATCH
#define XG_PZ_BATCH 2
#endif
constexpr int PA_MAXW = 6;  // 32-bit digit words per lane: 3 digits x k <= 768
#ifndef XG_PA_U
#define XG_PA_U 4
#endif
constexpr int PA_U = XG_PA_U;  // pixels in flight per warp
__global__ void __launch_bounds__(256) k_stream_proj_acc(StreamParams p) {
  // warp w of the CTA takes nonzeros zb + w, zb + w + 8, ...; lane L holds
  // the 32-bit digit words L, L + 32, ... of the pixel's row (4 digits per
  // word), PA_U rows in flight; the 8 warps meet in shared memory, the PZ
  // slices in pacc (integer atomics: exact, order-free)
  __shared__ int32_t red[8][768];
  const int r = blockIdx.x;
  const int f = blockIdx.z;  // frame t + f of a batch (0 for a single push)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();  // ingest(t): nonzero lists, 1/|x_t|
  pdl_launch_dependents();
  const int koff = p.ring_koff[r];
  const int n = p.nz_n[f * p.n_rings + r];
  const int32_t* nz_col = p.nz_col + f * p.nz_bstride;
  const uint8_t* nz_val = p.nz_val + f * p.nz_bstride;
  const int zb = static_cast<int>((static_cast<int64_t>(n) * blockIdx.y) / gridDim.y);
  const int ze = static_cast<int>((static_cast<int64_t>(n) * (blockIdx.y + 1)) / gridDim.y);
  const int nw = p.vdt_ld >> 2;
  int32_t acc[PA_MAXW][4];
#pragma unroll
  for (int m = 0; m < PA_MAXW; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[m][q] = 0;
  for (int e0 = zb + warp; e0 < ze; e0 += 8 * PA_U) {
    uint32_t wv[PA_U][PA_MAXW];
    int xv[PA_U];
#pragma unroll
    for (int u = 0; u < PA_U; ++u) {
      const int e = e0 + 8 * u;
      const bool in = e < ze;
      const int col = in ? nz_col[koff + e] : 0;
      xv[u] = in ? nz_val[koff + e] : 0;
      const uint32_t* row = reinterpret_cast<const uint32_t*>(p.vdt + static_cast<int64_t>(col) * p.vdt_ld);
#pragma unroll
      for (int m = 0; m < PA_MAXW; ++m) {
        const int wi = lane + 32 * m;
        wv[u][m] = (in && wi < nw) ? __ldg(row + wi) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < PA_U; ++u)
#pragma unroll
      for (int m = 0; m < PA_MAXW; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          acc[m][q] += xv[u] * static_cast<int>(static_cast<int8_t>((wv[u][m] >> (8 * q)) & 0xFFu));
  }
#pragma unroll
  for (int m = 0; m < PA_MAXW; ++m) {
    const int wi = lane + 32 * m;
    if (wi < nw && 4 * wi < 768)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[warp][4 * wi + q] = acc[m][q];
  }
  __syncthreads();
  const int nacc = p.n_digits * p.k;  // <= 768
  int32_t* pa = p.pacc + f * p.pacc_bstride + static_cast<int64_t>(r) * 768;
  for (int j = threadIdx.x; j < nacc; j += 256) {
    int32_t tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w][j];
    if (tot) atomicAdd(pa + j, tot);
  }
}

// K6a': digit sums -> coefficients with the batch projection's expression
// (bitwise-equal rows); resets pacc.
__global__ void __launch_bounds__(128) k_stream_proj_fin(StreamParams p) {
  const int r = blockIdx.x;
  const int64_t t = p.t + blockIdx.y;  // frame t + f of a batch
  pdl_wait();  // proj_acc(t): the digit sums
  pdl_launch_dependents();
  int32_t* pa = p.pacc + blockIdx.y * p.pacc_bstride + static_cast<int64_t>(r) * 768;
  const double inv = p.inv[static_cast<int64_t>(r) * p.inv_ld + t];
  for (int j = threadIdx.x; j < p.k; j += blockDim.x) {
    const int32_t a0 = pa[j], a1 = p.n_digits > 1 ? pa[p.k + j] : 0;
    const int32_t a2 = p.n_digits > 2 ? pa[2 * p.k + j] : 0;
    const double y =
        combine_digits(a0, a1, a2, p.n_digits, p.scale[static_cast<int64_t>(r) * p.k + j], inv);
    p.y[(static_cast<int64_t>(r) * p.y_ld + t) * p.k + j] = y;
    p.yf[(static_cast<int64_t>(r) * p.y_ld + t) * p.kq + j] = static_cast<float>(y);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < p.n_digits * p.k; j += blockDim.x) pa[j] = 0;
}

// K6b (single pushes): the new frame's C~ column, grid (ceil((t+1)/SR_ROWS),
// rings), a warp per 8 history rows, SIMT fp32 (per-lane fmaf chains, an
// xor-butterfly across lanes), the lag sums updated in place.  A single
// column is HBM-bound and K6b streams it at ~0.9 of HBM; the tensor-core K6
// below (batches) reached ~0.7 for one column.  The two differ in rounding
// within fp32 (both within the 1e-5 compressed contract).
template <int MAXV>
__global__ void __launch_bounds__(SR_THREADS, 4) k_stream_cmp(StreamParams p) {
  // fp32 coefficient history (C~ is fp32-accurate by contract), rows padded
  // to kq = k rounded up to 4 (zero pad): lane L holds float4 chunks L, L+32,
  // ... of the new row; a warp's 8 history rows are loaded (16 B per lane per
  // row) before any arithmetic; fp32 products summed over k, lags in f64
  const int r = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();  // proj_fin(t): y_t
  pdl_launch_dependents();
  const int kq = p.kq, nv = kq >> 2;
  const float* ybase = p.yf + static_cast<int64_t>(r) * p.y_ld * kq;
  float4 yn[MAXV];
#pragma unroll
  for (int m = 0; m < MAXV; ++m) {
    const int v = lane + 32 * m;
    yn[m] = v < nv ? *reinterpret_cast<const float4*>(ybase + p.t * kq + 4 * v)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const double inv_t = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  constexpr int RPW = SR_ROWS / (SR_THREADS / 32);
  const int64_t s_first = static_cast<int64_t>(blockIdx.x) * SR_ROWS + warp * RPW;
  float part[RPW];
#pragma unroll
  for (int q = 0; q < RPW; ++q) part[q] = 0.f;
#pragma unroll
  for (int m = 0; m < MAXV; ++m) {
    if (32 * m >= nv) break;
    const int v = lane + 32 * m;
    float4 ld[RPW];
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
      const int64_t s = s_first + q;
      ld[q] = (v < nv && s <= p.t)
                  ? __ldcs(reinterpret_cast<const float4*>(ybase + s * kq + 4 * v))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < RPW; ++q)
      part[q] = fmaf(ld[q].x, yn[m].x,
                     fmaf(ld[q].y, yn[m].y, fmaf(ld[q].z, yn[m].z, fmaf(ld[q].w, yn[m].w, part[q]))));
  }
  float mine = 0.f;
#pragma unroll
  for (int q = 0; q < RPW; ++q) {
    float a = part[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == q) mine = a;
  }
  const int64_t s = s_first + lane;
  if (lane < RPW && s <= p.t) {
    const double acc = mine;
    const double inv_s = p.inv[static_cast<int64_t>(r) * p.inv_ld + s];
    const int64_t gi = static_cast<int64_t>(r) * p.g2_ld + (p.t - s);
    p.cg2sum[gi] += acc;
    p.cg2cnt[gi] += (inv_s != 0.0 && inv_t != 0.0) ? 1 : 0;
    if (p.ccol) p.ccol[static_cast<int64_t>(r) * p.col_ring_stride + s * p.col_ld + p.t] = mine;
  }
}

}  // namespace

// K1s: one warp per 128-column block of the ring-major row (blocks never
// straddle rings).  Lane l packs columns 4l..4l+3 from the raster through the
// column -> pixel table, stores them, and adds the block's exact |x|^2 into
// its ring.  Sparse mode: nonzero columns are compacted per ring (positions
// from one atomic per warp; any order, the column sums are integer) and
// scattered into the pixel-major history.
__global__ void __launch_bounds__(128) k_stream_ingest(StreamParams p) {
  if (blockIdx.x == 0)  // the next push's counters
    for (int r = threadIdx.x; r < p.n_rings; r += blockDim.x) {
      if (p.nz_next) p.nz_next[r] = 0;
      if (p.norm2_next) p.norm2_next[r] = 0ull;
    }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk = static_cast<int64_t>(blockIdx.x) * 4 + warp;
  if (blk * 128 >= p.ktot) return;  // warp-uniform
  const int64_t c = blk * 128 + lane * 4;
  const int4 px = *reinterpret_cast<const int4*>(p.colpix + c);
  const uint32_t v0 = px.x >= 0 ? p.frame[px.x] : 0u, v1 = px.y >= 0 ? p.frame[px.y] : 0u;
  const uint32_t v2 = px.z >= 0 ? p.frame[px.z] : 0u, v3 = px.w >= 0 ? p.frame[px.w] : 0u;
  const uint32_t word = v0 | (v1 << 8) | (v2 << 16) | (v3 << 24);
  *reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(p.x) + p.t * p.ktot + c) = word;  // the stream owns x
  const uint32_t sq = __reduce_add_sync(0xffffffffu, __dp4a(word, word, 0u));
  const int r = p.blk_ring[blk];
  if (lane == 0 && sq) atomicAdd(p.norm2 + p.t * p.n_rings + r, static_cast<unsigned long long>(sq));
  if (p.nz_n) {
    const int cnt = (v0 != 0u) + (v1 != 0u) + (v2 != 0u) + (v3 != 0u);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (tot == 0) return;
    int base = 0;
    if (lane == 31) base = atomicAdd(p.nz_n + r, tot);
    base = __shfl_sync(0xffffffffu, base, 31);
    int pos = p.ring_koff[r] + base + incl - cnt;
    const uint32_t v[4] = {v0, v1, v2, v3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (v[j]) {
        p.nz_col[pos] = static_cast<int32_t>(c + j);
        p.nz_val[pos] = static_cast<uint8_t>(v[j]);
        if (p.hist) p.hist[(c + j) * p.hp + p.t] = static_cast<uint8_t>(v[j]);
        ++pos;
      }
    }
  }
}

// K1s (sparse mode): the new frame in pixel order, 1024 pixels per CTA (4
// per thread, one 32-bit load).  Only nonzero pixels look up their packed
// (ring << 22 | column) entry; the CTA counts them per ring in shared memory,
// reserves each ring's run of the nonzero list with ONE global atomic, then
// writes (column, value) and hist[column][t].  |x_t|^2 per ring likewise
// meets in shared memory first (integer sums: exact, order-free).  Block 0
// clears the next push's counters (nz_next, norm2 row t + 1).
constexpr int SI_THREADS = 256;
// pixels per thread: 4 for a single frame (16 per thread = 256 CTAs measured
// slower: 10.2 -> 14.2 us), 16 for a batch (16 frames x 1024 CTAs of 4 were
// bound by the CTAs' fixed costs -- barriers, ring counters)
constexpr int SI_MAXQ = 1024;
template <int SI_PX>
__global__ void __launch_bounds__(SI_THREADS) k_stream_ingest_sparse(StreamParams p) {
  __shared__ uint32_t cnt[SI_MAXQ], sq[SI_MAXQ];
  __shared__ int32_t base[SI_MAXQ];
  pdl_launch_dependents();
  // frame t + f of a batch (f = 0 for a single push)
  const int f = blockIdx.y;
  const int64_t tf = p.t + f;
  const uint8_t* frame = p.frame + static_cast<int64_t>(f) * p.pixels;
  int32_t* nz_col = p.nz_col + f * p.nz_bstride;
  uint8_t* nz_val = p.nz_val + f * p.nz_bstride;
  int32_t* nz_n = p.nz_n + f * p.n_rings;
  if (blockIdx.x == 0 && f == 0 && p.nz_next)
    for (int r = threadIdx.x; r < p.n_rings; r += blockDim.x) {
      p.nz_next[r] = 0;
      if (p.norm2_next) p.norm2_next[r] = 0ull;
    }
  for (int r = threadIdx.x; r < p.n_rings; r += blockDim.x) cnt[r] = sq[r] = 0;
  // SI_PX pixels per thread (one 32-bit load)
  const int64_t px0 = (static_cast<int64_t>(blockIdx.x) * SI_THREADS + threadIdx.x) * SI_PX;
  uint32_t wv[SI_PX / 4];
  if (px0 + SI_PX <= p.pixels) {
    if (SI_PX == 16) {
      const uint4 q = __ldcs(reinterpret_cast<const uint4*>(frame + px0));
      wv[0] = q.x;
      wv[SI_PX / 4 > 1 ? 1 : 0] = q.y;
      wv[SI_PX / 4 > 2 ? 2 : 0] = q.z;
      wv[SI_PX / 4 > 3 ? 3 : 0] = q.w;
    } else {
      wv[0] = __ldcs(reinterpret_cast<const uint32_t*>(frame + px0));
    }
  } else {
#pragma unroll
    for (int k = 0; k < SI_PX / 4; ++k) {
      wv[k] = 0;
      for (int b = 0; b < 4; ++b)
        if (px0 + 4 * k + b < p.pixels)
          wv[k] |= static_cast<uint32_t>(frame[px0 + 4 * k + b]) << (8 * b);
    }
  }
  int ent[SI_PX], loc[SI_PX];
  __syncthreads();
#pragma unroll
  for (int b = 0; b < SI_PX; ++b) {
    ent[b] = -1;
    const uint32_t v = (wv[b >> 2] >> (8 * (b & 3))) & 0xFFu;
    if (!v) continue;
    const int e = p.pixcol[px0 + b];
    if (e < 0) continue;
    ent[b] = e;
    const int r = e >> 22;
    loc[b] = static_cast<int>(atomicAdd(&cnt[r], 1u));
    atomicAdd(&sq[r], v * v);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < p.n_rings; r += blockDim.x) {
    if (cnt[r]) {
      base[r] = p.ring_koff[r] + atomicAdd(nz_n + r, static_cast<int>(cnt[r]));
      atomicAdd(p.norm2 + tf * p.n_rings + r, static_cast<unsigned long long>(sq[r]));
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < SI_PX; ++b) {
    if (ent[b] < 0) continue;
    const int r = ent[b] >> 22, col = ent[b] & 0x3FFFFF;
    const uint8_t v = static_cast<uint8_t>((wv[b >> 2] >> (8 * (b & 3))) & 0xFFu);
    const int64_t e = base[r] + loc[b];
    nz_col[e] = col;
    nz_val[e] = v;
    if (p.hist) p.hist[static_cast<int64_t>(col) * p.hp + tf] = v;
  }
  // the last CTA of frame t + f to finish computes its norms, 1/|x|, nonzero
  // bit and zero-frame bookkeeping (k_norms' expressions; the zero count and
  // first zero are order-free atomics) -- no separate launch
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(p.done + f, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  pdl_wait();  // the previous push's column kernel has completed (see above)
  if (!last) return;
  __threadfence();
  for (int r = threadIdx.x; r < p.n_rings; r += blockDim.x) {
    const int64_t tt = tf;
    const long long n2 = static_cast<long long>(atomicAdd(p.norm2 + tt * p.n_rings + r, 0ull));
    const double nrm = sqrt(static_cast<double>(n2));
    p.norms_w[r * p.inv_ld + tt] = nrm;
    p.inv_w[r * p.inv_ld + tt] = n2 > 0 ? 1.0 / nrm : 0.0;
    if (n2 > 0) {
      atomicOr(p.nz_bits + static_cast<int64_t>(r) * p.nz_words + (tt >> 5), 1u << (tt & 31));
    } else {
      atomicAdd(reinterpret_cast<unsigned long long*>(p.zero_count + r), 1ull);
      atomicMin(reinterpret_cast<long long*>(p.first_zero + r), static_cast<long long>(tt));
    }
    if (n2 >= (1ll << 31) && p.ovf_check) atomicOr(p.err, 4);
  }
  if (threadIdx.x == 0) p.done[f] = 0u;
}

// K5s: grid (ceil((t+1)/SS_F), rings), 8 warps.  A CTA owns SS_F = 32 SS_V
// history frames s: lane L of every warp holds SS_V consecutive s and warp w
// walks the nonzeros i = w, w+8, ... of the ring, one coalesced SS_V-byte
// load of hist[c_i][s..] per nonzero (SS_U of them in flight); the 8 warps'
// integer partial sums meet in shared memory (exact, fixed order), and the
// CTA finishes its column entries itself: C, g2 lag sums, optional stored
// column -- the dense K5's expressions, so the results equal it bitwise.  No
// atomics, no second pass.
constexpr int SS_CHUNK = 1024;
#ifndef XG_SS_V
#define XG_SS_V 8
#endif
#ifndef XG_SS_U
#define XG_SS_U 12
#endif
constexpr int SS_V = XG_SS_V;  // history frames per lane (one 8- or 16-byte load)
constexpr int SS_U = XG_SS_U;  // loads in flight per lane
constexpr int SS_F = 32 * SS_V;  // history frames per CTA
#ifndef XG_SS_W
#define XG_SS_W 8
#endif
constexpr int SS_W = XG_SS_W;  // warps per CTA, splitting the ring's nonzeros
// 12 loads in flight per lane at 4 CTAs per SM (64 registers): 41.5 -> 40.1
// us per push at depth 8192 (8 loads at 4-5 CTAs: 40.5-41.5 us; 16 loads at 3
// CTAs: 50 us).  A persistent form (CTAs walking (ring, window) items, warps
// reading their nonzero entries straight from global, one warp finishing an
// item while the others stream the next) ran 71 us: each item became a longer
// chain of dependent round trips.
constexpr int SS_MINB = 4;
template <int V> struct SsVec;
template <> struct SsVec<8> {
  using T = uint2;
  __device__ static void words(const T& v, uint32_t* w) { w[0] = v.x; w[1] = v.y; }
  __device__ static T zero() { return make_uint2(0u, 0u); }
};
template <> struct SsVec<16> {
  using T = uint4;
  __device__ static void words(const T& v, uint32_t* w) { w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w; }
  __device__ static T zero() { return make_uint4(0u, 0u, 0u, 0u); }
};
// BATCH: grid.z = frame t + j of a batch (its nonzero lists in slot j); the
// column entries go to the scratch column (r, j) and k_stream_fold adds them
// to the lag sums in frame order -- the frames' loads all overlap.
template <bool BATCH>
__global__ void __launch_bounds__(32 * SS_W, SS_MINB) k_stream_sparse(StreamParams p) {
  using VT = typename SsVec<SS_V>::T;
  __shared__ int32_t sc[SS_CHUNK];
  __shared__ uint32_t sv[SS_CHUNK];
  __shared__ uint32_t red[SS_W][SS_F + 1];
  const int r = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = BATCH ? static_cast<int>(blockIdx.z) : 0;
  const int64_t t = p.t + j;
  const int64_t sb = (BATCH ? p.s_begin : 0) + static_cast<int64_t>(blockIdx.x) * SS_F;
  if (BATCH && sb > t) return;  // CTA-uniform
  const int32_t* nz_col = p.nz_col + j * p.nz_bstride;
  const uint8_t* nz_val = p.nz_val + j * p.nz_bstride;
  // this push's ingest has completed: nonzero lists, hist column t, 1/|x_t|
  // (waited for here, or transitively through the compressed kernels; in a
  // photon-event batch the ingest of every frame completed before the
  // batch's first K5s started, so K5s(t+1) may stream its history while
  // K5s(t) still runs and waits for it only before touching the g2 sums)
  if (!BATCH) {
    if (!p.pdl_wait_end && !p.pdl_wait_fin) pdl_wait();
    pdl_launch_dependents();
  }
  const int koff = p.ring_koff[r];
  const int n = p.nz_n[j * p.n_rings + r];
  const int64_t s0 = sb + SS_V * lane;
  uint32_t acc[SS_V];
#pragma unroll
  for (int j = 0; j < SS_V; ++j) acc[j] = 0;
  const uint8_t* h = p.hist + s0;
  for (int c0 = 0; c0 < n; c0 += SS_CHUNK) {
    const int cn = n - c0 < SS_CHUNK ? n - c0 : SS_CHUNK;
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += 32 * SS_W) {
      sc[i] = nz_col[koff + c0 + i];
      sv[i] = nz_val[koff + c0 + i];
    }
    __syncthreads();
    if (s0 <= t) {
      // SS_U independent loads in flight per lane before any use
      for (int i0 = warp; i0 < cn; i0 += SS_W * SS_U) {
        VT wv[SS_U];
        uint32_t vv[SS_U];
#pragma unroll
        for (int u = 0; u < SS_U; ++u) {
          const int i = i0 + SS_W * u;
          const bool in = i < cn;
          vv[u] = in ? sv[i] : 0u;
          wv[u] = in ? __ldcs(reinterpret_cast<const VT*>(h + static_cast<int64_t>(sc[i]) * p.hp))
                     : SsVec<SS_V>::zero();
        }
#pragma unroll
        for (int u = 0; u < SS_U; ++u) {
          uint32_t ww[SS_V / 4];
          SsVec<SS_V>::words(wv[u], ww);
          // byte j of a history word times the new count: one dp4a against
          // the count placed in byte lane j (exact integer arithmetic)
          const int b0 = static_cast<int>(vv[u]);
#pragma unroll
          for (int q = 0; q < SS_V / 4; ++q)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              acc[4 * q + j] = static_cast<uint32_t>(
                  __dp4a(ww[q], static_cast<unsigned>(b0) << (8 * j), acc[4 * q + j]));
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < SS_V; ++q) red[warp][SS_V * lane + q] = acc[q];
  if (!BATCH && p.pdl_wait_fin) pdl_wait();  // K5s(t-1) done: lag sums in push order
  __syncthreads();
  const double inv_t = BATCH ? 0.0 : p.inv[static_cast<int64_t>(r) * p.inv_ld + t];
#pragma unroll
  for (int f = threadIdx.x; f < SS_F; f += 32 * SS_W) {
    const int64_t s = sb + f;
    if (s > t) break;
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < SS_W; ++w) tot += red[w][f];
    const int accv = static_cast<int>(tot);
    if (BATCH) {
      p.gscr[(static_cast<int64_t>(r) * p.scr_nb + j) * p.scr_ld + s] = accv;
    } else {
      const double inv_s = p.inv[static_cast<int64_t>(r) * p.inv_ld + s];
      const int64_t gi = static_cast<int64_t>(r) * p.g2_ld + (t - s);
      p.g2sum[gi] += static_cast<double>(accv) * (inv_s * inv_t);
      p.g2cnt[gi] += (inv_s != 0.0 && inv_t != 0.0) ? 1 : 0;
    }
    if (p.gcol) p.gcol[static_cast<int64_t>(r) * p.col_ring_stride + s * p.col_ld + t] = accv;
  }
  if (!BATCH && p.pdl_wait_end) pdl_wait();  // cmp(t) has completed too (see above)
}

// K6 (batches): the compressed columns C~(s, t + j) of the nb <= 16 frames
// of a push_many batch on tensor cores, grid (ceil((t + nb) / 128), rings),
// a warp per 16 history rows: mma.sync m16n8k8 tf32 -> fp32, the history
// rows as A (straight from global into registers), the new rows as B
// (shared memory).  3xTF32: every fp32 value x = big + small with big = x's
// top 19 bits (what the tensor core reads) and small = x - big (exact);
// big*big + big*small + small*big carry ~2^-21 relative (small*small
// dropped), the fp32-accurate contract's 1e-5 with margin.  Inside each
// 8-wide k-step thread q of a quad reads physical columns (2q, 2q+1) as
// logical k (q, q+4), so its A and B fragments are single 8-byte loads (the
// set of products summed is unchanged).  The history is read once per 16
// frames; the entries go to scratch columns for the fold.
__device__ __forceinline__ void mma1688(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void tf32_split(float x, uint32_t& big, uint32_t& small) {
  big = __float_as_uint(x) & 0xFFFFE000u;
  small = __float_as_uint(x - __uint_as_float(big));
}
constexpr int CB_MAXNB = 16;
constexpr int TC_KMAX = 256;
constexpr int TC_BLD = TC_KMAX + 8;  // plane row pitch: conflict-free 8-byte B loads
#ifndef XG_TC_KG
#define XG_TC_KG 4
#endif
#ifndef XG_TC_MINB
#define XG_TC_MINB 4
#endif
constexpr int TC_KG = XG_TC_KG;  // k-steps of A loaded before their MMAs
template <int NT, int KG>
__global__ void __launch_bounds__(256, XG_TC_MINB) k_stream_cmp_tc(StreamParams p) {
  __shared__ __align__(16) float bsm[2][8 * NT][TC_BLD];  // big / small planes of the new rows
  const int r = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  pdl_wait();  // proj_fin: the new rows
  pdl_launch_dependents();
  const int kq = p.kq, ks = (kq + 7) >> 3, nb = p.scr_nb;
  const float* ybase = p.yf + static_cast<int64_t>(r) * p.y_ld * kq;
  for (int i = threadIdx.x; i < 8 * NT * ks * 8; i += 256) {
    const int jj = i / (ks * 8), kk = i % (ks * 8);
    const float v = (jj < nb && kk < kq) ? ybase[(p.t + jj) * kq + kk] : 0.f;
    uint32_t bg, sm;
    tf32_split(v, bg, sm);
    bsm[0][jj][kk] = __uint_as_float(bg);
    bsm[1][jj][kk] = __uint_as_float(sm);
  }
  __syncthreads();
  const int64_t t_last = p.t + nb - 1;
  const int64_t s_base = static_cast<int64_t>(blockIdx.x) * 128 + warp * 16;
  if (s_base > t_last) return;  // warp-uniform, no barrier follows
  const int64_t ra = s_base + gid, rb = ra + 8;
  const float* rowa = ybase + ra * kq;
  const float* rowb = ybase + rb * kq;
  const bool va = ra <= t_last, vb = rb <= t_last;
  // two accumulator chains per n-tile (the cross products; big * big),
  // summed at the end
  float acc[NT][4], acs[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[nt][q] = acs[nt][q] = 0.f;
  for (int kb0 = 0; kb0 < ks; kb0 += KG) {
    float2 la[KG], lb[KG];
#pragma unroll
    for (int g = 0; g < KG; ++g) {
      const int c = (kb0 + g) * 8 + 2 * tig;
      const float2 z = make_float2(0.f, 0.f);
      la[g] = (va && c < kq) ? __ldcs(reinterpret_cast<const float2*>(rowa + c)) : z;
      lb[g] = (vb && c < kq) ? __ldcs(reinterpret_cast<const float2*>(rowb + c)) : z;
    }
#pragma unroll
    for (int g = 0; g < KG; ++g) {
      const int kb = kb0 + g;
      if (kb >= ks) break;
      uint32_t ab[4], as[4];
      tf32_split(la[g].x, ab[0], as[0]);  // (row gid,     logical k q)
      tf32_split(lb[g].x, ab[1], as[1]);  // (row gid + 8, logical k q)
      tf32_split(la[g].y, ab[2], as[2]);  // (row gid,     logical k q + 4)
      tf32_split(lb[g].y, ab[3], as[3]);  // (row gid + 8, logical k q + 4)
      const int c = kb * 8 + 2 * tig;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int n = nt * 8 + gid;
        const float2 bb = *reinterpret_cast<const float2*>(&bsm[0][n][c]);
        const float2 bs = *reinterpret_cast<const float2*>(&bsm[1][n][c]);
        mma1688(acs[nt], as, __float_as_uint(bb.x), __float_as_uint(bb.y));
        mma1688(acs[nt], ab, __float_as_uint(bs.x), __float_as_uint(bs.y));
        mma1688(acc[nt], ab, __float_as_uint(bb.x), __float_as_uint(bb.y));
      }
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float v = acc[nt][q] + acs[nt][q];
      const int j = nt * 8 + tig * 2 + (q & 1);
      const int64_t srow = q < 2 ? ra : rb;
      const int64_t t = p.t + j;
      if (j < nb && srow <= t) {
        p.cscr[(static_cast<int64_t>(r) * nb + j) * p.scr_ld + srow] = v;
        if (p.ccol) p.ccol[static_cast<int64_t>(r) * p.col_ring_stride + srow * p.col_ld + t] = v;
      }
    }
}

template <int NT>
static cudaError_t launch_cmp_tc(const StreamParams& p, int32_t n_rings, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>((p.t + p.scr_nb + 127) / 128), n_rings);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_stream_cmp_tc<NT, TC_KG>, p);
}

// ---------------------------------------------------------- event history
// Photon-event data at mu ~ 0.02 leaves ~98% of the dense history bytes
// zero, and the dense column reads all of them (nnz * t bytes per frame).
// A sealed block of EV tb frames keeps, per pixel column, the list of its
// (s_local, count) events: a column entry then costs one 8-byte index load
// plus ~tb * occupancy 4-byte events instead of tb bytes.

// nonzero bytes of a 32-bit word
__device__ __forceinline__ uint32_t nzbytes(uint32_t x) {
  return __popc((((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u);
}

constexpr int EV_MAXTB = 8192;  // frames of a segment (its column entries in shared memory)
// Seal: grid ceil(ktot / 256), 8 warps; warp w takes pixel columns c0 + 32 w
// .. + 32 one at a time, lane L the words [L wpl, (L + 1) wpl) of the row's
// block (wpl = tb / 128).  Pass 1 counts each column's events; the CTA scans
// its 256 counts and reserves its run of the block's list with one atomic;
// pass 2 re-reads the rows (L2) and writes the events in ascending s.
__global__ void __launch_bounds__(256) k_stream_seal(SealParams p) {
  __shared__ int32_t cnt[256], offs[256];
  __shared__ int32_t wsum[8];
  __shared__ long long base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 256;
  const int wpl = p.tb >> 7;
  const int64_t boff = static_cast<int64_t>(p.block) * p.tb;
  for (int i = 0; i < 32; ++i) {
    const int64_t c = c0 + warp * 32 + i;
    uint32_t n = 0;
    if (c < p.ktot) {
      const uint32_t* row = reinterpret_cast<const uint32_t*>(p.hist + c * p.hp + boff) + lane * wpl;
      for (int w = 0; w < wpl; ++w) n += nzbytes(row[w]);
    }
    n = __reduce_add_sync(0xffffffffu, n);
    if (lane == 0) cnt[warp * 32 + i] = static_cast<int32_t>(n);
  }
  __syncthreads();
  // exclusive scan of the 256 counts (thread = column)
  const int mine = cnt[threadIdx.x];
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int wb = 0;
  for (int w = 0; w < warp; ++w) wb += wsum[w];
  const int excl = wb + incl - mine;
  offs[threadIdx.x] = excl;
  if (threadIdx.x == 255) {
    const long long tot = wb + incl;
    base = tot ? static_cast<long long>(atomicAdd(p.cursor + p.slot, static_cast<unsigned long long>(tot)))
               : 0ll;
    if (base + tot > p.cap) {
      atomicExch(p.dense + p.slot, 1);
      base = -1;
    }
  }
  __syncthreads();
  if (base < 0) return;  // the block stays dense
  if (c0 + threadIdx.x < p.ktot)  // offsets relative to the block's list
    p.evidx[static_cast<int64_t>(p.slot) * p.ktot + c0 + threadIdx.x] =
        make_int2(static_cast<int>(base + excl), mine);
  uint32_t* evb = p.ev + static_cast<int64_t>(p.slot) * p.cap;
  for (int i = 0; i < 32; ++i) {
    const int cl = warp * 32 + i;
    const int64_t c = c0 + cl;
    if (c >= p.ktot || cnt[cl] == 0) continue;  // warp-uniform
    const uint32_t* row = reinterpret_cast<const uint32_t*>(p.hist + c * p.hp + boff) + lane * wpl;
    uint32_t wv[8];
    uint32_t n = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      wv[w] = w < wpl ? row[w] : 0u;
      n += nzbytes(wv[w]);
    }
    uint32_t pre = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += v;
    }
    pre -= n;
    int64_t pos = base + offs[cl] + pre;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      if (w >= wpl) break;
      uint32_t x = wv[w];
      while (x) {
        const int b = (__ffs(x) - 1) >> 3;
        const uint32_t v = (x >> (8 * b)) & 0xFFu;
        evb[pos++] = (static_cast<uint32_t>((lane * wpl + w) * 4 + b) << 8) | v;
        x &= ~(0xFFu << (8 * b));
      }
    }
  }
}

// Merge: grid ceil(ktot / 256), thread = pixel column for the counts and
// scan, then warp w copies the lists of its 32 columns one column at a time
// (lanes over events, coalesced), adding b tb to the s_local of block b.
__global__ void __launch_bounds__(256) k_stream_merge(MergeParams p) {
  __shared__ int32_t offs[256];
  __shared__ int32_t wsum[8];
  __shared__ long long base;
  __shared__ int dense;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    int d = 0;
    for (int b = 0; b < p.nf; ++b) d |= p.dense0[b];
    dense = d;
    if (d && blockIdx.x == 0) p.dense1[p.seg] = 1;
  }
  __syncthreads();
  if (dense) return;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  int mine = 0;
  if (c < p.ktot)
    for (int b = 0; b < p.nf; ++b) mine += p.evidx0[b * p.ktot + c].y;
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int wb = 0;
  for (int w = 0; w < warp; ++w) wb += wsum[w];
  offs[threadIdx.x] = wb + incl - mine;
  if (threadIdx.x == 255) {
    const long long tot = wb + incl;
    base = tot ? static_cast<long long>(atomicAdd(p.cursor1 + p.seg, static_cast<unsigned long long>(tot)))
               : 0ll;
    if (base + tot > p.cap1) {
      atomicExch(p.dense1 + p.seg, 1);
      base = -1;
    }
  }
  __syncthreads();
  if (base < 0) return;
  if (c < p.ktot)
    p.evidx1[static_cast<int64_t>(p.seg) * p.ktot + c] =
        make_int2(static_cast<int>(base + offs[threadIdx.x]), mine);
  uint32_t* dst0 = p.ev1 + static_cast<int64_t>(p.seg) * p.cap1 + base;
  for (int i = 0; i < 32; ++i) {
    const int cl = warp * 32 + i;
    const int64_t cc = static_cast<int64_t>(blockIdx.x) * 256 + cl;
    if (cc >= p.ktot) break;
    uint32_t* dst = dst0 + offs[cl];
    for (int b = 0; b < p.nf; ++b) {
      const int2 e = p.evidx0[b * p.ktot + cc];
      const uint32_t* src = p.ev0 + b * p.cap0 + e.x;
      const uint32_t add = static_cast<uint32_t>(b * p.tb) << 8;
      for (int k = lane; k < e.y; k += 32) dst[k] = __ldg(src + k) + add;
      dst += e.y;
    }
  }
}

// K5e: grid (segments, rings, nb) for one level; CTA (g, r, j) forms the
// column entries G(s, t + j) of segment g's frames for ring r from the new
// frame's nonzero pixels: a thread per pixel walks the pixel's event list
// and adds count x count into shared memory (integer atomics: exact, order-
// free); a dense-flagged segment is read from the dense history instead.
#ifndef XG_EV_U4
#define XG_EV_U4 8
#endif
#ifndef XG_EV_MINB
#define XG_EV_MINB 4
#endif
constexpr int EV_U4 = XG_EV_U4;  // 16-byte event words in flight per thread
__global__ void __launch_bounds__(256, XG_EV_MINB) k_stream_events(StreamParams p, int lvl) {
  extern __shared__ int32_t acc[];
  const int g = blockIdx.x, r = blockIdx.y, j = blockIdx.z;
  const int64_t t = p.t + j;
  const int tb = p.ev_tb[lvl];
  const int seg = p.ev_first[lvl] + g;
  const int slot = p.ev_ring[lvl] ? seg % p.ev_ring[lvl] : seg;
  for (int i = threadIdx.x; i < tb; i += 256) acc[i] = 0;
  __syncthreads();
  const int koff = p.ring_koff[r];
  const int n = p.nz_n[j * p.n_rings + r];
  const int32_t* nz_col = p.nz_col + j * p.nz_bstride + koff;
  const uint8_t* nz_val = p.nz_val + j * p.nz_bstride + koff;
  const int64_t s0 = static_cast<int64_t>(seg) * tb;
  if (!p.ev_dense[lvl][slot]) {
    const int2* idx = p.evidx[lvl] + static_cast<int64_t>(slot) * p.ktot;
    const uint32_t* ev = p.ev[lvl] + static_cast<int64_t>(slot) * p.ev_cap[lvl];
    // a thread per pixel: its list read as aligned 16-byte words (4 events;
    // a scalar load per event made the L1 the limit: 89% busy), EV_U4 of
    // them in flight before the first atomic
    const uint4* ev4 = reinterpret_cast<const uint4*>(ev);
    for (int i = threadIdx.x; i < n; i += 256) {
      const int col = nz_col[i];
      const int xv = nz_val[i];
      const int2 e = __ldg(idx + col);
      const int end = e.x + e.y;
      int k = e.x & ~3;
      uint4 w[EV_U4];
#pragma unroll
      for (int u = 0; u < EV_U4; ++u)
        w[u] = k + 4 * u < end ? __ldg(ev4 + ((k >> 2) + u)) : make_uint4(0u, 0u, 0u, 0u);
      while (k < end) {
#pragma unroll
        for (int u = 0; u < EV_U4; ++u) {
          const uint32_t ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int at = k + 4 * u + c;
            if (at >= e.x && at < end)
              atomicAdd(&acc[ww[c] >> 8], static_cast<int>(ww[c] & 0xFFu) * xv);
          }
        }
        k += 4 * EV_U4;
#pragma unroll
        for (int u = 0; u < EV_U4; ++u)
          w[u] = k + 4 * u < end ? __ldg(ev4 + ((k >> 2) + u)) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpl = tb >> 7;
    for (int i = warp; i < n; i += 8) {
      const int col = nz_col[i];
      const int xv = nz_val[i];
      const uint32_t* row = reinterpret_cast<const uint32_t*>(p.hist + static_cast<int64_t>(col) * p.hp + s0) + lane * wpl;
      for (int w = 0; w < wpl; ++w) {
        uint32_t x = row[w];
        while (x) {
          const int bb = (__ffs(x) - 1) >> 3;
          atomicAdd(&acc[(lane * wpl + w) * 4 + bb], static_cast<int>((x >> (8 * bb)) & 0xFFu) * xv);
          x &= ~(0xFFu << (8 * bb));
        }
      }
    }
  }
  __syncthreads();
  int32_t* dst = p.gscr + (static_cast<int64_t>(r) * p.scr_nb + j) * p.scr_ld + s0;
  for (int i = threadIdx.x; i < tb; i += 256) {
    dst[i] = acc[i];
    if (p.gcol) p.gcol[static_cast<int64_t>(r) * p.col_ring_stride + (s0 + i) * p.col_ld + t] = acc[i];
  }
}

// The lag sums of a batch: thread per lag d of ring r, frames in ascending
// order -- exactly the per-push updates of K5s (RAW) / K6b, in push order.
template <bool RAW>
__global__ void __launch_bounds__(256) k_stream_fold(StreamParams p) {
  pdl_wait();  // single pushes: chained after the column kernel
  pdl_launch_dependents();
  const int r = blockIdx.y;
  const int nb = p.scr_nb;
  const int64_t d = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  if (d > p.t + nb - 1) return;
  const int64_t gi = static_cast<int64_t>(r) * p.g2_ld + d;
  double* sump = RAW ? p.g2sum : p.cg2sum;
  int64_t* cntp = RAW ? p.g2cnt : p.cg2cnt;
  double sum = sump[gi];
  int64_t cnt = cntp[gi];
  const double* inv = p.inv + static_cast<int64_t>(r) * p.inv_ld;
  for (int j = 0; j < nb; ++j) {
    const int64_t t = p.t + j, s = t - d;
    if (s < 0) continue;
    const double inv_s = inv[s], inv_t = inv[t];
    const int64_t si = (static_cast<int64_t>(r) * nb + j) * p.scr_ld + s;
    if (RAW) {
      const int accv = p.gscr[si];
      sum += static_cast<double>(accv) * (inv_s * inv_t);
    } else {
      const double acc = p.cscr[si];
      sum += acc;
    }
    cnt += (inv_s != 0.0 && inv_t != 0.0) ? 1 : 0;
  }
  sump[gi] = sum;
  cntp[gi] = cnt;
}

cudaError_t launch_stream_ingest(const StreamParams& p, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((p.ktot / 128 + 3) / 4);
  k_stream_ingest<<<blocks, 128, 0, s>>>(p);
  return cudaGetLastError();
}

template <typename K>
static cudaError_t launch_maybe_pdl(K kernel, dim3 grid, dim3 block, cudaStream_t s, bool pdl,
                                   const StreamParams& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

cudaError_t launch_stream_ingest_sparse(const StreamParams& p, cudaStream_t s, bool pdl,
                                        int32_t n_frames) {
  if (p.n_rings > SI_MAXQ) return cudaErrorInvalidValue;
  // 16 pixels per thread need 16-byte aligned frames (the batched path's)
  const bool wide = n_frames > 1 && (p.pixels & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(p.frame) & 15u) == 0;
  const int px = wide ? 16 : 4;
  const unsigned blocks = static_cast<unsigned>((p.pixels + px * SI_THREADS - 1) / (px * SI_THREADS));
  if (wide)
    return launch_maybe_pdl(k_stream_ingest_sparse<16>, dim3(blocks, n_frames), dim3(SI_THREADS), s,
                            pdl, p);
  return launch_maybe_pdl(k_stream_ingest_sparse<4>, dim3(blocks, n_frames), dim3(SI_THREADS), s,
                          pdl, p);
}

cudaError_t launch_stream_sparse(const StreamParams& p, int32_t n_rings, cudaStream_t s, bool pdl) {
  dim3 grid(static_cast<unsigned>((p.t + 1 + SS_F - 1) / SS_F), n_rings);
  return launch_maybe_pdl(k_stream_sparse<false>, grid, dim3(32 * SS_W), s, pdl, p);
}

cudaError_t launch_stream_batch(const StreamParams& p, int32_t n_rings, bool raw, bool cmp,
                                cudaStream_t s) {
  const int nb = p.scr_nb;
  if (nb < 1 || nb > CB_MAXNB) return cudaErrorInvalidValue;
  const int64_t rows = p.t + nb;
  const dim3 fold_grid(static_cast<unsigned>((rows + 255) / 256), n_rings);
  if (cmp) {
    // a batch has nb x rings CTAs without slicing a ring's nonzeros (PZ
    // slices per frame multiplied the integer atomics on pacc: 78 us / 16)
    k_stream_proj_acc<<<dim3(n_rings, XG_PZ_BATCH, nb), 256, 0, s>>>(p);
    k_stream_proj_fin<<<dim3(n_rings, nb), 128, 0, s>>>(p);
    if (p.kq > TC_KMAX) return cudaErrorInvalidValue;
    const cudaError_t e = launch_cmp_tc<2>(p, n_rings, s, false);
    if (e != cudaSuccess) return e;
    k_stream_fold<false><<<fold_grid, 256, 0, s>>>(p);
  }
  if (raw) {
    for (int l = 0; l < 2; ++l) {
      if (p.ev_n[l] <= 0) continue;
      if (p.ev_tb[l] > EV_MAXTB || p.ev_tb[l] % 128) return cudaErrorInvalidValue;
      const size_t smem = static_cast<size_t>(p.ev_tb[l]) * sizeof(int32_t);
      if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(
            k_stream_events, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
      }
      k_stream_events<<<dim3(p.ev_n[l], n_rings, nb), 256, smem, s>>>(p, l);
    }
    const dim3 grid(static_cast<unsigned>((rows - p.s_begin + SS_F - 1) / SS_F), n_rings, nb);
    k_stream_sparse<true><<<grid, 32 * SS_W, 0, s>>>(p);
    k_stream_fold<true><<<fold_grid, 256, 0, s>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_stream_merge(const MergeParams& p, cudaStream_t s) {
  if (int64_t{p.nf} * p.tb > EV_MAXTB || int64_t{p.nf} * p.tb >= (1 << 24)) return cudaErrorInvalidValue;
  k_stream_merge<<<static_cast<unsigned>((p.ktot + 255) / 256), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_stream_seal(const SealParams& p, cudaStream_t s) {
  if (p.tb > 1024 || p.tb % 128) return cudaErrorInvalidValue;
  k_stream_seal<<<static_cast<unsigned>((p.ktot + 255) / 256), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_stream_raw(const StreamParams& p, int32_t n_rings, int64_t max_kpad,
                              cudaStream_t s) {
  const size_t smem = static_cast<size_t>(max_kpad);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_stream_raw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(static_cast<unsigned>((p.t + 1 + SR_ROWS - 1) / SR_ROWS), n_rings);
  k_stream_raw<<<grid, SR_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_stream_cmp(const StreamParams& p, int32_t n_rings, cudaStream_t s, bool pdl) {
  // one frame: K6a (projection) -> K6b (column + lag sums), PDL-chained
  cudaError_t e = launch_maybe_pdl(k_stream_proj_acc, dim3(n_rings, PZ), dim3(256), s, pdl, p);
  if (e != cudaSuccess) return e;
  e = launch_maybe_pdl(k_stream_proj_fin, dim3(n_rings), dim3(128), s, pdl, p);
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((p.t + 1 + SR_ROWS - 1) / SR_ROWS), n_rings);
  const int nv = p.kq / 4;  // float4 chunks per coefficient row (k <= 256)
  if (nv <= 32) return launch_maybe_pdl(k_stream_cmp<1>, grid, dim3(SR_THREADS), s, pdl, p);
  return launch_maybe_pdl(k_stream_cmp<2>, grid, dim3(SR_THREADS), s, pdl, p);
}

}  // namespace xg
