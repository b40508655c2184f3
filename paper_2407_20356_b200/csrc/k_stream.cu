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
constexpr int PZ = 8;
__global__ void __launch_bounds__(256) k_stream_proj_acc(StreamParams p) {
  const int r = blockIdx.x;
  const int koff = p.ring_koff[r];
  const int n = p.nz_n[r];
  const int zb = static_cast<int>((static_cast<int64_t>(n) * blockIdx.y) / PZ);
  const int ze = static_cast<int>((static_cast<int64_t>(n) * (blockIdx.y + 1)) / PZ);
  const int nacc = p.n_digits * p.k;  // <= 768
  __shared__ int32_t sc[256];
  __shared__ int32_t sv[256];
  int32_t acc[3] = {0, 0, 0};
  for (int c0 = zb; c0 < ze; c0 += 256) {
    const int cn = ze - c0 < 256 ? ze - c0 : 256;
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < cn) {
      sc[threadIdx.x] = p.nz_col[koff + c0 + threadIdx.x];
      sv[threadIdx.x] = p.nz_val[koff + c0 + threadIdx.x];
    }
    __syncthreads();
#pragma unroll 8
    for (int e = 0; e < cn; ++e) {
      const int8_t* vd = p.vdt + static_cast<int64_t>(sc[e]) * p.vdt_ld;
      const int xv = sv[e];
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int j = threadIdx.x + 256 * m;
        if (j < nacc) acc[m] += xv * vd[j];
      }
    }
  }
  int32_t* pa = p.pacc + static_cast<int64_t>(r) * 768;
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const int j = threadIdx.x + 256 * m;
    if (j < nacc && acc[m]) atomicAdd(pa + j, acc[m]);
  }
}

// K6a': digit sums -> coefficients with the batch projection's expression
// (bitwise-equal rows); resets pacc (and nz_n when this is the last pass).
__global__ void __launch_bounds__(128) k_stream_proj_fin(StreamParams p) {
  const int r = blockIdx.x;
  int32_t* pa = p.pacc + static_cast<int64_t>(r) * 768;
  const double inv = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  for (int j = threadIdx.x; j < p.k; j += blockDim.x) {
    const int32_t a0 = pa[j], a1 = p.n_digits > 1 ? pa[p.k + j] : 0;
    const int32_t a2 = p.n_digits > 2 ? pa[2 * p.k + j] : 0;
    const double y =
        combine_digits(a0, a1, a2, p.n_digits, p.scale[static_cast<int64_t>(r) * p.k + j], inv);
    p.y[(static_cast<int64_t>(r) * p.y_ld + p.t) * p.k + j] = y;
    p.yf[(static_cast<int64_t>(r) * p.y_ld + p.t) * p.k + j] = static_cast<float>(y);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < p.n_digits * p.k; j += blockDim.x) pa[j] = 0;
  if (threadIdx.x == 0 && p.nz_reset == 2) p.nz_n[r] = 0;
}

// K6b: grid (ceil((t+1)/SR_ROWS), rings); a warp per history row.
__global__ void __launch_bounds__(SR_THREADS) k_stream_cmp(StreamParams p) {
  // fp32 coefficient history (C~ is fp32-accurate by contract): half the
  // bytes of the f64 rows; products summed in fp32 over k, lags in f64
  __shared__ float yt[1024];
  const int r = blockIdx.y;
  const float* ybase = p.yf + static_cast<int64_t>(r) * p.y_ld * p.k;
  for (int j = threadIdx.x; j < p.k; j += blockDim.x) yt[j] = ybase[p.t * p.k + j];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double inv_t = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  // a warp's 8 rows are independent: all their loads go out before any
  // reduction, and lanes 0..7 then update the 8 lags in parallel
  constexpr int RPW = SR_ROWS / (SR_THREADS / 32);
  const int64_t s_first = static_cast<int64_t>(blockIdx.x) * SR_ROWS + warp * RPW;
  float part[RPW];
#pragma unroll
  for (int q = 0; q < RPW; ++q) {
    const int64_t s = s_first + q;
    float a = 0.f;
    if (s <= p.t) {
      const float* ys = ybase + s * p.k;
      for (int j = lane; j < p.k; j += 32) a = fmaf(__ldcs(ys + j), yt[j], a);
    }
    part[q] = a;
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

// K5s-b: grid (ceil((t+1)/2048), rings, SS_Z).  A thread owns 8 consecutive
// history frames s and walks its z-slice of the ring's nonzeros: one
// coalesced 64-bit load of hist[c][s..s+7] per nonzero; the slices' partial
// integer sums meet in colbuf (integer atomics: exact, order-free).
constexpr int SS_THREADS = 256;
constexpr int SS_S = 8;             // history frames per thread
constexpr int SS_CHUNK = 1024;
constexpr int SS_Z = 8;
__global__ void __launch_bounds__(SS_THREADS) k_stream_sparse_col(StreamParams p) {
  __shared__ int32_t sc[SS_CHUNK];
  __shared__ uint32_t sv[SS_CHUNK];
  const int r = blockIdx.y;
  const int koff = p.ring_koff[r];
  const int n = p.nz_n[r];
  const int zb = static_cast<int>((static_cast<int64_t>(n) * blockIdx.z) / SS_Z);
  const int ze = static_cast<int>((static_cast<int64_t>(n) * (blockIdx.z + 1)) / SS_Z);
  const int64_t s0 = static_cast<int64_t>(blockIdx.x) * (SS_S * SS_THREADS) + SS_S * threadIdx.x;
  uint32_t acc[SS_S];
#pragma unroll
  for (int j = 0; j < SS_S; ++j) acc[j] = 0;
  for (int c0 = zb; c0 < ze; c0 += SS_CHUNK) {
    const int cn = ze - c0 < SS_CHUNK ? ze - c0 : SS_CHUNK;
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += SS_THREADS) {
      sc[i] = p.nz_col[koff + c0 + i];
      sv[i] = p.nz_val[koff + c0 + i];
    }
    __syncthreads();
    if (s0 <= p.t) {
      const uint8_t* h = p.hist + s0;
      // latency-bound on the scattered history rows: keep 16 loads in flight
#pragma unroll 16
      for (int i = 0; i < cn; ++i) {
        const uint2 w = __ldcs(reinterpret_cast<const uint2*>(h + static_cast<int64_t>(sc[i]) * p.hp));
        const uint32_t v = sv[i];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[j] += v * ((w.x >> (8 * j)) & 0xFFu);
          acc[4 + j] += v * ((w.y >> (8 * j)) & 0xFFu);
        }
      }
    }
  }
  if (s0 > p.t) return;
  int32_t* col = p.colbuf + static_cast<int64_t>(r) * p.hp + s0;
#pragma unroll
  for (int j = 0; j < SS_S; ++j)
    if (acc[j] && s0 + j <= p.t) atomicAdd(col + j, static_cast<int>(acc[j]));
}

// K5s-c: the finished column -> C, g2 lag sums and the optional stored column
// (the dense K5's expressions, so equal bitwise); resets colbuf and nz_n.
__global__ void __launch_bounds__(256) k_stream_sparse_fin(StreamParams p) {
  const int r = blockIdx.y;
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.nz_reset == 1) p.nz_n[r] = 0;
  if (s > p.t) return;
  int32_t* col = p.colbuf + static_cast<int64_t>(r) * p.hp + s;
  const int acc = *col;
  *col = 0;
  const double inv_t = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  const double inv_s = p.inv[static_cast<int64_t>(r) * p.inv_ld + s];
  const int64_t gi = static_cast<int64_t>(r) * p.g2_ld + (p.t - s);
  p.g2sum[gi] += static_cast<double>(acc) * (inv_s * inv_t);
  p.g2cnt[gi] += (inv_s != 0.0 && inv_t != 0.0) ? 1 : 0;
  if (p.gcol) p.gcol[static_cast<int64_t>(r) * p.col_ring_stride + s * p.col_ld + p.t] = acc;
}

cudaError_t launch_stream_ingest(const StreamParams& p, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((p.ktot / 128 + 3) / 4);
  k_stream_ingest<<<blocks, 128, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_stream_sparse(const StreamParams& p, int32_t n_rings, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((p.t + 1 + SS_S * SS_THREADS - 1) / (SS_S * SS_THREADS)),
            n_rings, SS_Z);
  k_stream_sparse_col<<<grid, SS_THREADS, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2(static_cast<unsigned>((p.t + 1 + 255) / 256), n_rings);
  k_stream_sparse_fin<<<g2, 256, 0, s>>>(p);
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

cudaError_t launch_stream_cmp(const StreamParams& p, int32_t n_rings, cudaStream_t s) {
  k_stream_proj_acc<<<dim3(n_rings, PZ), 256, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_stream_proj_fin<<<n_rings, 128, 0, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((p.t + 1 + SR_ROWS - 1) / SR_ROWS), n_rings);
  k_stream_cmp<<<grid, SR_THREADS, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace xg
