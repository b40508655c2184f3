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
//   K6a proj: y_t = (x_t/|x_t|) V from the NONZERO pixels of the new frame
//             only (the reference's project_row skips zeros too,
//             compress.cpp:17) against a pixel-major copy of the int8 basis
//             digits; the f64 combination is the same expression as the
//             batch projection (k_project.cu), so streamed coefficients equal
//             batch coefficients bitwise.
//   K6b cmp:  C~(s,t) = y_s . y_t (f64) for s <= t over the coefficient
//             history, g2 accumulated like K5.  HBM-bound: t * Q * k * 8 B.
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

// K6a: one CTA per ring; threads own (digit, coefficient) accumulators.
__global__ void __launch_bounds__(512) k_stream_project(StreamParams p) {
  __shared__ int32_t nz_col[1024];
  __shared__ int32_t nz_val[1024];
  __shared__ int nz_count;
  __shared__ int32_t accs[3 * 256];
  const int r = blockIdx.x;
  const int64_t koff = p.ring_koff[r];
  const int64_t kpad = static_cast<int64_t>(p.ring_nkb[r]) * 128;
  const int nacc = p.n_digits * p.k;  // <= 768
  const uint8_t* xrow = p.x + p.t * p.ktot + koff;
  int32_t acc0 = 0, acc1 = 0;  // thread owns entries tid and tid + blockDim
  for (int64_t c0 = 0; c0 < kpad; c0 += 1024) {  // <= 1024 nonzeros per chunk
    if (threadIdx.x == 0) nz_count = 0;
    __syncthreads();
    // compact the nonzero pixels of this chunk (16 bytes per thread step)
    for (int64_t v = c0 / 16 + threadIdx.x; v < (c0 + 1024) / 16 && v < kpad / 16;
         v += blockDim.x) {
      const uint4 w = reinterpret_cast<const uint4*>(xrow)[v];
      if ((w.x | w.y | w.z | w.w) == 0u) continue;
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      for (int b = 0; b < 16; ++b) {
        const uint32_t val = (ws[b >> 2] >> (8 * (b & 3))) & 0xFFu;
        if (val) {
          const int slot = atomicAdd(&nz_count, 1);
          nz_col[slot] = static_cast<int32_t>(v * 16 + b);
          nz_val[slot] = static_cast<int32_t>(val);
        }
      }
    }
    __syncthreads();
    const int n = nz_count;
    // integer accumulation: order-free, exact
    for (int e = 0; e < n; ++e) {
      const int8_t* vd = p.vdt + (koff + nz_col[e]) * static_cast<int64_t>(p.vdt_ld);
      const int xv = nz_val[e];
      if (static_cast<int>(threadIdx.x) < nacc) acc0 += xv * vd[threadIdx.x];
      if (static_cast<int>(threadIdx.x + blockDim.x) < nacc) acc1 += xv * vd[threadIdx.x + blockDim.x];
    }
    __syncthreads();
  }
  if (static_cast<int>(threadIdx.x) < nacc) accs[threadIdx.x] = acc0;
  if (static_cast<int>(threadIdx.x + blockDim.x) < nacc) accs[threadIdx.x + blockDim.x] = acc1;
  __syncthreads();
  const double inv = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  for (int j = threadIdx.x; j < p.k; j += blockDim.x) {
    // same f64 expression as k_project's epilogue (bitwise-equal coefficients)
    p.y[(static_cast<int64_t>(r) * p.y_ld + p.t) * p.k + j] = combine_digits(
        accs[j], p.n_digits > 1 ? accs[p.k + j] : 0, p.n_digits > 2 ? accs[2 * p.k + j] : 0,
        p.n_digits, p.scale[static_cast<int64_t>(r) * p.k + j], inv);
  }
}

// K6b: grid (ceil((t+1)/SR_ROWS), rings); a warp per history row.
__global__ void __launch_bounds__(SR_THREADS) k_stream_cmp(StreamParams p) {
  __shared__ double yt[1024];
  const int r = blockIdx.y;
  const double* ybase = p.y + static_cast<int64_t>(r) * p.y_ld * p.k;
  for (int j = threadIdx.x; j < p.k; j += blockDim.x) yt[j] = ybase[p.t * p.k + j];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double inv_t = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  const int64_t s_begin = static_cast<int64_t>(blockIdx.x) * SR_ROWS;
  for (int64_t s = s_begin + warp; s < s_begin + SR_ROWS && s <= p.t; s += SR_THREADS / 32) {
    const double* ys = ybase + s * p.k;
    double acc = 0.0;
    for (int j = lane; j < p.k; j += 32) acc = fma(__ldcs(ys + j), yt[j], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const double inv_s = p.inv[static_cast<int64_t>(r) * p.inv_ld + s];
      const int64_t gi = static_cast<int64_t>(r) * p.g2_ld + (p.t - s);
      p.cg2sum[gi] += acc;
      p.cg2cnt[gi] += (inv_s != 0.0 && inv_t != 0.0) ? 1 : 0;
      if (p.ccol) p.ccol[static_cast<int64_t>(r) * p.col_ring_stride + s * p.col_ld + p.t] =
          static_cast<float>(acc);
    }
  }
}

}  // namespace

// K5s-a: one CTA per ring.  The new frame's nonzero ring columns (any order:
// the column sums below are integer, so order-free) and their scatter into
// the pixel-major history.
__global__ void __launch_bounds__(512) k_stream_sparse_gather(StreamParams p) {
  __shared__ int cnt;
  const int r = blockIdx.x;
  const int koff = p.ring_koff[r];
  const int n = p.ring_nkb[r] * 128;
  const uint8_t* row = p.x + p.t * p.ktot + koff;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int i0 = 0; i0 < n; i0 += 4 * blockDim.x) {
    const int i = i0 + 4 * threadIdx.x;
    const uint32_t w = i < n ? *reinterpret_cast<const uint32_t*>(row + i) : 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t v = (w >> (8 * j)) & 0xFFu;
      const uint32_t m = __ballot_sync(0xffffffffu, v != 0u);
      int base = 0;
      if (lane == 0 && m) base = atomicAdd(&cnt, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (v) {
        const int pos = base + __popc(m & ((1u << lane) - 1u));
        const int c = koff + i + j;
        p.nz_col[koff + pos] = c;
        p.nz_val[koff + pos] = static_cast<uint8_t>(v);
        p.hist[static_cast<int64_t>(c) * p.hp + p.t] = static_cast<uint8_t>(v);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) p.nz_n[r] = cnt;
}

// K5s-b: grid (ceil((t+1)/1024), rings); a thread owns 4 consecutive history
// frames s and walks the ring's nonzeros: one coalesced 32-bit load of
// hist[c][s..s+3] per nonzero.  Same C, g2 and column outputs as K5.
constexpr int SS_THREADS = 256;
constexpr int SS_CHUNK = 1024;
__global__ void __launch_bounds__(SS_THREADS) k_stream_sparse_col(StreamParams p) {
  __shared__ int32_t sc[SS_CHUNK];
  __shared__ uint32_t sv[SS_CHUNK];
  const int r = blockIdx.y;
  const int koff = p.ring_koff[r];
  const int n = p.nz_n[r];
  const int64_t s0 = static_cast<int64_t>(blockIdx.x) * (4 * SS_THREADS) + 4 * threadIdx.x;
  uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int c0 = 0; c0 < n; c0 += SS_CHUNK) {
    const int cn = n - c0 < SS_CHUNK ? n - c0 : SS_CHUNK;
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += SS_THREADS) {
      sc[i] = p.nz_col[koff + c0 + i];
      sv[i] = p.nz_val[koff + c0 + i];
    }
    __syncthreads();
    if (s0 <= p.t) {
      const uint8_t* h = p.hist + s0;
#pragma unroll 4
      for (int i = 0; i < cn; ++i) {
        const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(h + static_cast<int64_t>(sc[i]) * p.hp));
        const uint32_t v = sv[i];
        acc0 += v * (w & 0xFFu);
        acc1 += v * ((w >> 8) & 0xFFu);
        acc2 += v * ((w >> 16) & 0xFFu);
        acc3 += v * (w >> 24);
      }
    }
  }
  const double inv_t = p.inv[static_cast<int64_t>(r) * p.inv_ld + p.t];
  const uint32_t acc[4] = {acc0, acc1, acc2, acc3};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t s = s0 + j;
    if (s > p.t) break;
    const double inv_s = p.inv[static_cast<int64_t>(r) * p.inv_ld + s];
    const int64_t gi = static_cast<int64_t>(r) * p.g2_ld + (p.t - s);
    p.g2sum[gi] += static_cast<double>(static_cast<int>(acc[j])) * (inv_s * inv_t);
    p.g2cnt[gi] += (inv_s != 0.0 && inv_t != 0.0) ? 1 : 0;
    if (p.gcol) p.gcol[static_cast<int64_t>(r) * p.col_ring_stride + s * p.col_ld + p.t] =
        static_cast<int>(acc[j]);
  }
}

cudaError_t launch_stream_sparse(const StreamParams& p, int32_t n_rings, cudaStream_t s) {
  k_stream_sparse_gather<<<n_rings, 512, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((p.t + 1 + 4 * SS_THREADS - 1) / (4 * SS_THREADS)), n_rings);
  k_stream_sparse_col<<<grid, SS_THREADS, 0, s>>>(p);
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
  k_stream_project<<<n_rings, 512, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((p.t + 1 + SR_ROWS - 1) / SR_ROWS), n_rings);
  k_stream_cmp<<<grid, SR_THREADS, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace xg
