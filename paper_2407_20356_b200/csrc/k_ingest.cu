// k_ingest.cu -- K1: detector frames -> ring-major u8 layout + statistics.
//
// Replaces the per-ring column gather `apply_mask` (src/model.cpp:42-59) and
// the norm pass of `row_normalize` (src/linalg.cpp:441-456, the dot at :445):
// one pass over the raw frames writes every q-ring's pixels (in mask order,
// i.e. ascending pixel index) into its own 16-byte aligned column range of a
// frame-major row, and accumulates per (frame, ring) the exact sum of squares
// (|x_t|^2, integer), the sum and the max count.
//
// HBM-bound: reads M bytes and writes ~M bytes per frame.  A CTA owns one
// detector band (8192 pixels) and loops over frames: the band is staged in
// shared memory with 16-byte loads, its gather table (u16 source offset per
// output byte, padding = 0xFFFF) stays resident in shared memory, and each
// warp emits whole ring segments with coalesced 4-byte-per-lane stores, so
// the per-(frame, ring) statistics need one warp reduction per segment.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

constexpr int INGEST_THREADS = 256;

__device__ __forceinline__ uint32_t pick(const uint8_t* band, uint32_t e) {
  return e == 0xFFFFu ? 0u : static_cast<uint32_t>(band[e]);
}

__global__ void __launch_bounds__(INGEST_THREADS)
    k_ingest(IngestParams p) {
  extern __shared__ uint4 ismem[];
  const int b = blockIdx.x;
  uint8_t* band = reinterpret_cast<uint8_t*>(ismem);
  uint16_t* tab = reinterpret_cast<uint16_t*>(band + ((p.band + 15) & ~15));

  const int tab0 = p.band_tab[b];
  const int ntab = p.band_tab[b + 1] - tab0;
  for (int i = threadIdx.x; i < ntab; i += blockDim.x) tab[i] = p.tab[tab0 + i];

  const int seg0 = p.band_seg[b];
  const int nseg = p.band_seg[b + 1] - seg0;
  const int64_t pix0 = static_cast<int64_t>(b) * p.band;
  const int64_t blen = (p.pixels - pix0) < p.band ? (p.pixels - pix0) : p.band;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;

  const int64_t f_begin = static_cast<int64_t>(blockIdx.y) * p.frames_per_cta;
  int64_t f_end = f_begin + p.frames_per_cta;
  if (f_end > p.n_frames) f_end = p.n_frames;

  for (int64_t f = f_begin; f < f_end; ++f) {
    __syncthreads();  // previous frame fully consumed (and table loaded)
    const uint8_t* src = p.raster + f * p.pixels + pix0;
    if (((reinterpret_cast<uintptr_t>(src) | blen) & 15) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* d4 = reinterpret_cast<uint4*>(band);
      for (int i = threadIdx.x; i < blen / 16; i += blockDim.x) d4[i] = __ldcs(s4 + i);
    } else {
      for (int i = threadIdx.x; i < blen; i += blockDim.x) band[i] = src[i];
    }
    __syncthreads();

    const int64_t t = p.t0 + f;
    uint8_t* xrow = p.x + t * p.ktot;
    for (int s = warp; s < nseg; s += nwarps) {
      const Segment sg = p.segs[seg0 + s];
      const uint16_t* st = tab + sg.taboff;
      uint32_t sq = 0, sm = 0, mx = 0;
      for (int off = lane * 4; off < sg.len; off += 128) {
        const uint2 e = *reinterpret_cast<const uint2*>(st + off);
        const uint32_t v0 = pick(band, e.x & 0xFFFFu), v1 = pick(band, e.x >> 16);
        const uint32_t v2 = pick(band, e.y & 0xFFFFu), v3 = pick(band, e.y >> 16);
        *reinterpret_cast<uint32_t*>(xrow + sg.dst + off) = v0 | (v1 << 8) | (v2 << 16) | (v3 << 24);
        sq += v0 * v0 + v1 * v1 + v2 * v2 + v3 * v3;
        sm += v0 + v1 + v2 + v3;
        mx = max(max(mx, max(v0, v1)), max(v2, v3));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane == 0 && sm != 0) {
        const int64_t k = t * p.n_rings + sg.ring;
        atomicAdd(reinterpret_cast<unsigned long long*>(p.norm2 + k), sq);
        atomicAdd(reinterpret_cast<unsigned long long*>(p.sum1 + k), sm);
        atomicMax(p.maxc + k, static_cast<int>(mx));
      }
    }
  }
}

__global__ void k_norms(NormParams p) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (t >= p.n_frames) return;
  const int64_t n2 = p.norm2[t * p.n_rings + r];
  const double nrm = sqrt(static_cast<double>(n2));
  p.norms[r * p.ld + t] = nrm;
  p.inv[r * p.ld + t] = n2 > 0 ? 1.0 / nrm : 0.0;
  if (n2 == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p.zero_count + r), 1ull);
    atomicMin(reinterpret_cast<long long*>(p.first_zero + r), static_cast<long long>(t));
  }
  if (n2 >= (1ll << 31)) atomicOr(p.err, 4);
}

}  // namespace

cudaError_t launch_ingest(const IngestParams& p, cudaStream_t s) {
  const size_t smem = ((p.band + 15) & ~15) + static_cast<size_t>(p.max_tab) * 2 + 16;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_ingest, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t groups = (p.n_frames + p.frames_per_cta - 1) / p.frames_per_cta;
  dim3 grid(p.n_bands, static_cast<unsigned>(groups));
  k_ingest<<<grid, INGEST_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_norms(const NormParams& p, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((p.n_frames + 255) / 256), p.n_rings);
  k_norms<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace xg
