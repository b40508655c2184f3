// k_ingest.cu -- K1: detector frames -> ring-major u8 layout + statistics.
//
// Replaces the per-ring column gather `apply_mask` (src/model.cpp:42-59) and
// the norm pass of `row_normalize` (src/linalg.cpp:441-456, the dot at :445):
// one pass over the raw frames writes every q-ring's pixels (in mask order,
// i.e. ascending pixel index) into its own 4-byte aligned column range of a
// frame-major row, and records per (frame, segment) the exact sum of squares
// and sum of the counts.  K1b (k_norms) folds segments into per-(frame, ring)
// norms in a fixed order -- no atomics anywhere, so the statistics are exact
// and deterministic.
//
// HBM-bound (reads M bytes, writes ~M bytes per frame).  A CTA owns one
// detector band (8192 pixels) and a run of frames: band bytes are
// streamed into a 4-deep ring of shared-memory buffers by TMA bulk copies
// (cp.async.bulk + mbarrier: 4 frames in flight per CTA), the band's gather table (u16 source offset
// per output byte, 0xFFFF = zero padding) stays resident in shared memory,
// and each warp emits whole ring segments, 4 output bytes per lane per step,
// as coalesced 128-byte warp stores.  Band pieces of 512 B sit at a 528 B
// smem pitch so consecutive detector rows do not alias to the same banks.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

constexpr int INGEST_THREADS = 256;
constexpr int NBUF = 4;      // frames in flight per CTA
constexpr int PIECE = 512;   // band bytes per bulk copy
constexpr int PITCH = 528;   // smem pitch of a piece: +16 B skews consecutive
                             // 512-byte detector rows by 4 banks

__host__ __device__ constexpr int band_stride(int band) {
  return ((band + PIECE - 1) / PIECE) * PITCH + 16;  // + 16 zero bytes (padding source)
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Warp roles: warps 0..7 consume (each owns a fixed, length-balanced set of
// the band's segments, assigned on the host by LPT), warp 8 produces (one
// lane issues the TMA bulk copies).  full/empty mbarriers per ring slot let
// the consumer warps run up to NBUF frames apart, so per-frame imbalance
// between warps averages out instead of stalling at a block barrier.
constexpr int CONSUMERS = 8;

__global__ void __launch_bounds__(INGEST_THREADS + 32)
    k_ingest(IngestParams p) {
  extern __shared__ uint4 ismem[];
  __shared__ __align__(8) uint64_t full[NBUF];
  __shared__ __align__(8) uint64_t empty[NBUF];
  const int b = blockIdx.x;
  // band buffer: pieces of 512 B at a 528 B pitch, then 16 zero bytes that
  // the padding entries of the table point to
  const int bstride = band_stride(p.band);
  uint8_t* bufs = reinterpret_cast<uint8_t*>(ismem);  // NBUF x bstride
  uint16_t* tab = reinterpret_cast<uint16_t*>(bufs + NBUF * bstride);
  const int tab0 = p.band_tab[b];
  const int ntab = p.band_tab[b + 1] - tab0;
  // group table: one word per 4 output bytes -- the smem source offset when
  // the 4 sources are consecutive (fetched as two aligned words + a funnel
  // shift), else 0x80000000 (per-byte gather through `tab`)
  uint32_t* gtab = reinterpret_cast<uint32_t*>(tab + ((ntab + 7) & ~7));

  const int zero_at = bstride - 16;
  for (int i = threadIdx.x; i < ntab; i += blockDim.x) {
    const uint32_t e = p.tab[tab0 + i];
    tab[i] = static_cast<uint16_t>(e == 0xFFFFu ? zero_at : e + 16u * (e / PIECE));
  }
  if (threadIdx.x < NBUF * 4)
    reinterpret_cast<uint32_t*>(bufs + (threadIdx.x >> 2) * bstride + zero_at)[threadIdx.x & 3] = 0;
  __syncthreads();
  for (int g = threadIdx.x; g < ntab / 4; g += blockDim.x) {
    const uint32_t e0 = tab[4 * g], e1 = tab[4 * g + 1], e2 = tab[4 * g + 2], e3 = tab[4 * g + 3];
    gtab[g] = (e1 == e0 + 1 && e2 == e0 + 2 && e3 == e0 + 3) ? e0 : 0x80000000u;
  }

  const int seg0 = p.band_seg[b];
  const int64_t pix0 = static_cast<int64_t>(b) * p.band;
  const int blen = static_cast<int>((p.pixels - pix0) < p.band ? (p.pixels - pix0) : p.band);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool bulk = ((p.pixels | blen) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(p.raster) & 15) == 0;

  const int64_t f_begin = static_cast<int64_t>(blockIdx.y) * p.frames_per_cta;
  int64_t f_end = f_begin + p.frames_per_cta;
  if (f_end > p.n_frames) f_end = p.n_frames;
  if (f_begin >= f_end) return;
  const int64_t nf = f_end - f_begin;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&empty[i])),
                   "r"(CONSUMERS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // barriers, table and zero bytes visible

  auto wait = [](uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred P;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, P;\n\t}"
          : "=r"(ok)
          : "r"(smem_addr(bar)), "r"(parity)
          : "memory");
    }
  };

  if (warp == CONSUMERS) {
    // ------------------------------------------------------------ producer
    for (int64_t i = 0; i < nf; ++i) {
      const int slot = static_cast<int>(i % NBUF);
      const int64_t use = i / NBUF;
      if (use > 0) wait(&empty[slot], static_cast<uint32_t>((use - 1) & 1));
      uint8_t* dst = bufs + slot * bstride;
      const uint8_t* src = p.raster + (f_begin + i) * p.pixels + pix0;
      if (bulk) {
        if (lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                           smem_addr(&full[slot])),
                       "r"(blen)
                       : "memory");
          for (int o = 0; o < blen; o += PIECE) {
            const int len = blen - o < PIECE ? blen - o : PIECE;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                "%2, [%3];" ::"r"(smem_addr(dst + (o / PIECE) * PITCH)),
                "l"(src + o), "r"(len), "r"(smem_addr(&full[slot]))
                : "memory");
          }
        }
      } else {
        for (int k = lane; k < blen; k += 32) dst[k + 16 * (k / PIECE)] = src[k];
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&full[slot]))
                       : "memory");
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int w0 = p.band_wseg[b * (CONSUMERS + 1) + warp];
  const int w1 = p.band_wseg[b * (CONSUMERS + 1) + warp + 1];
  for (int64_t i = 0; i < nf; ++i) {
    const int slot = static_cast<int>(i % NBUF);
    wait(&full[slot], static_cast<uint32_t>((i / NBUF) & 1));
    const uint8_t* band = bufs + slot * bstride;
    const int64_t t = p.t0 + f_begin + i;
    uint8_t* xrow = p.x + t * p.ktot;
    uint2* srow = p.seg_stats + t * p.n_segs + seg0;
    for (int w = w0; w < w1; ++w) {
      const int sidx = p.seg_order[w];  // segment index within the band
      const Segment sg = p.segs[seg0 + sidx];
      const uint16_t* st = tab + sg.taboff;
      const uint32_t* gt = gtab + sg.taboff / 4;
      const uint32_t* band32 = reinterpret_cast<const uint32_t*>(band);
      uint32_t sq = 0, sm = 0;
      // 4 output bytes per lane, a warp covers 128 consecutive output bytes
      for (int off = lane * 4; off < sg.len; off += 128) {
        const uint32_t e = gt[off >> 2];
        uint32_t word;
        if (!(e & 0x80000000u)) {  // consecutive sources: 2 aligned words
          const uint32_t lo = band32[e >> 2], hi = band32[(e >> 2) + 1];
          word = __funnelshift_r(lo, hi, (e & 3u) * 8u);
        } else {                   // run boundary / padding: byte gather
          const uint2 ee = *reinterpret_cast<const uint2*>(st + off);
          const uint32_t v0 = band[ee.x & 0xFFFFu], v1 = band[ee.x >> 16];
          const uint32_t v2 = band[ee.y & 0xFFFFu], v3 = band[ee.y >> 16];
          word = __byte_perm(v0 | (v1 << 8), v2 | (v3 << 8), 0x5410);
        }
        *reinterpret_cast<uint32_t*>(xrow + sg.dst + off) = word;
        sq = __dp4a(word, word, sq);
        sm = __dp4a(word, 0x01010101u, sm);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
      }
      if (lane == 0) srow[sidx] = make_uint2(sq, sm);
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[slot]))
                   : "memory");
  }
}

// Per (frame, ring): fold the ring's segments in ascending band order.
__global__ void k_norms(NormParams p) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (i >= p.n_frames) return;
  const int64_t t = p.t0 + i;
  const uint2* srow = p.seg_stats + t * p.n_segs;
  int64_t n2 = 0, s1 = 0;
  for (int i = p.ring_seg_begin[r]; i < p.ring_seg_begin[r + 1]; ++i) {
    const uint2 v = srow[p.ring_seg_list[i]];
    n2 += v.x;
    s1 += v.y;
  }
  p.norm2[t * p.n_rings + r] = n2;
  p.sum1[t * p.n_rings + r] = s1;
  const double nrm = sqrt(static_cast<double>(n2));
  p.norms[r * p.ld + t] = nrm;
  p.inv[r * p.ld + t] = n2 > 0 ? 1.0 / nrm : 0.0;
  if (n2 > 0) atomicOr(p.nz_bits + static_cast<int64_t>(r) * p.nz_words + (t >> 5), 1u << (t & 31));
  if (n2 == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p.zero_count + r), 1ull);
    atomicMin(reinterpret_cast<long long*>(p.first_zero + r), static_cast<long long>(t));
  }
  if (n2 >= (1ll << 31)) atomicOr(p.err, 4);
  if (p.max_norm2) atomicMax(p.max_norm2, static_cast<unsigned long long>(n2));
}

}  // namespace

cudaError_t launch_ingest(const IngestParams& p, cudaStream_t s) {
  const size_t smem = NBUF * static_cast<size_t>(band_stride(p.band)) +
                      static_cast<size_t>((p.max_tab + 7) & ~7) * 2 +
                      static_cast<size_t>(p.max_tab) + 16;  // byte table + group table
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_ingest, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t groups = (p.n_frames + p.frames_per_cta - 1) / p.frames_per_cta;
  dim3 grid(p.n_bands, static_cast<unsigned>(groups));
  k_ingest<<<grid, INGEST_THREADS + 32, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_norms(const NormParams& p, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((p.n_frames + 255) / 256), p.n_rings);
  k_norms<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace xg
