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
#ifndef XG_NBUF
#define XG_NBUF 4
#endif
#ifndef XG_CPASYNC
#define XG_CPASYNC 0
#endif
#ifndef XG_EXP
#define XG_EXP 0
#endif
constexpr int NBUF = XG_NBUF;  // frames in flight per CTA
#ifndef XG_PIECE
#define XG_PIECE 512
#endif
constexpr int PIECE = XG_PIECE;   // band bytes per bulk copy
constexpr int PITCH = XG_PIECE + 16;   // smem pitch of a piece: +16 B skews consecutive
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
  // Group table: 8 bytes per 4 output bytes.  A ring's pixels arrive as runs
  // of consecutive detector pixels (one per row crossing), so a group's bytes
  // come from at most two runs A, B in the common case; each run is fetched
  // as two aligned smem words + a funnel shift and a byte permute merges them:
  //   x = word offset of A | word offset of B << 16
  //   y = 8*(A mod 4) | 8*(B mod 4) << 8 | permute selector << 16
  // (B = A for single-run groups).  Groups touching three or more runs (rings
  // thinner than 4 px) hold the four byte offsets and bit 31 of y set.
  uint2* gtab = reinterpret_cast<uint2*>(bufs + NBUF * bstride);
  const int tab0 = p.band_tab[b];
  const int ntab = p.band_tab[b + 1] - tab0;
  const int zero_at = bstride - 16;
  auto smap = [&](uint32_t e) -> uint32_t {
    return e == 0xFFFFu ? static_cast<uint32_t>(zero_at) : e + 16u * (e / PIECE);
  };
  for (int g = threadIdx.x; g < ntab / 4; g += blockDim.x) {
    const uint2 raw = *reinterpret_cast<const uint2*>(p.tab + tab0 + 4 * g);
    const uint32_t s0 = smap(raw.x & 0xFFFFu), s1 = smap(raw.x >> 16);
    const uint32_t s2 = smap(raw.y & 0xFFFFu), s3 = smap(raw.y >> 16);
    const bool c1 = s1 == s0 + 1, c2 = c1 && s2 == s0 + 2, c3 = c2 && s3 == s0 + 3;
    const uint32_t na = 1 + c1 + c2 + c3;
    const uint32_t sb = na == 1 ? s1 : na == 2 ? s2 : na == 3 ? s3 : s0;
    const bool ok = na == 1 ? (s2 == s1 + 1 && s3 == s1 + 2) : na == 2 ? s3 == s2 + 1 : true;
    uint2 ent;
    if (ok) {
      uint32_t sel = 0;
      for (uint32_t j = 0; j < 4; ++j) sel |= (j < na ? j : 4 + j - na) << (4 * j);
      ent.x = (s0 & ~3u) | ((sb & ~3u) << 16);
      ent.y = 8 * (s0 & 3u) | (8 * (sb & 3u)) << 8 | sel << 16;
    } else {
      ent.x = s0 | (s1 << 16);
      ent.y = s2 | (s3 << 16) | 0x80000000u;
    }
    gtab[g] = ent;
  }
  if (threadIdx.x < NBUF * 4)
    reinterpret_cast<uint32_t*>(bufs + (threadIdx.x >> 2) * bstride + zero_at)[threadIdx.x & 3] = 0;
  // the band's segment descriptors in consumer-warp order (seg_order)
  const int seg0 = p.band_seg[b];
  const int wb = p.band_wseg[b * (CONSUMERS + 1)];
  int4* sdesc = reinterpret_cast<int4*>(gtab + ((p.max_tab / 4 + 1) & ~1));
  for (int i = threadIdx.x; i < p.band_wseg[b * (CONSUMERS + 1) + CONSUMERS] - wb;
       i += blockDim.x) {
    const Segment sg = p.segs[seg0 + p.seg_order[wb + i]];
    sdesc[i] = make_int4(sg.ring, sg.dst, sg.len / 4, sg.taboff / 4);
  }
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
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&full[i])),
                   "r"(XG_CPASYNC ? 32 : 1));
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
          "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, 1000000;\n\t"
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
      if (XG_CPASYNC && bulk) {
        for (int o = lane * 16; o < blen; o += 512)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           smem_addr(dst + o + 16 * (o / PIECE))),
                       "l"(src + o)
                       : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         smem_addr(&full[slot]))
                     : "memory");
      } else if (bulk) {
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
    unsigned long long* nrow = p.norm2 + t * p.n_rings;
    for (int w = w0; w < (XG_EXP == 2 ? w0 : w1); ++w) {
      const int4 sg = sdesc[w - wb];  // {ring, dst, groups, group offset}
      const uint2* gt = gtab + sg.w;
      uint32_t* out = reinterpret_cast<uint32_t*>(
          xrow + (XG_EXP == 3 ? static_cast<int64_t>(b) * p.band + 4 * sg.w
                 : XG_EXP == 5 ? static_cast<int64_t>(b) * p.band + ((4 * sg.w) & ~127) : sg.y));
      uint32_t sq = 0;
      // 4 output bytes per lane, a warp covers 128 consecutive output bytes
      for (int g = lane; g < sg.z; g += 32) {
        const uint2 e = gt[g];
        uint32_t word;
        if (XG_EXP == 1 || XG_EXP == 3 || XG_EXP == 5) {
          word = *reinterpret_cast<const uint32_t*>(band + ((4 * g) & 8191));
        } else if (!(e.y & 0x80000000u)) {
          const uint8_t* pa = band + (e.x & 0xFFFFu);
          const uint8_t* pb = band + (e.x >> 16);
          const uint32_t wa = __funnelshift_r(*reinterpret_cast<const uint32_t*>(pa),
                                              *reinterpret_cast<const uint32_t*>(pa + 4), e.y);
          const uint32_t wb = __funnelshift_r(*reinterpret_cast<const uint32_t*>(pb),
                                              *reinterpret_cast<const uint32_t*>(pb + 4), e.y >> 8);
          word = __byte_perm(wa, wb, e.y >> 16);
        } else {
          const uint32_t v0 = band[e.x & 0xFFFFu], v1 = band[e.x >> 16];
          const uint32_t v2 = band[e.y & 0xFFFFu], v3 = band[(e.y >> 16) & 0x7FFFu];
          word = __byte_perm(v0 | (v1 << 8), v2 | (v3 << 8), 0x5410);
        }
        out[g] = word;
        sq = __dp4a(word, word, sq);
      }
      // exact: integer sums, any order (a piece's sum is < 2^32)
      sq = __reduce_add_sync(0xffffffffu, sq);
      if (lane == 0) atomicAdd(nrow + sg.x, static_cast<unsigned long long>(sq));
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[slot]))
                   : "memory");
  }
}

// Per (frame, ring): norms, inverse norms, zero-frame bookkeeping.
__global__ void k_norms(NormParams p) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const bool valid = i < p.n_frames;
  const int64_t t = p.t0 + i;
  const int64_t n2 = valid ? p.norm2[t * p.n_rings + r] : 0;
  if (valid) {
    const double nrm = sqrt(static_cast<double>(n2));
    p.norms[r * p.ld + t] = nrm;
    p.inv[r * p.ld + t] = n2 > 0 ? 1.0 / nrm : 0.0;
  }
  // warp-aggregated bookkeeping: one atomic per warp, not per frame
  const uint32_t nz = __ballot_sync(0xffffffffu, valid && n2 > 0);
  const uint32_t zero = __ballot_sync(0xffffffffu, valid && n2 == 0);
  const uint32_t ovf = __ballot_sync(0xffffffffu, n2 >= (1ll << 31));
  unsigned long long mx = static_cast<unsigned long long>(n2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = v > mx ? v : mx;
  }
  const int64_t tw = t - lane;  // frame of lane 0
  uint32_t* words = p.nz_bits + static_cast<int64_t>(r) * p.nz_words;
  if ((tw & 31) == 0) {
    if (lane == 0 && nz) atomicOr(words + (tw >> 5), nz);
  } else if (valid && n2 > 0) {
    atomicOr(words + (t >> 5), 1u << (t & 31));
  }
  if (lane == 0) {
    if (zero) {
      atomicAdd(reinterpret_cast<unsigned long long*>(p.zero_count + r),
                static_cast<unsigned long long>(__popc(zero)));
      atomicMin(reinterpret_cast<long long*>(p.first_zero + r),
                static_cast<long long>(tw + __ffs(zero) - 1));
    }
    if (ovf) atomicOr(p.err, 4);
    if (p.max_norm2) atomicMax(p.max_norm2, mx);
  }
}

}  // namespace

cudaError_t launch_ingest(const IngestParams& p, cudaStream_t s) {
  const size_t smem = NBUF * static_cast<size_t>(band_stride(p.band)) +
                      static_cast<size_t>((p.max_tab / 4 + 1) & ~1) * 8 +  // group table
                      static_cast<size_t>(p.max_band_segs) * 16 + 16;       // descriptors
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
