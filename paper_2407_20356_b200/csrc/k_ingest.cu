// k_ingest.cu -- K1: detector frames -> ring-major u8 layout + statistics.
//
// Replaces the per-ring column gather `apply_mask` (src/model.cpp:42-59) and
// the norm pass of `row_normalize` (src/linalg.cpp:441-456, the dot at :445):
// one pass over the raw frames writes every q-ring's pixels into its own
// column range of a frame-major row and accumulates the exact |x|^2 of every
// (frame, ring).  K1b (k_norms) turns those into norms, 1/|x| (f64 and its
// (hi, lo) float split for the FP32 fused g2) and the zero-frame bookkeeping.
//
// HBM-bound (reads M bytes, writes ~M bytes per frame).  A CTA owns one
// detector band (16384 pixels) and a run of frames.  Warp 8 streams band
// bytes into a 4-deep ring of shared-memory buffers with TMA bulk copies
// (cp.async.bulk + full/empty mbarriers); 512-byte pieces sit at a 528-byte
// pitch so consecutive detector rows land 4 banks apart.  The band's output
// is a list of segments (one per ring), each = whole source words (all 4
// pixels in the ring; copied with one bank-conflict-free 32-bit load, the
// host orders them round-robin over banks) followed by the leftover pixels
// packed 4 per group (byte gather).  The host cuts every band into 8
// cost-balanced runs of "pieces" (segment fragments), one per consumer warp;
// each consumer pass serves two frames, so a table entry and the piece
// bookkeeping are paid once per two frames.  |x|^2 per piece: __dp4a + warp
// redux + an integer red.add into the (frame, ring) total (exact, order-free).
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

constexpr int INGEST_THREADS = 32 * INGEST_CONSUMERS;
constexpr int NBUF = 4;  // frames in flight per CTA (6 / 8: slower at C2 and C5, fewer CTAs per SM)
constexpr int FR = 2;    // frames per consumer pass (divides NBUF)
static_assert(NBUF % FR == 0, "NBUF must be a multiple of FR");
constexpr int PIECE = INGEST_PIECE, PITCH = INGEST_PITCH;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ void stg_u32(uint8_t* p, uint32_t v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Warp roles: warps 0..7 consume (each owns a cost-balanced run of the band's
// pieces, cut on the host), warp 8 produces (one lane issues the TMA bulk
// copies).  full/empty mbarriers per ring slot let the consumer warps run up
// to NBUF frames apart.
constexpr int CONSUMERS = INGEST_CONSUMERS;

__global__ void __launch_bounds__(INGEST_THREADS + 32)
    k_ingest(IngestParams p) {
  extern __shared__ uint4 ismem[];
  __shared__ __align__(8) uint64_t full[NBUF];
  __shared__ __align__(8) uint64_t empty[NBUF];
  const int b = blockIdx.x;
  const int bstride = ingest_band_stride(p.band);
  const int zero_at = bstride - 16;
  // shared memory: NBUF band buffers | word table | byte table | pieces
  uint8_t* bufs = reinterpret_cast<uint8_t*>(ismem);
  uint16_t* swords = reinterpret_cast<uint16_t*>(bufs + NBUF * bstride);
  uint2* sbytes = reinterpret_cast<uint2*>(swords + ((p.max_words + 7) & ~7));
  int4* spieces = reinterpret_cast<int4*>(sbytes + ((p.max_bytes + 1) & ~1));
  {
    const int w0 = p.band_word[b], nw = p.band_word[b + 1] - w0;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) swords[i] = p.words[w0 + i];
    const int g0 = p.band_byte[b], ng = p.band_byte[b + 1] - g0;
    for (int i = threadIdx.x; i < ng; i += blockDim.x)
      sbytes[i] = reinterpret_cast<const uint2*>(p.bytes)[g0 + i];
    const int pc0 = p.band_piece[b * (CONSUMERS + 1)];
    const int npc = p.band_piece[b * (CONSUMERS + 1) + CONSUMERS] - pc0;
    for (int i = threadIdx.x; i < 2 * npc; i += blockDim.x)
      spieces[i] = reinterpret_cast<const int4*>(p.pieces + pc0)[i];
  }
  if (threadIdx.x < NBUF * 4)
    reinterpret_cast<uint32_t*>(bufs + (threadIdx.x >> 2) * bstride + zero_at)[threadIdx.x & 3] = 0;

  // 1D band: pixels [pix0, pix0 + blen).  2D band: rows [y0, y0 + rows) x
  // columns [x0, x0 + bw) of a width-wide detector, pix0 = its first pixel,
  // one piece per row.
  const bool two_d = p.width > 0;
  int64_t pix0;
  int blen, rows = 0, bw = 0;
  if (two_d) {
    const int y0 = (b / p.blocks_x) * kBandH, x0 = (b % p.blocks_x) * kBandW;
    rows = min(kBandH, p.height - y0);
    bw = min(kBandW, p.width - x0);
    pix0 = static_cast<int64_t>(y0) * p.width + x0;
    blen = rows * bw;
  } else {
    pix0 = static_cast<int64_t>(b) * p.band;
    blen = static_cast<int>((p.pixels - pix0) < p.band ? (p.pixels - pix0) : p.band);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool bulk = ((two_d ? (p.width | bw) : (p.pixels | blen)) & 15) == 0 &&
                    (p.pixels & 15) == 0 && (reinterpret_cast<uintptr_t>(p.raster) & 15) == 0;

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
  __syncthreads();  // barriers, tables and zero bytes visible

  // waiting warps back off so they do not take issue slots from the copiers
  auto wait = [](uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    for (;;) {
      asm volatile(
          "{\n\t.reg .pred P;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, P;\n\t}"
          : "=r"(ok)
          : "r"(smem_addr(bar)), "r"(parity)
          : "memory");
      if (ok) break;
      __nanosleep(64);
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
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                           smem_addr(&full[slot])),
                       "r"(blen)
                       : "memory");
        __syncwarp();
        // one piece per lane: the band's bulk copies are issued in parallel
        if (two_d) {
          for (int rr = lane; rr < rows; rr += 32)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                "%2, [%3];" ::"r"(smem_addr(dst + rr * PITCH)),
                "l"(src + static_cast<int64_t>(rr) * p.width), "r"(bw),
                "r"(smem_addr(&full[slot]))
                : "memory");
        } else {
          for (int o = lane * PIECE; o < blen; o += 32 * PIECE) {
            const int len = blen - o < PIECE ? blen - o : PIECE;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                "%2, [%3];" ::"r"(smem_addr(dst + (o / PIECE) * PITCH)),
                "l"(src + o), "r"(len), "r"(smem_addr(&full[slot]))
                : "memory");
          }
        }
      } else if (two_d) {
        for (int k = lane; k < blen; k += 32) {
          const int rr = k / bw, cc = k % bw;
          dst[rr * PITCH + cc] = src[static_cast<int64_t>(rr) * p.width + cc];
        }
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&full[slot]))
                       : "memory");
      } else {
        for (int k = lane; k < blen; k += 32) dst[ingest_smem_offset(k)] = src[k];
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&full[slot]))
                       : "memory");
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int pc0 = p.band_piece[b * (CONSUMERS + 1)];
  const int k0 = p.band_piece[b * (CONSUMERS + 1) + warp] - pc0;
  const int k1 = p.band_piece[b * (CONSUMERS + 1) + warp + 1] - pc0;
  const uint32_t words_s = smem_addr(swords), bytes_s = smem_addr(sbytes);
  const uint32_t bufs_s = smem_addr(bufs);
  // FR frames per pass: a table entry is read once and serves FR frames, and
  // the per-piece bookkeeping is paid once per FR frames.
  for (int64_t i = 0; i < nf; i += FR) {
    const int slot = static_cast<int>(i % NBUF);  // FR consecutive slots
    const int nfr = nf - i < FR ? static_cast<int>(nf - i) : FR;
    uint32_t band_s[FR];
    int64_t xrow[FR];  // frame's row in x
    uint8_t* xbase[FR];  // interleaved rows: the frame's ring-major row
    unsigned long long* nrow[FR];
#pragma unroll
    for (int f = 0; f < FR; ++f) {
      const int ff = f < nfr ? f : 0;  // missing tail frames redo frame 0 (not stored)
      if (f < nfr) wait(&full[slot + f], static_cast<uint32_t>(((i + f) / NBUF) & 1));
      band_s[f] = bufs_s + (slot + ff) * bstride;
      const int64_t t = p.t0 + f_begin + i + ff;
      xrow[f] = t - p.x_row0;
      xbase[f] = p.x + xrow[f] * p.ktot;
      nrow[f] = p.norm2 + t * p.n_rings;
      asm volatile("" : "+l"(xrow[f]), "+l"(xbase[f]), "+l"(nrow[f]));  // once per frame
    }
    for (int k = k0; k < k1; ++k) {
      const int4 pa = spieces[2 * k], pb = spieces[2 * k + 1];  // see Piece
      // the piece's output: row xrow[f] of its ring's block (ring-blocked x)
      // or of the interleaved ring-major row
      uint8_t* xseg[FR];
#pragma unroll
      for (int f = 0; f < FR; ++f)
        xseg[f] = p.blocked ? p.x + p.xmax * pb.z + xrow[f] * pb.w + (pa.y - pb.z)
                            : xbase[f] + pa.y;
      uint32_t sq[FR];
#pragma unroll
      for (int f = 0; f < FR; ++f) sq[f] = 0;
      // whole source words: one conflict-free 32-bit load per output word
      const uint32_t wt = words_s + 2u * static_cast<uint32_t>(pa.w);
#pragma unroll 1
      for (int g = lane; g < pa.z; g += 32) {
        const uint32_t w4 = 4u * lds_u16(wt + 2u * g);
#pragma unroll
        for (int f = 0; f < FR; ++f) {
          const uint32_t word = lds_u32(band_s[f] + w4);
          if (f < nfr) stg_u32(xseg[f] + 4 * g, word);
          sq[f] = __dp4a(word, word, sq[f]);
        }
      }
      // leftover pixels: 4-byte gather
      const int ob = 4 * pa.z;
      const uint32_t bt = bytes_s + 8u * static_cast<uint32_t>(pb.y);
#pragma unroll 1
      for (int g = lane; g < pb.x; g += 32) {
        const uint2 e = lds_v2(bt + 8u * g);
        const uint32_t o0 = e.x & 0xFFFFu, o1 = e.x >> 16, o2 = e.y & 0xFFFFu, o3 = e.y >> 16;
#pragma unroll
        for (int f = 0; f < FR; ++f) {
          const uint32_t v0 = lds_u8(band_s[f] + o0), v1 = lds_u8(band_s[f] + o1);
          const uint32_t v2 = lds_u8(band_s[f] + o2), v3 = lds_u8(band_s[f] + o3);
          const uint32_t word = prmt(v0 | (v1 << 8), v2 | (v3 << 8), 0x5410);
          if (f < nfr) stg_u32(xseg[f] + ob + 4 * g, word);
          sq[f] = __dp4a(word, word, sq[f]);
        }
      }
      // exact: integer sums, any order (a piece's sum is < 2^32)
#pragma unroll
      for (int f = 0; f < FR; ++f) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, sq[f]);
        if (lane == 0 && f < nfr) red_add_u64(nrow[f] + pa.x, v);
      }
    }
    __syncwarp();
    if (lane == 0)
      for (int f = 0; f < nfr; ++f)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                         smem_addr(&empty[slot + f]))
                     : "memory");
  }
}

// Per (frame, ring): norms, inverse norms, zero-frame bookkeeping.
__global__ void k_norms(NormParams p) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = p.ring0 + static_cast<int>(blockIdx.y);
  const int lane = threadIdx.x & 31;
  const bool valid = i < p.n_frames;
  const int64_t t = p.t0 + i;
  const int64_t n2 = valid ? p.norm2[t * p.n_rings + r] : 0;
  if (valid) {
    const double nrm = sqrt(static_cast<double>(n2));
    p.norms[r * p.ld + t] = nrm;
    const double iv = n2 > 0 ? 1.0 / nrm : 0.0;
    p.inv[r * p.ld + t] = iv;
    if (p.inv2) {
      const float hi = static_cast<float>(iv);
      p.inv2[r * p.ld + t] = make_float2(hi, static_cast<float>(iv - static_cast<double>(hi)));
    }
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
    if (ovf && p.err) atomicOr(p.err, 4);  // raw streams only; K2 checks batch series
    if (p.max_norm2) atomicMax(p.max_norm2, mx);
  }
}

}  // namespace

cudaError_t launch_ingest(const IngestParams& p, cudaStream_t s) {
  const size_t smem = NBUF * static_cast<size_t>(ingest_band_stride(p.band)) +
                      static_cast<size_t>((p.max_words + 7) & ~7) * 2 +  // word table
                      static_cast<size_t>((p.max_bytes + 1) & ~1) * 8 +  // byte table
                      static_cast<size_t>(p.max_band_pieces) * sizeof(Piece);
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
  dim3 grid(static_cast<unsigned>((p.n_frames + 255) / 256),
            p.ring_count >= 0 ? p.ring_count : p.n_rings);
  k_norms<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// K1e: CTA = frame.  Threads stride over the frame's events (coalesced
// pix/val reads), look up (ring, column), store the count into the cleared
// ring-major row and add its square into the ring's shared-memory |x|^2;
// the CTA then writes the frame's |x|^2 row (exact integers: the same
// statistics as K1 on the dense raster).
__global__ void __launch_bounds__(256) k_ingest_events(EventIngestParams p) {
  extern __shared__ unsigned long long sq[];
  const int64_t f = p.t0 + blockIdx.x;
  for (int r = threadIdx.x; r < p.n_rings; r += blockDim.x) sq[r] = 0ull;
  __syncthreads();
  const int64_t e0 = p.frame_off[f], e1 = p.frame_off[f + 1];
  for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
    const int32_t px = p.pix[i];
    if (px < 0 || px >= p.pixels) {
      atomicOr(p.err, 8);
      continue;
    }
    const int32_t e = p.pixcol[px];
    if (e < 0) continue;
    const int r = e >> 22, col = e & 0x3FFFFF;
    const uint32_t v = p.val[i];
    const int64_t koff = p.ring_koff[r];
    uint8_t* row = p.blocked
                       ? p.x + p.xmax * koff + f * (static_cast<int64_t>(p.ring_nkb[r]) * 128) + (col - koff)
                       : p.x + f * p.ktot + col;
    *row = static_cast<uint8_t>(v);
    atomicAdd(&sq[r], static_cast<unsigned long long>(v * v));
  }
  __syncthreads();
  for (int r = threadIdx.x; r < p.n_rings; r += blockDim.x) p.norm2[f * p.n_rings + r] = sq[r];
}

cudaError_t launch_ingest_events(const EventIngestParams& p, cudaStream_t s) {
  if (p.n_frames < 1) return cudaSuccess;
  const size_t smem = static_cast<size_t>(p.n_rings) * sizeof(unsigned long long);
  k_ingest_events<<<static_cast<unsigned>(p.n_frames), 256, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace xg
