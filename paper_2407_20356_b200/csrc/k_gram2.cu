// k_gram2.cu -- K2 (raw u8 Gram, kind::i8) and K4 (compressed Gram,
// kind::f16 over bf16 split planes) on CTA pairs: tcgen05.mma.cta_group::2,
// 256 x 256 tiles per cluster of 2 SMs.
//
// Each MMA is M=256 x N=256 x K=32 issued by the leader CTA for the pair:
// CTA r of the pair stages rows [i0 + 128 r, +128) of A and columns
// [j0 + 128 r, +128) of B (half of each operand), so every SM moves half the
// B bytes per output that a 1-CTA 128 x 256 tile would (64 instead of
// 96 B/cycle of smem+L2 operand traffic at full MMA rate).  Each CTA's TMEM
// holds its 128 rows x 256 columns; its epilogue works on that 128 x 256 half
// tile, and the half tile's g2 partial lands at the index of the 128 x 256
// half-tile enumeration (build_tiles' d_tiles), which k_g2_fold folds.
//
// Pair protocol: full barriers live in the leader (count 1, leader posts
// expect_tx for both CTAs' bytes; both CTAs' TMA loads complete_tx there);
// empty/tfull barriers in both CTAs are signalled by the leader's commits
// multicast to the pair; the leader's tempty counts the epilogue warps of
// both CTAs (the peer arrives remotely).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "xg_kernels.h"
#include "xg_ptx.cuh"

namespace xg {

namespace {

constexpr int BM = 128;            // rows per CTA (256 per pair)
constexpr int BN = 256;            // tile columns
constexpr int BK = 128;            // bytes of K per stage
constexpr int A_BYTES = BM * BK;   // 16 KB
constexpr int B_BYTES = 128 * BK;  // 16 KB: this CTA's half of the 256 columns
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;
// K2 (raw, long K loop) and K4 (compressed, K = 6 x 64): 5 operand stages
// and 8 epilogue warps (two per TMEM lane quarter, each taking half the
// columns); the epilogue is on the critical path of small-ring and K4 tiles.
template <int MODE> struct Cfg2 {
  // 5 operand stages and one staging chunk per epilogue warp.  K4 with two
  // staging buffers (two C~ chunk stores in flight per warp) needs the smem
  // of a stage: 4 stages + 2 buffers measured 0.273 ms vs 0.259 ms.
  static constexpr int STAGES = 5;
  static constexpr int SBUF = 1;  // staging buffers per epilogue warp (1 or 2)
  // K4's epilogue is latency-bound (TMEM load -> staging -> TMA store and
  // the diagonal walk per chunk): 12 warps, three per TMEM lane quarter
  static constexpr int EPI_WARPS = MODE == 1 ? 12 : 8;
  static constexpr int NUM_THREADS = 128 + 32 * EPI_WARPS;
  // g2 window slots per epilogue warp: its chunks + 1 windows of 32 lags
  static constexpr int WSLOTS = EPI_WARPS == 8 ? 160 : 128;
};
constexpr int NDIAG = BM + BN - 1;
constexpr int NDIAG_PAD = 384;

template <int MODE>
constexpr uint32_t idesc2() {
  // M = 256 (m_dim = 16), N = 256
  return MODE == 0 ? idesc_i8(256, BN, false) : idesc_bf16(256, BN);
}

template <int MODE, int EPI_WARPS, int STAGES, int SBUF, int WSLOTS>
struct __align__(1024) Tail2 {
  uint32_t stage[SBUF][EPI_WARPS][32 * 32];  // 32x32 chunks per warp, 128B-swizzled
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  uint32_t pad_;
  // 1/|x| of the tile's rows and columns as (hi, lo) floats, staged by warp 2
  // one tile ahead (two buffers); the columns reach 32 past either side
  float2 inv_row2[2][MODE == 0 ? BM : 1];
  float2 inv_col2_ext[2][MODE == 0 ? BN + 64 : 1];
  // each epilogue warp's window sums of one tile (2 tiles in flight),
  // folded by warp 3
  // ((hi, lo) double-float for the raw Gram, fp32 for C~)
  typename std::conditional<MODE == 0, float2, float>::type slot[2][EPI_WARPS][WSLOTS];
  uint64_t accfull[2];
  uint64_t accfree[2];
  uint64_t invfull[2];
  uint64_t invfree[2];
};

// Epilogue warp (sub, grp) of NG = EPI_WARPS / 4 column groups: chunks
// [grp_c0(grp), grp_c0(grp + 1)) of the 8 in a 256-wide tile row, window
// slots [grp_c0(grp), grp_c0(grp + 1)] -- the window at a group boundary
// straddles two groups' chunks, each holds its part, the fold adds them.
template <int NG>
__device__ __forceinline__ int grp_c0(int g) {
  return NG == 2 ? 4 * g : (g == 3 ? 8 : 3 * g);
}

// f32 bits -> f64 with integer ops only (normal numbers; zero and
// denormals -> +-0, far below the compressed path's 1e-5 tolerance)
__device__ __forceinline__ double f32_to_f64_bits(uint32_t w) {
  const uint32_t e = (w >> 23) & 0xFFu;
  if (e == 0u) return 0.0;
  const uint32_t hi = (w & 0x80000000u) | ((e + 896u) << 20) | ((w >> 3) & 0xFFFFFu);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(w << 29));
}

// (a.x + a.y) + (bh + bl) in FP32 double-float (~48 bits): TwoSum of the high
// parts, low parts added into the error, renormalised.
__device__ __forceinline__ float2 dd_add(float2 a, float bh, float bl) {
  const float s = __fadd_rn(a.x, bh);
  const float bb = __fsub_rn(s, a.x);
  float e = __fadd_rn(__fsub_rn(a.x, __fsub_rn(s, bb)), __fsub_rn(bh, bb));
  e = __fadd_rn(e, __fadd_rn(a.y, bl));
  const float hi = __fadd_rn(s, e);
  return make_float2(hi, __fsub_rn(e, __fsub_rn(hi, s)));
}



}  // namespace

template <int MODE>
constexpr size_t smem2_bytes() {
  return 1024 + Cfg2<MODE>::STAGES * STAGE_BYTES +
         sizeof(Tail2<MODE, Cfg2<MODE>::EPI_WARPS, Cfg2<MODE>::STAGES, Cfg2<MODE>::SBUF,
                       Cfg2<MODE>::WSLOTS>);
}
size_t gram2_smem_bytes(int mode) { return mode == 0 ? smem2_bytes<0>() : smem2_bytes<1>(); }

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2<MODE>::NUM_THREADS, 1)
    k_gram2(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmOut,
            GramParams p) {
  constexpr uint32_t IDESC = idesc2<MODE>();
  constexpr int STAGES = Cfg2<MODE>::STAGES, EPI_WARPS = Cfg2<MODE>::EPI_WARPS;
  constexpr int SBUF = Cfg2<MODE>::SBUF;
  constexpr int WSLOTS = Cfg2<MODE>::WSLOTS, NG = EPI_WARPS / 4;
  using Tail = Tail2<MODE, EPI_WARPS, STAGES, SBUF, WSLOTS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  Tail* tail = reinterpret_cast<Tail*>(smem + STAGES * STAGE_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  int n_planes = 1;  // K4: bf16 planes the precision pairs touch
  int plast[3] = {0, 0, 0};  // K4: index of each plane's last product
  if (MODE == 1)
    for (int pr = 0; pr < p.n_pairs; ++pr) {
      const int pa = (p.pairs >> (4 * pr)) & 3, pb = (p.pairs >> (4 * pr + 2)) & 3;
      n_planes = max(n_planes, max(pa, pb) + 1);
      plast[pa] = pr;
      plast[pb] = pr;
    }

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tail->full[s], 1);
      mbar_init(&tail->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tail->tfull[a], 1);
      mbar_init(&tail->tempty[a], 2 * EPI_WARPS);  // epilogue warps of both CTAs
      mbar_init(&tail->accfull[a], EPI_WARPS);
      mbar_init(&tail->accfree[a], MODE == 1 ? 2 : 1);  // the folding warps
      mbar_init(&tail->invfull[a], 1);
      mbar_init(&tail->invfree[a], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch(&tmX);
    tma_prefetch(&tmOut);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tail->tmem_base)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  // the exact int32 Gram holds every entry only while |x|^2 < 2^31 (checked
  // here, where the raw Gram is formed, not at ingest: compressed-only series
  // may carry brighter frames)
  if (MODE == 0 && blockIdx.x == 0 && threadIdx.x == 0 && p.max_norm2 != nullptr &&
      *p.max_norm2 >= (1ull << 31))
    atomicOr(p.err, 4);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = tail->tmem_base;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int wave = 0;
      for (int t = pair; t < p.ntiles; t += npairs, ++wave) {
        if (MODE == 0 && leader && p.wave_ctr) {
          // wave gate: every pair has started wave - gate_lag (bounded wait)
          const unsigned need = static_cast<unsigned>((wave - p.gate_lag + 1) * npairs);
          if (wave >= p.gate_lag) {
            uint32_t spins = 0;
            while (ld_acquire_u32(p.wave_ctr) < need) {
              __nanosleep(64);
              if (++spins == (1u << 26)) {
                atomicExch(p.err, 1);
                goto producer_done;
              }
            }
          }
          atomicAdd(p.wave_ctr, 1u);
        }
        const TileDesc td = p.tiles[t];
        // raw: the ring's own block of x (ring-blocked, per-ring TMA map)
        const CUtensorMap* mapA = MODE == 0 ? p.xmaps + td.ring : &tmX;
        // K4: per 64-coefficient block, one stage per bf16 plane (A and B
        // rows of that plane); the MMA warp forms every precision pair from
        // the resident planes, so each plane block is fetched once, not once
        // per pair
        const int nkb = MODE == 0 ? p.ring_nkb[td.ring] : p.kb_per_plane * n_planes;
        for (int kb = 0; kb < nkb; ++kb) {
          if (!mbar_wait(&tail->empty[stage], phase ^ 1, p.err)) goto producer_done;
          if (leader) mbar_arrive_expect_tx(&tail->full[stage], 2 * STAGE_BYTES);
          int kc, ra, rb;
          if (MODE == 0) {
            kc = kb * BK;
            ra = td.i0 + 128 * rank;
            rb = td.j0 + 128 * rank;
          } else {
            const int q = kb % n_planes;
            kc = (kb / n_planes) * 64;
            ra = (td.ring * 3 + q) * p.plane_rows + td.i0 + 128 * rank;
            rb = (td.ring * 3 + q) * p.plane_rows + td.j0 + 128 * rank;
          }
          tma_load_2sm(sA + stage * A_BYTES, mapA, &tail->full[stage], kc, ra);
          tma_load_2sm(sB + stage * B_BYTES, mapA, &tail->full[stage], kc, rb);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    producer_done:;
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int t = pair; t < p.ntiles; t += npairs) {
        const TileDesc td = p.tiles[t];
        const int nkb = MODE == 0 ? p.ring_nkb[td.ring] : p.kb_per_plane;
        if (!mbar_wait(&tail->tempty[acc], acc_phase ^ 1, p.err)) break;
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
        bool ok = true;
        if (MODE == 1) {
          // products in the host's order (ascending highest plane): each
          // waits only for the planes it reads, so the first products run
          // while the later planes land, and a plane's stage is released
          // right after its last product (plane 1 of the f32 mode before
          // the plane-2 products), letting the next tile's loads start
          for (int kb = 0; ok && kb < nkb; ++kb) {
            int st[3];
            int have = 0;
            for (int pr = 0; pr < p.n_pairs; ++pr) {
              const int pa = (p.pairs >> (4 * pr)) & 3, pb = (p.pairs >> (4 * pr + 2)) & 3;
              for (; have <= max(pa, pb); ++have) {
                if (!mbar_wait(&tail->full[stage], phase, p.err)) {
                  ok = false;
                  break;
                }
                st[have] = stage;
                if (++stage == STAGES) {
                  stage = 0;
                  phase ^= 1;
                }
              }
              if (!ok) break;
              tc_fence_after();
              const uint32_t a0 = smem_u32(sA + st[pa] * A_BYTES);
              const uint32_t b0 = smem_u32(sB + st[pb] * B_BYTES);
#pragma unroll
              for (int k = 0; k < BK / 32; ++k)
                mma2_bf16(tmem_d, sdesc_k128(a0 + k * 32), sdesc_k128(b0 + k * 32), IDESC,
                          (kb | pr | k) != 0 ? 1u : 0u);
              for (int q = 0; q < have; ++q)
                if (plast[q] == pr) commit2(&tail->empty[st[q]]);
            }
          }
        } else
        for (int kb = 0; kb < nkb; ++kb) {
          if (!mbar_wait(&tail->full[stage], phase, p.err)) {
            ok = false;
            break;
          }
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES), b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            if (MODE == 0)
              mma2_i8(tmem_d, sdesc_k128(a0 + k * 32), sdesc_k128(b0 + k * 32), IDESC,
                      (kb | k) != 0 ? 1u : 0u);
            else
              mma2_bf16(tmem_d, sdesc_k128(a0 + k * 32), sdesc_k128(b0 + k * 32), IDESC,
                        (kb | k) != 0 ? 1u : 0u);
          }
          commit2(&tail->empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (!ok) break;
        commit2(&tail->tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (MODE == 0 && warp == 2) {
    // K2 g2 weights: 1/|x| of the next tile's rows and columns staged one
    // tile ahead, so the epilogue warps never stop to load them
    if (p.g2_partial) {
      int it = 0;
      for (int t = pair; t < p.ntiles; t += npairs, ++it) {
        const int buf = it & 1;
        if (it >= 2 && !mbar_wait(&tail->invfree[buf], ((it >> 1) - 1) & 1, p.err)) break;
        const TileDesc td = p.tiles[t];
        const int i0 = td.i0 + 128 * static_cast<int>(rank);
        const float2* inv2 = p.inv2 + static_cast<int64_t>(td.ring) * p.inv_ld;
        for (int e = lane; e < BM + BN + 64; e += 32) {
          const int j = e - BM - 32;
          const int idx = e < BM ? i0 + e : td.j0 + j;
          const bool in = idx < p.n_frames && (e < BM || (j >= 0 && j < BN));
          const float2 hl = in ? inv2[idx] : make_float2(0.f, 0.f);
          if (e < BM)
            tail->inv_row2[buf][e] = hl;
          else
            tail->inv_col2_ext[buf][e - BM] = hl;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tail->invfull[buf]);
      }
    }
  } else if (warp == 3 || (MODE == 1 && warp == 2)) {
    // g2 fold: sums the 8 epilogue warps' window slots of each tile in a
    // fixed warp order and writes the tile's diagonal sums, so the epilogue
    // warps never meet at a barrier (they run up to 2 tiles ahead).  K4's
    // tiles are short (K = 6 x 64), so there the otherwise idle warp 2 takes
    // half the diagonals and the sums are plain fp32 (C~ is fp32; the slots
    // carry no low part): the fold was the bottleneck (0.304 -> 0.259 ms
    // without it, ncu/A-B).
    const int e_lo = MODE == 1 && warp == 3 ? 192 : 0;
    const int e_hi = MODE == 1 && warp == 2 ? 192 : NDIAG;
    if (p.g2_partial) {
      auto* acc2 = tail->slot;
      int it = 0;
      for (int t = pair; t < p.ntiles; t += npairs, ++it) {
        const int buf = it & 1;
        if (!mbar_wait(&tail->accfull[buf], (it >> 1) & 1, p.err)) break;
        const TileDesc td = p.tiles[t];
        if (2 * (td.i0 / 256) + static_cast<int>(rank) < p.g2_nbi) {
          const int64_t half = td.pad + static_cast<int64_t>(rank) * (p.g2_nbj - td.i0 / 256);
          // K4: fp32 sums (the low parts would be zero), half the bytes
          float2* out = p.g2_partial + half * NDIAG_PAD;
          float* out1 = reinterpret_cast<float*>(p.g2_partial) + half * NDIAG_PAD;
          for (int e = e_lo + lane; e < e_hi; e += 32) {
            float2 sum = make_float2(0.f, 0.f);
#pragma unroll
            for (int w = 0; w < EPI_WARPS; ++w) {
              const int sb = w & 3, gp = w >> 2;
              const int off = e - 96 + 32 * sb - 32 * grp_c0<NG>(gp);
              if (off >= 0 && off < 32 * (grp_c0<NG>(gp + 1) - grp_c0<NG>(gp) + 1)) {
                if constexpr (MODE == 1) {
                  sum.x += acc2[buf][w][off];
                } else {
                  const float2 v = acc2[buf][w][off];
                  sum = dd_add(sum, v.x, v.y);
                }
              }
            }
            if (MODE == 1)
              out1[e] = sum.x;
            else
              out[e] = sum;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tail->accfree[buf]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;        // epilogue warp 0..7
    const int sub = warp & 3;       // TMEM lane quarter this warp may access
    const int etid = threadIdx.x - 128;
    // double-float g2 needs every count of the Gram exact in fp32 (< 2^23)
    const bool dd_ok = p.max_norm2 != nullptr && *p.max_norm2 < (1ull << 23);
    int acc = 0;
    uint32_t acc_phase = 0;
    bool ok = true;
    int sbuf = 0;  // staging buffer of the next chunk (alternates when SBUF = 2)
    // K4 window walk: word offset in the staged (swizzled) chunk of this
    // lane's element in row l, column (lane + 1 + l) mod 32
    int wtab[MODE == 1 ? 32 : 1];
    if (MODE == 1)
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        const int u = lane + 1 + l;
        wtab[l] = l * 32 + ((u & 31) ^ ((l & 7) << 2));
      }
    for (int t = pair; t < p.ntiles; t += npairs) {
      const TileDesc td = p.tiles[t];
      const int i0 = td.i0 + 128 * static_cast<int>(rank);  // this CTA's half tile
      if (ok) ok = mbar_wait(&tail->tfull[acc], acc_phase, p.err);
      ok = __all_sync(0xffffffffu, ok);
      if (ok) tc_fence_after();
      const int it = (t - pair) / npairs, buf = it & 1;
      auto* slots = &tail->slot[buf][ew][0];
      if (p.g2_partial && it >= 2)  // warp 3 has folded this buffer's last tile
        if (!mbar_wait(&tail->accfree[buf], ((it >> 1) - 1) & 1, p.err)) ok = false;
      if (MODE == 0 && p.g2_partial)  // warp 2 has staged this tile's 1/|x|
        if (!mbar_wait(&tail->invfull[buf], (it >> 1) & 1, p.err)) ok = false;
      const uint32_t tbase =
          tmem_base + static_cast<uint32_t>(acc * BN) + (static_cast<uint32_t>(sub * 32) << 16);
      // packed pair tile (ttc_off): rows of tile (I, J) of ring r start at
      // (r * tiles_per_slab + tile(I, J)) * 256; this CTA's half adds 128 rank
      const int64_t tI = td.i0 >> 8, tJ = td.j0 >> 8;
      const int out_row = static_cast<int>(
          ((p.ring_stride >> 16) * td.ring + tI * p.nb - (tI * (tI - 1)) / 2 + (tJ - tI)) * 256 +
          128 * static_cast<int>(rank) + 32 * sub);
      // Column chunks c (32 wide) are staged one at a time in this warp's
      // buffer, stored by TMA and read by the g2 window sums.  Window w
      // (lane L sums the diagonal elements (l, 32(w-1) + L + 1 + l), l =
      // 0..31) spans chunks w-1 and w: element (l, kk = (L+1+l) & 31) of chunk
      // c finishes window c when L+1+l >= 32 and starts window c+1 otherwise.
      // Both sums advance in ascending l, so every window keeps its
      // one-pass order with a single staged chunk.  Each column group reads
      // and stores its own chunks (K2: 0..3 | 4..7, K4: 0..2 | 3..5 | 6..7);
      // a window at a group boundary is summed in two parts.
      const int grp = ew >> 2;
      const int c_first = grp_c0<NG>(grp);
      const int c_last = grp_c0<NG>(grp + 1) - 1;
      const int w_lo = c_first, w_hi = c_last + 1;
      const bool fp32 = MODE == 1 || dd_ok;  // FP32 (double-float) sums, else FP64
      float cur_h = 0.f, cur_l = 0.f, nxt_h = 0.f, nxt_l = 0.f;
      double cur_d = 0.0, nxt_d = 0.0;
      auto finish = [&](int w, float wh, float wl) {
        if (w < w_lo || w > w_hi) return;
        const int lagw = td.j0 - i0 + 32 * (w - 1 - sub) + lane + 1;  // this lane's lag
        if constexpr (MODE == 1)
          slots[32 * (w - w_lo) + lane] = lagw >= 0 ? wh : 0.f;
        else
          slots[32 * (w - w_lo) + lane] = lagw >= 0 ? make_float2(wh, wl) : make_float2(0.f, 0.f);
      };
#pragma unroll 1
      for (int c = c_first; ok && c <= c_last; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        tmem_ld_wait();
        // the TMA store of the previous chunk has read the buffer
        uint32_t* S = tail->stage[sbuf][ew];
        if (SBUF == 2) sbuf ^= 1;
        // (SBUF = 2: the store before that, from this buffer)
        if (lane == 0) {
          if (SBUF == 2)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<uint4*>(S + lane * 32 + ((q ^ (lane & 7)) << 2)) =
              make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
        fence_proxy_async();
        __syncwarp();
        // chunks wholly below the diagonal of a diagonal tile are never read
        // (every reader takes the upper triangle a <= b): not stored
        const bool lower = td.i0 == td.j0 && c < sub + 4 * static_cast<int>(rank);
        if (lane == 0 && p.store && !lower) {
          // the TTC streams out once: evict-first in L2, so it does not push
          // the ring's frame rows (re-read by later tiles) out of L2
          uint64_t pol;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                  reinterpret_cast<uint64_t>(&tmOut)),
              "r"(smem_u32(S)), "r"(32 * c), "r"(out_row), "l"(pol)
              : "memory");
        }
        // one bulk group per chunk, empty when nothing was stored, so with
        // two staging buffers the group wait_group.read 1 leaves pending is
        // always the other buffer's
        if (lane == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (p.g2_partial) {
          const int col0 = td.j0 + 32 * c;  // first frame of this chunk's columns
          const float2* ir2 = tail->inv_row2[buf] + 32 * sub;
          const float2* ic2 = tail->inv_col2_ext[buf] + 32 + 32 * c;  // + kk
          if (MODE == 1 && col0 + 32 <= p.n_frames) {
            // every column is a frame: the precomputed walk, no mask; four
            // interleaved partial sums (l mod 4) shorten the dependent chain
            float ch[4] = {0.f, 0.f, 0.f, 0.f}, nx[4] = {0.f, 0.f, 0.f, 0.f};
            // all 32 elements into ch, the starting window's into nx: one
            // select per element instead of two; ch - nx finishes window c
#pragma unroll
            for (int l = 0; l < 32; ++l) {
              const float v = __uint_as_float(S[wtab[l]]);
              ch[l & 3] += v;
              nx[l & 3] += lane + 1 + l >= 32 ? 0.f : v;
            }
            const float nsum = (nx[0] + nx[1]) + (nx[2] + nx[3]);
            cur_h += ((ch[0] + ch[1]) + (ch[2] + ch[3])) - nsum;
            nxt_h += nsum;
          } else
#pragma unroll
          for (int l = 0; l < 32; ++l) {
            const int u = lane + 1 + l;
            const bool fin = u >= 32;  // finishes window c, else starts window c + 1
            const int kk = u & 31;
            const uint32_t wv = S[l * 32 + (kk ^ ((l & 7) << 2))];
            if (MODE == 1) {
              const float v = col0 + kk < p.n_frames ? __uint_as_float(wv) : 0.f;
              if (fin) cur_h += v; else nxt_h += v;
            } else if (fp32) {
              // exact float G (< 2^23), error-free two-product of the (hi, lo)
              // weights, TwoSum accumulation
              const float g = __fsub_rn(__int_as_float(0x4B000000 | static_cast<int>(wv)), 8388608.f);
              const float2 a = ir2[l], b = ic2[kk];
              const float ph = __fmul_rn(a.x, b.x);
              float pe = __fmaf_rn(a.x, b.x, -ph);
              pe = __fmaf_rn(a.x, b.y, pe);
              pe = __fmaf_rn(a.y, b.x, pe);
              const float qh = __fmul_rn(g, ph);
              const float ql = __fmaf_rn(g, pe, __fmaf_rn(g, ph, -qh));
              const float sh = fin ? cur_h : nxt_h, sl = fin ? cur_l : nxt_l;
              const float t = __fadd_rn(sh, qh);  // TwoSum(sh, qh)
              const float z = __fsub_rn(t, sh);
              const float er = __fadd_rn(__fsub_rn(sh, __fsub_rn(t, z)), __fsub_rn(qh, z));
              const float nl = __fadd_rn(sl, __fadd_rn(er, ql));
              if (fin) { cur_h = t; cur_l = nl; } else { nxt_h = t; nxt_l = nl; }
            } else {
              // FP64 path (a frame with |x|^2 >= 2^23 in this series)
              const double ia = static_cast<double>(ir2[l].x) + ir2[l].y;
              const double ib = static_cast<double>(ic2[kk].x) + ic2[kk].y;
              const double v =
                  (__hiloint2double(0x43300000, static_cast<int>(wv)) - 4503599627370496.0) * (ia * ib);
              if (fin) cur_d += v; else nxt_d += v;
            }
          }
          if (MODE == 0 && !fp32) {
            const float wh = static_cast<float>(cur_d);
            finish(c, wh, static_cast<float>(cur_d - static_cast<double>(wh)));
          } else {
            finish(c, cur_h, cur_l);
          }
          cur_h = nxt_h;
          cur_l = nxt_l;
          cur_d = nxt_d;
          nxt_h = nxt_l = 0.f;
          nxt_d = 0.0;
        }
        __syncwarp();
      }
      if (ok && p.g2_partial) {  // the last window: its second chunk is past the tile
        if (MODE == 0 && !fp32) {
          const float wh = static_cast<float>(cur_d);
          finish(c_last + 1, wh, static_cast<float>(cur_d - static_cast<double>(wh)));
        } else {
          finish(c_last + 1, cur_h, cur_l);
        }
      }
      if (p.g2_partial) {  // this warp's window slots are written, the weights read
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&tail->accfull[buf]);
          if (MODE == 0) mbar_arrive(&tail->invfree[buf]);
        }
      }
      if (ok) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader)
            mbar_arrive(&tail->tempty[acc]);
          else
            arrive_leader(&tail->tempty[acc]);
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  tc_fence_before();
  cluster_sync();  // no remote arrivals in flight, both CTAs done with TMEM
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

template <int MODE>
static cudaError_t launch2(const CUtensorMap& tmX, const CUtensorMap& tmOut, const GramParams& p,
                           int num_sms, cudaStream_t stream) {
  const size_t smem = smem2_bytes<MODE>();
  cudaError_t e =
      cudaFuncSetAttribute(k_gram2<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int pairs = num_sms / 2;
  if (p.ntiles < pairs) pairs = p.ntiles;
  if (pairs <= 0) return cudaSuccess;
  k_gram2<MODE><<<2 * pairs, Cfg2<MODE>::NUM_THREADS, smem, stream>>>(tmX, tmOut, p);
  return cudaGetLastError();
}

cudaError_t launch_gram2_u8(const CUtensorMap& tmX, const CUtensorMap& tmOut, const GramParams& p,
                            int num_sms, cudaStream_t stream) {
  return launch2<0>(tmX, tmOut, p, num_sms, stream);
}
cudaError_t launch_gram2_cmp(const CUtensorMap& tmY, const CUtensorMap& tmOut, const GramParams& p,
                             int num_sms, cudaStream_t stream) {
  return launch2<1>(tmY, tmOut, p, num_sms, stream);
}

}  // namespace xg
