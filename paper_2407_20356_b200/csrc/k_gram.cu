// k_gram.cu -- K2: per-ring raw two-time Gram G_q = X_q X_q^T on tcgen05.
//
// Replaces the reference's hot loop `gram` (src/linalg.cpp:127-156) as used by
// `ttc_raw` (src/correlate.cpp:19-25).  Photon counts are u8, so the Gram is
// computed EXACTLY as u8 x u8 -> s32 (tcgen05.mma kind::i8) and equals
// xpcs::gram of the same counts bit for bit (all partial sums are integers
// < 2^31, checked by the host from the diagonal bound 255^2 * M_q or the
// ingest statistics).
//
// Design (sm_100a):
//   * persistent kernel, one CTA per SM, static round-robin over a host-built
//     list of upper-triangle tiles (ring, i0, j0) of 128 x 256 outputs;
//   * warp 0: TMA producer (128-byte swizzled K-major boxes of the ring-major
//     frame matrix, 4-stage smem ring, mbarrier full/empty pipeline);
//   * warp 1: single-thread tcgen05.mma issuer, accumulator in TMEM
//     (2 x 256 columns, double buffered so the epilogue of tile n overlaps the
//     MMAs of tile n+1);
//   * warp 2: TMEM allocator;  warps 4-7: epilogue, tcgen05.ld -> int32 rows
//     -> 128-byte vector stores of the exact Gram tile.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"
#include "xg_ptx.cuh"

namespace xg {

namespace {

constexpr int BM = 128;                    // tile rows   (frames t1)
constexpr int BN = 256;                    // tile cols   (frames t2)
constexpr int BK = 128;                    // bytes of K per stage (= 4 MMAs of K=32)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;           // 16 KB
constexpr int B_BYTES = BN * BK;           // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;             // 2 accumulators x 256 s32 columns
constexpr int NUM_THREADS = 256;
// MODE 0: raw u8 x u8 -> s32 (kind::i8);  MODE 1: compressed bf16 x bf16 ->
// f32 (kind::f16) over split-precision coefficient planes (see k_project.cu).
template <int MODE>
constexpr uint32_t gram_idesc() {
  return MODE == 0 ? idesc_i8(BM, BN, false) : idesc_bf16(BM, BN);
}

constexpr int NDIAG = BM + BN - 1;         // tile diagonals j-i in [-127, 255]
constexpr int NDIAG_PAD = 384;

struct __align__(1024) GramSmemTail {
  uint32_t stage[4][32 * 32];              // per-warp 32x32 output chunk, 128B-swizzled
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  uint32_t pad_;
  // fused-g2 epilogue scratch
  double inv_row[BM];                      // 1/|x_i| of the tile rows (0 beyond T / zero frame)
  double inv_col[BN];                      // 1/|x_j| of the tile columns
  double acc[4][NDIAG_PAD];                // per-warp diagonal sums of the tile
};

__device__ __forceinline__ void epi_bar() {  // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

}  // namespace

size_t gram_u8_smem_bytes() { return 1024 + STAGES * STAGE_BYTES + sizeof(GramSmemTail); }

template <int MODE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gram_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmOut,
              GramParams p) {
  constexpr uint32_t IDESC = gram_idesc<MODE>();
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms; offsetting the shared
  // array itself (not a uintptr_t round trip) keeps accesses in the shared
  // state space (LDS/STS rather than generic LD/ST).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  GramSmemTail* tail = reinterpret_cast<GramSmemTail*>(smem + STAGES * STAGE_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tail->full[s], 1);
      mbar_init(&tail->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tail->tfull[a], 1);
      mbar_init(&tail->tempty[a], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
    tma_prefetch(&tmX);
    tma_prefetch(&tmOut);
  }
  if (warp == 2) tmem_alloc(&tail->tmem_base, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tail->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------- TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const TileDesc td = p.tiles[t];
        const int koff = MODE == 0 ? p.ring_koff[td.ring] : 0;
        const int nkb = MODE == 0 ? p.ring_nkb[td.ring] : p.n_pairs * p.kb_per_plane;
        for (int kb = 0; kb < nkb; ++kb) {
          if (!mbar_wait(&tail->empty[stage], phase ^ 1, p.err)) goto producer_done;
          mbar_arrive_expect_tx(&tail->full[stage], STAGE_BYTES);
          int kc, ra, rb;
          if (MODE == 0) {  // byte column of the ring, frame rows
            kc = koff + kb * BK;
            ra = td.i0;
            rb = td.j0;
          } else {  // K block = (precision pair, 64-element block of the plane)
            const int pr = kb / p.kb_per_plane;
            kc = (kb - pr * p.kb_per_plane) * 64;
            const int plane_a = (p.pairs >> (4 * pr)) & 3, plane_b = (p.pairs >> (4 * pr + 2)) & 3;
            ra = (td.ring * 3 + plane_a) * p.plane_rows + td.i0;
            rb = (td.ring * 3 + plane_b) * p.plane_rows + td.j0;
          }
          tma_load_2d(sA + stage * A_BYTES, &tmX, &tail->full[stage], kc, ra);
          tma_load_2d(sB + stage * B_BYTES, &tmX, &tail->full[stage], kc, rb);
          tma_load_2d(sB + stage * B_BYTES + BK * 128, &tmX, &tail->full[stage], kc, rb + 128);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    producer_done:;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const TileDesc td = p.tiles[t];
        const int nkb = MODE == 0 ? p.ring_nkb[td.ring] : p.n_pairs * p.kb_per_plane;
        if (!mbar_wait(&tail->tempty[acc], acc_phase ^ 1, p.err)) break;
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
        bool ok = true;
        for (int kb = 0; kb < nkb; ++kb) {
          if (!mbar_wait(&tail->full[stage], phase, p.err)) {
            ok = false;
            break;
          }
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            if (MODE == 0)
              mma_i8(tmem_d, sdesc_k128(a0 + k * 32), sdesc_k128(b0 + k * 32), IDESC,
                     (kb | k) != 0 ? 1u : 0u);
            else
              mma_bf16(tmem_d, sdesc_k128(a0 + k * 32), sdesc_k128(b0 + k * 32), IDESC,
                       (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit(&tail->empty[stage]);  // smem slot free once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (!ok) break;
        tc_commit(&tail->tfull[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------- epilogue
    // TMEM -> registers -> exact int32 Gram rows (global) and, when g2 is
    // fused, the per-tile diagonal sums of C(i,j) = G_ij / (|x_i||x_j|) for
    // j >= i: each 32x32 chunk goes through shared memory and lane L sums
    // the chunk diagonals m = L-31 and m = L+1 in ascending row order; the
    // four warps' tile sums are folded in warp order -> deterministic.
    const int sub = warp & 3;  // TMEM lane quarter this warp may access
    const int row = sub * 32 + lane;
    const int etid = threadIdx.x - 128;
    int acc = 0;
    uint32_t acc_phase = 0;
    bool ok = true;  // after a pipeline failure keep hitting the named barriers
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const TileDesc td = p.tiles[t];
      if (ok) ok = mbar_wait(&tail->tfull[acc], acc_phase, p.err);
      ok = __all_sync(0xffffffffu, ok);
      if (ok) tc_fence_after();
      if (p.g2_partial) {
        epi_bar();  // previous tile's fold has finished with inv/acc
        const double* inv = MODE == 0 ? p.inv + static_cast<int64_t>(td.ring) * p.inv_ld : nullptr;
        for (int e = etid; e < BM + BN; e += 128) {
          const int idx = e < BM ? td.i0 + e : td.j0 + (e - BM);
          const double v = idx < p.n_frames ? (MODE == 0 ? inv[idx] : 1.0) : 0.0;
          if (e < BM)
            tail->inv_row[e] = v;
          else
            tail->inv_col[e - BM] = v;
        }
        for (int e = lane; e < NDIAG_PAD; e += 32) tail->acc[sub][e] = 0.0;
        epi_bar();
      }
      const uint32_t tbase =
          tmem_base + static_cast<uint32_t>(acc * BN) + (static_cast<uint32_t>(sub * 32) << 16);
      // output rows of this warp in the [ring*ld + row][col] view of the map
      const int out_row = td.ring * p.ld + td.i0 + 32 * sub;
      uint32_t* S = tail->stage[sub];  // 32 rows x 128 B, 128B-swizzled
#pragma unroll 1
      for (int c = 0; ok && c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        tmem_ld_wait();
        // the previous chunk's TMA store must have finished reading S
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        // row `lane`, 16-byte chunk q stored at chunk q ^ (lane & 7)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<uint4*>(S + lane * 32 + ((q ^ (lane & 7)) << 2)) =
              make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
        fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA engine
        __syncwarp();
        if (lane == 0 && p.store) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                  reinterpret_cast<uint64_t>(&tmOut)),
              "r"(smem_u32(S)), "r"(td.j0 + 32 * c), "r"(out_row)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (p.g2_partial) {
          // global lag of chunk element (l, k): D0 + (k - l)
          const int D0 = td.j0 + 32 * c - td.i0 - 32 * sub;
          const double* ir = tail->inv_row + 32 * sub;
          const double* ic = tail->inv_col + 32 * c;
          // Lane L sums chunk diagonals m_B = L+1 (rows l < 31-L) then
          // m_A = L-31 (rows l >= 31-L): element (l, (l+L+1) mod 32) at step l,
          // one warp-uniform 32-step loop, conflict-free rows of S.
          // four interleaved partial sums (l mod 4) keep the f64 chains short
          double sa = 0.0, sb = 0.0, r0 = 0.0, r1 = 0.0, r2 = 0.0, r3 = 0.0;
          const int ma = lane - 31, mb = lane + 1;
          const bool use_a = D0 + ma >= 0, use_b = lane < 31 && D0 + mb >= 0;
#pragma unroll
          for (int l = 0; l < 32; ++l) {
            if (l == 31 - lane) {
              sb = (r0 + r1) + (r2 + r3);
              r0 = r1 = r2 = r3 = 0.0;
            }
            const int k = (l + lane + 1) & 31;
            const uint32_t w = S[l * 32 + ((((k >> 2) ^ (l & 7))) << 2) + (k & 3)];
            double v;
            if (MODE == 0)
              v = static_cast<double>(static_cast<int32_t>(w)) * (ir[l] * ic[k]);
            else  // compressed: C~ is already normalised (inv = 1 inside T)
              v = ic[k] != 0.0 ? static_cast<double>(__uint_as_float(w)) : 0.0;
            if ((l & 3) == 0) r0 += v;
            else if ((l & 3) == 1) r1 += v;
            else if ((l & 3) == 2) r2 += v;
            else r3 += v;
          }
          sa = (r0 + r1) + (r2 + r3);
          if (!use_a) sa = 0.0;
          if (!use_b) sb = 0.0;
          // tile diagonal index (j-i) + 127
          const int base = 32 * c - 32 * sub + 127;
          tail->acc[sub][base + ma] += sa;
          if (lane < 31) tail->acc[sub][base + mb] += sb;
          __syncwarp();
        }
      }
      if (ok) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tail->tempty[acc]);  // TMEM buffer free for tile n+2
      }
      if (p.g2_partial) {
        epi_bar();
        if (ok) {
          float2* out = p.g2_partial + static_cast<int64_t>(t) * NDIAG_PAD;
          for (int e = etid; e < NDIAG; e += 128) {
            const double v = ((tail->acc[0][e] + tail->acc[1][e]) + tail->acc[2][e]) + tail->acc[3][e];
            const float hi = static_cast<float>(v);
            out[e] = make_float2(hi, static_cast<float>(v - static_cast<double>(hi)));
          }
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
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <int MODE>
static cudaError_t launch_gram_mode(const CUtensorMap& tmX, const CUtensorMap& tmOut,
                                    const GramParams& p, int num_sms, cudaStream_t stream) {
  const size_t smem = gram_u8_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(k_gram_tc<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = p.ntiles < num_sms ? p.ntiles : num_sms;
  if (grid <= 0) return cudaSuccess;
  k_gram_tc<MODE><<<grid, NUM_THREADS, smem, stream>>>(tmX, tmOut, p);
  return cudaGetLastError();
}

cudaError_t launch_gram_u8(const CUtensorMap& tmX, const CUtensorMap& tmOut, const GramParams& p,
                           int num_sms, cudaStream_t stream) {
  return launch_gram_mode<0>(tmX, tmOut, p, num_sms, stream);
}

cudaError_t launch_gram_cmp(const CUtensorMap& tmY, const CUtensorMap& tmOut, const GramParams& p,
                            int num_sms, cudaStream_t stream) {
  return launch_gram_mode<1>(tmY, tmOut, p, num_sms, stream);
}

}  // namespace xg
