// k_g2.cu -- K7: g2(tau) diagonal averages and TTC readback expansion.
//
// g2 replaces `g2_from_ttc` (src/correlate.cpp:67-85): g2[d] is the mean of
// C(t, t+d) over t, accumulated in ascending t like the reference.  Each
// thread owns one lag d of one ring and one segment of `seg` frames; a warp
// covers 32 consecutive lags so every step of the t-loop is one coalesced
// 128-byte row read of the Gram.  C(t,t+d) is formed in f64 from the exact
// integer Gram and the f64 norms (so the only rounding is the normalisation
// and the sums).  Segment partials are combined in ascending segment order:
// the result is deterministic and independent of launch geometry.
//
// Zero-norm frames (inv = 0) are excluded from both the sum and the count;
// without them count[d] = N - d exactly as in the reference.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

template <int MODE>
__global__ void __launch_bounds__(128) k_g2_partial(G2Params p) {
  const int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  const int r = blockIdx.z;
  if (d >= p.n_frames) return;
  const int64_t t_begin = static_cast<int64_t>(s) * p.seg;
  int64_t t_end = t_begin + p.seg;
  if (t_end > p.n_frames - d) t_end = p.n_frames - d;
  double acc = 0.0;
  int64_t cnt = 0;
  const double* inv = p.inv + r * p.inv_ld;
  if (MODE == 0) {
    const int32_t* g = p.gram + r * p.ring_stride;
#pragma unroll 4
    for (int64_t t = t_begin; t < t_end; ++t) {
      const double a = inv[t], b = inv[t + d];
      const int32_t v = __ldcs(g + ttc_off(t, t + d, p.ld, p.nb));
      acc += static_cast<double>(v) * (a * b);
      cnt += (a != 0.0 && b != 0.0);
    }
  } else {
    const float* c = p.cf32 + r * p.ring_stride;
#pragma unroll 4
    for (int64_t t = t_begin; t < t_end; ++t) {
      acc += static_cast<double>(__ldcs(c + ttc_off(t, t + d, p.ld, p.nb)));
      ++cnt;
    }
  }
  const int64_t o = (static_cast<int64_t>(r) * p.n_seg + s) * p.n_frames + d;
  p.partial[o] = acc;
  p.pcount[o] = cnt;
}

__global__ void k_g2_final(G2Params p) {
  const int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (d >= p.n_frames) return;
  double acc = 0.0;
  int64_t cnt = 0;
  for (int s = 0; s < p.n_seg; ++s) {
    const int64_t o = (static_cast<int64_t>(r) * p.n_seg + s) * p.n_frames + d;
    if (static_cast<int64_t>(s) * p.seg < p.n_frames - d) {
      acc += p.partial[o];
      cnt += p.pcount[o];
    }
  }
  p.g2[r * p.g2_ld + d] = cnt > 0 ? acc / static_cast<double>(cnt) : 0.0;
  p.counts[r * p.g2_ld + d] = cnt;
}

// Full symmetric readback of one ring: out(i,j) from the upper triangle
// (i <= j) of the source, through a 32 x 33 shared tile so that lower-
// triangle tiles are read coalesced and written transposed.
__global__ void k_expand(ExpandParams p, int src_mode) {
  __shared__ double tile[32][33];
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32;
  const bool lower = i0 > j0;  // whole tile below the diagonal (tiles are aligned)
  // source tile origin in the upper triangle
  const int64_t si0 = lower ? j0 : i0, sj0 = lower ? i0 : j0;
  for (int rr = threadIdx.y; rr < 32; rr += blockDim.y) {
    const int64_t si = si0 + rr, sj = sj0 + threadIdx.x;
    double v = 0.0;
    if (si < p.n && sj < p.n) {
      // inside a diagonal tile the lower half is taken from its mirror
      const int64_t a = si <= sj ? si : sj, b = si <= sj ? sj : si;
      if (src_mode == 0) {
        const int32_t g = p.gram[ttc_off(a, b, p.ld, p.nb)];
        v = p.out_dtype == 2 ? static_cast<double>(g)
                             : static_cast<double>(g) * (p.inv[a] * p.inv[b]);
      } else {
        v = static_cast<double>(p.cf32[ttc_off(a, b, p.ld, p.nb)]);
      }
    }
    tile[rr][threadIdx.x] = v;
  }
  __syncthreads();
  for (int rr = threadIdx.y; rr < 32; rr += blockDim.y) {
    const int64_t i = i0 + rr, j = j0 + threadIdx.x;
    if (i >= p.n || j >= p.n) continue;
    const double v = lower ? tile[threadIdx.x][rr] : tile[rr][threadIdx.x];
    const int64_t o = i * p.out_ld + j;
    if (p.out_dtype == 0)
      static_cast<double*>(p.out)[o] = v;
    else if (p.out_dtype == 1)
      static_cast<float*>(p.out)[o] = static_cast<float>(v);
    else
      static_cast<int32_t*>(p.out)[o] = static_cast<int32_t>(v);
  }
}

// Fold of the K2/K4 epilogue's per-tile diagonal sums (fused g2), in two
// fixed-order passes.  A tile (half-tile row ib, column block jb) adds to
// lag d = 128 delta + e - 127 with delta = 2 jb - ib in [-1, 2 nbj - 2] and
// e its diagonal.  Pass 1 (k_g2_runs, one block per (delta, ring), one
// thread per diagonal e) sums the run of tiles of each delta in ascending
// ib: 384 consecutive partials per tile, coalesced.  Pass 2 (k_g2_fold, one
// thread per lag) adds its <= 3 runs in ascending delta.  (One thread per
// lag walking every tile: 27 us at C2; the walk split over 4 warps 19-21 us
// -- latency-bound; the two passes 16-18 us in ncu, ~4 us less in the step.
// Summing each run in k_gram2 by the CTA completing it stalled the
// epilogue: 4x slower.)
// Both passes are launched as programmatic dependents (of the Gram kernel,
// then of pass 1): the grid is set up while its predecessor drains and waits
// for it here before reading its output.
__device__ __forceinline__ void g2_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <bool SINGLE>
__global__ void __launch_bounds__(384) k_g2_runs(G2FoldParams p) {
  g2_pdl_wait();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t delta = static_cast<int64_t>(blockIdx.x) - 1;
  const int r = blockIdx.y, e = threadIdx.x;
  const int64_t ring_off = static_cast<int64_t>(r) * p.tiles_per_ring * 384;
  const float2* part = p.g2_partial + ring_off;
  const float* part1 = reinterpret_cast<const float*>(p.g2_partial) + ring_off;
  // (delta + ib) even; jb = (delta + ib) / 2 < nbj  <=>  ib < 2 nbj - delta
  const int ib0 = static_cast<int>(delta & 1);
  const int ib_end = static_cast<int>(min(static_cast<int64_t>(p.nbi), 2 * p.nbj - delta));
  double acc = 0.0;
  if (e < 383 && ib0 < ib_end) {
    // element offset of (ib, diagonal e) in the ring's tiles: rows ib hold
    // nbj - ib / 2 tiles, and jb - ib / 2 is constant along the run, so
    // o(ib + 2) = o(ib) + (2 nbj - ib) * 384
    const int nbj = static_cast<int>(p.nbj);
    const int jrel = static_cast<int>((delta + ib0) / 2) - (ib0 >> 1);
    int o = ((ib0 ? nbj : 0) + jrel) * 384 + e;
    // batches of 16 predicated loads issued back to back (a runtime-count
    // loop left the remainder iterations as dependent L2 round trips)
    constexpr int U = 16;
    for (int ib1 = ib0; ib1 < ib_end; ib1 += 2 * U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ib = ib1 + 2 * u;
        v[u] = 0.0;
        if (ib < ib_end) {
          if (SINGLE) {
            v[u] = static_cast<double>(part1[o]);
          } else {
            const float2 hl = part[o];
            v[u] = static_cast<double>(hl.x) + static_cast<double>(hl.y);
          }
        }
        o += (2 * nbj - ib) * 384;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u];
    }
  }
  p.runs[(static_cast<int64_t>(r) * 2 * p.nbj + blockIdx.x) * 384 + e] = acc;
}

__global__ void __launch_bounds__(128) k_g2_fold(G2FoldParams p) {
  g2_pdl_wait();
  __shared__ double part_sum[4][32];
  __shared__ long long part_cnt[4][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t d = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  const int r = blockIdx.y;
  const bool live = d < p.n_frames;
  double acc = 0.0;
  if (live && w == 0) {
    // delta range: ceil((d-255)/128) .. floor((d+127)/128), at most 3 runs
    const int64_t dlo = (d - 255 >= 0) ? (d - 255 + 127) / 128 : -((255 - d) / 128);
    const int64_t dhi = (d + 127) / 128;
    const double* runs = p.runs + static_cast<int64_t>(r) * 2 * p.nbj * 384;
    for (int64_t delta = max(dlo, static_cast<int64_t>(-1)); delta <= dhi; ++delta) {
      const int dl = static_cast<int>(d - 128 * delta + 127);
      if (dl < 0 || dl >= 383 || delta > 2 * p.nbj - 2) continue;
      acc += runs[(delta + 1) * 384 + dl];
    }
  }
  // valid pairs: sum_t nz(t) nz(t+d), t <= T-1-d (integer: split freely)
  int64_t cnt = 0;
  const int64_t last = p.n_frames - 1 - d;
  if (live) {
    if (p.zero_count[r] == 0) {
      if (w == 0) cnt = last + 1;  // no zero-norm frame in this ring
    } else {
      const uint32_t* W = p.nz_bits + static_cast<int64_t>(r) * p.nz_words;
      for (int i = w; i < p.nz_words; i += 4) {
        const int64_t t0 = 32ll * i;
        if (t0 > last) break;
        const int64_t sft = t0 + d;
        const int w0 = static_cast<int>(sft >> 5), sh = static_cast<int>(sft & 31);
        const uint32_t lo = w0 < p.nz_words ? W[w0] : 0u;
        const uint32_t hi = w0 + 1 < p.nz_words ? W[w0 + 1] : 0u;
        uint32_t m = W[i] & __funnelshift_r(lo, hi, sh);
        const int64_t lim = last - t0;
        if (lim < 31) m &= (2u << lim) - 1u;
        cnt += __popc(m);
      }
    }
  }
  part_sum[w][lane] = acc;
  part_cnt[w][lane] = cnt;
  __syncthreads();
  if (w == 0 && live) {
    const double sum = (part_sum[0][lane] + part_sum[1][lane]) +
                       (part_sum[2][lane] + part_sum[3][lane]);
    const int64_t c = part_cnt[0][lane] + part_cnt[1][lane] + part_cnt[2][lane] + part_cnt[3][lane];
    p.g2[r * p.g2_ld + d] = c > 0 ? sum / static_cast<double>(c) : 0.0;
    p.counts[r * p.g2_ld + d] = c;
  }
}

// Streaming g2: running lag sums / pair counts.
__global__ void k_g2_div(const double* sum, const int64_t* cnt, double* out, int64_t n) {
  const int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d < n) out[d] = cnt[d] > 0 ? sum[d] / static_cast<double>(cnt[d]) : 0.0;
}

// Block b of ring r takes rows b, b + REL_BLOCKS, ... of the upper triangle
// (balanced: row a has n - a entries); off-diagonal entries count twice.
__global__ void __launch_bounds__(256) k_rel_error(RelErrParams p) {
  __shared__ double2 red[256];
  const int r = blockIdx.y;
  const int32_t* g = p.gram + r * p.ring_stride;
  const float* cf = p.cgram + r * p.ring_stride;
  const double* inv = p.inv + static_cast<int64_t>(r) * p.inv_ld;
  double num = 0.0, den = 0.0;
  for (int64_t a = blockIdx.x; a < p.n; a += REL_BLOCKS) {
    const double ia = inv[a];
    for (int64_t b = a + threadIdx.x; b < p.n; b += blockDim.x) {
      const int64_t o = ttc_off(a, b, p.ld, p.nb);
      const double c = static_cast<double>(g[o]) * (ia * inv[b]);
      const double e = c - static_cast<double>(cf[o]);
      const double w = a == b ? 1.0 : 2.0;
      num += w * e * e;
      den += w * c * c;
    }
  }
  red[threadIdx.x] = make_double2(num, den);
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) {
      red[threadIdx.x].x += red[threadIdx.x + o].x;
      red[threadIdx.x].y += red[threadIdx.x + o].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) p.partial[static_cast<int64_t>(r) * REL_BLOCKS + blockIdx.x] = red[0];
}

__global__ void k_rel_error_fin(RelErrParams p) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p.n_rings) return;
  double num = 0.0, den = 0.0;
  for (int b = 0; b < REL_BLOCKS; ++b) {
    num += p.partial[static_cast<int64_t>(r) * REL_BLOCKS + b].x;
    den += p.partial[static_cast<int64_t>(r) * REL_BLOCKS + b].y;
  }
  p.out[r] = den > 0.0 ? sqrt(num / den) : -1.0;  // -1: all-zero reference TTC
}

}  // namespace

cudaError_t launch_rel_error(const RelErrParams& p, cudaStream_t s) {
  k_rel_error<<<dim3(REL_BLOCKS, p.n_rings), 256, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_rel_error_fin<<<(p.n_rings + 127) / 128, 128, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_g2_div(const double* sum, const int64_t* cnt, double* out, int64_t n,
                          cudaStream_t s) {
  k_g2_div<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(sum, cnt, out, n);
  return cudaGetLastError();
}

template <typename K>
static cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, cudaStream_t s, const G2FoldParams& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

cudaError_t launch_g2_fold(const G2FoldParams& p, cudaStream_t s) {
  const dim3 rg(static_cast<unsigned>(2 * p.nbj), p.n_rings);
  cudaError_t e = p.single ? launch_pdl(k_g2_runs<true>, rg, dim3(384), s, p)
                           : launch_pdl(k_g2_runs<false>, rg, dim3(384), s, p);
  if (e != cudaSuccess) return e;
  const dim3 grid(static_cast<unsigned>((p.n_frames + 31) / 32), p.n_rings);
  return launch_pdl(k_g2_fold, grid, dim3(128), s, p);
}

cudaError_t launch_g2(const G2Params& p, int mode, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((p.n_frames + 127) / 128), p.n_seg, p.n_rings);
  if (mode == 0)
    k_g2_partial<0><<<grid, 128, 0, s>>>(p);
  else
    k_g2_partial<1><<<grid, 128, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2grid(static_cast<unsigned>((p.n_frames + 127) / 128), p.n_rings);
  k_g2_final<<<g2grid, 128, 0, s>>>(p);
  return cudaGetLastError();
}

// Upper-triangle rows [row0, row1) of one ring packed row after row (row i
// holds columns i .. n-1): the TTC tile sink's staging.  Same entry
// expressions as k_expand.
__global__ void k_pack_upper(ExpandParams p, int src_mode, int64_t row0) {
  const int64_t i = row0 + blockIdx.x;
  if (i >= p.n) return;
  const int64_t off = (i - row0) * p.n - ((i * (i - 1)) / 2 - (row0 * (row0 - 1)) / 2);
  for (int64_t j = i + threadIdx.x; j < p.n; j += blockDim.x) {
    const int64_t o = off + (j - i);
    if (src_mode == 0) {
      const int32_t g = p.gram[ttc_off(i, j, p.ld, p.nb)];
      if (p.out_dtype == 2)
        static_cast<int32_t*>(p.out)[o] = g;
      else
        static_cast<double*>(p.out)[o] = static_cast<double>(g) * (p.inv[i] * p.inv[j]);
    } else {
      static_cast<float*>(p.out)[o] = p.cf32[ttc_off(i, j, p.ld, p.nb)];
    }
  }
}

cudaError_t launch_pack_upper(const ExpandParams& p, int src_mode, int64_t row0, int64_t rows,
                              cudaStream_t s) {
  k_pack_upper<<<static_cast<unsigned>(rows), 256, 0, s>>>(p, src_mode, row0);
  return cudaGetLastError();
}

cudaError_t launch_expand(const ExpandParams& p, int src_mode, cudaStream_t s) {
  const unsigned nt = static_cast<unsigned>((p.n + 31) / 32);
  dim3 grid(nt, nt);
  dim3 block(32, 8);
  k_expand<<<grid, block, 0, s>>>(p, src_mode);
  return cudaGetLastError();
}

}  // namespace xg
