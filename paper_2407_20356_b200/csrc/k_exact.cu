// k_exact.cu -- K9: f64 kernels that reproduce the reference's floating-point
// operation ORDER, so the reference-facing f64 entry points return the
// reference's results bit for bit on the GPU (no FMA contraction: every
// product and sum is an explicit __dmul_rn / __dadd_rn, as the reference's
// Release build -- -O3, no -march -- emits separate mulsd/addsd).
//
//   dot        src/linalg.cpp:93-106   4 interleaved accumulators + tail,
//                                      ((s0+s1)+(s2+s3))+tail
//   gram       src/linalg.cpp:127-156  entry = ascending sum of 16384-pixel
//                                      stripe dots, mirrored
//   row_normalize src/linalg.cpp:441-456  norm = sqrt(dot(x,x)); x / norm
//   project_row   src/compress.cpp:12-22  ascending m, zeros skipped
//   g2_from_ttc   src/correlate.cpp:67-85 sequential ascending-t sum / (N-d)
//   ttc_rel_error src/correlate.cpp:87-108 sequential num/den sums
//
// Parallelism comes from independent output entries (each owns the exact
// sequential chain the reference computes for it); operands are staged in
// shared memory so the chains run at DP-pipe speed.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

constexpr int64_t kStripe = 16384;

// The reference dot over [a, a+n) . [b, b+n) (strided operands allowed).
__device__ __forceinline__ double ref_dot(const double* a, const double* b, int64_t n,
                                         int64_t sa = 1, int64_t sb = 1) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t k = 0;
  for (; k + 4 <= n; k += 4) {
    s0 = __dadd_rn(s0, __dmul_rn(a[k * sa], b[k * sb]));
    s1 = __dadd_rn(s1, __dmul_rn(a[(k + 1) * sa], b[(k + 1) * sb]));
    s2 = __dadd_rn(s2, __dmul_rn(a[(k + 2) * sa], b[(k + 2) * sb]));
    s3 = __dadd_rn(s3, __dmul_rn(a[(k + 3) * sa], b[(k + 3) * sb]));
  }
  double tail = 0.0;
  for (; k < n; ++k) tail = __dadd_rn(tail, __dmul_rn(a[k * sa], b[k * sb]));
  return __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)), tail);
}

// row_normalize: one warp per row.  The warp loads 32 consecutive elements
// per step (coalesced) and squares them in parallel; lane l < 4 owns the
// reference's accumulator s_l (elements k = 4q + l) and adds its 8 products
// of the step in ascending q through shuffles, so every chain is the
// reference's sequential one.  bad[0] = first zero row (atomicMin).
__global__ void __launch_bounds__(256) k_exact_rownorm(const double* x, int64_t n, int64_t m,
                                                       double* norms, unsigned long long* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  const double* row = x + i * m;
  const int64_t body = m / 4 * 4;
  double acc = 0.0;  // lane l < 4: s_l
  for (int64_t k0 = 0; k0 < body; k0 += 32) {
    const int64_t k = k0 + lane;
    const double v = k < body ? row[k] : 0.0;
    const double pr = __dmul_rn(v, v);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double t = __shfl_sync(0xffffffffu, pr, 4 * q + (lane & 3));
      if (k0 + 4 * q + (lane & 3) < body) acc = __dadd_rn(acc, t);
    }
  }
  double tail = 0.0;
  for (int64_t k = body; k < m; ++k) tail = __dadd_rn(tail, __dmul_rn(row[k], row[k]));
  const double s0 = __shfl_sync(0xffffffffu, acc, 0), s1 = __shfl_sync(0xffffffffu, acc, 1);
  const double s2 = __shfl_sync(0xffffffffu, acc, 2), s3 = __shfl_sync(0xffffffffu, acc, 3);
  if (lane == 0) {
    const double nr = sqrt(__dadd_rn(__dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)), tail));
    norms[i] = nr;
    if (nr == 0.0) atomicMin(bad, static_cast<unsigned long long>(i));
  }
}

// Elementwise division pass (coalesced) for the normalised copy.
__global__ void k_exact_divide(const double* x, const double* norms, int64_t n, int64_t m,
                               double* xn) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * m) return;
  const double nr = norms[idx / m];
  xn[idx] = nr == 0.0 ? 0.0 : __ddiv_rn(x[idx], nr);
}

// gram: 32 x 32 output tiles (upper triangle tiles only), each thread one
// entry (i, j); rows staged in shared memory in chunks of 64 elements.  The
// per-entry operation sequence is exactly the reference's: stripe by
// stripe, within a stripe four accumulators over k = 4q + l and a tail.
constexpr int GT = 32;
constexpr int GC = 64;  // chunk (multiple of 4)

__global__ void __launch_bounds__(GT * GT / 4) k_exact_gram(const double* x, int64_t n, int64_t m,
                                                         double* g) {
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;
  __shared__ double si[GT][GC + 1];
  __shared__ double sj[GT][GC + 1];
  // 256 threads, 4 entries each: (ti, tj + 8*e)
  const int tj = threadIdx.x & 31, ti0 = threadIdx.x >> 5;  // ti0 in [0, 8)
  const int64_t j = bj * GT + tj;
  double total[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t s0 = 0; s0 < m; s0 += kStripe) {
    const int64_t len = (m - s0 < kStripe) ? (m - s0) : kStripe;
    const int64_t body = len / 4 * 4;
    double a[4][4];
    double tail[4];
    for (int e = 0; e < 4; ++e) {
      a[e][0] = a[e][1] = a[e][2] = a[e][3] = 0.0;
      tail[e] = 0.0;
    }
    for (int64_t c0 = 0; c0 < len; c0 += GC) {
      const int64_t cl = (len - c0 < GC) ? (len - c0) : GC;
      __syncthreads();
      for (int idx = threadIdx.x; idx < GT * GC; idx += blockDim.x) {
        const int r = idx / GC, k = idx % GC;
        const int64_t gi = bi * GT + r, gj = bj * GT + r;
        si[r][k] = (gi < n && k < cl) ? x[gi * m + s0 + c0 + k] : 0.0;
        sj[r][k] = (gj < n && k < cl) ? x[gj * m + s0 + c0 + k] : 0.0;
      }
      __syncthreads();
      for (int e = 0; e < 4; ++e) {
        const int ti = ti0 + 8 * e;
        for (int k = 0; k < cl; ++k) {
          const int64_t kk = c0 + k;  // index within the stripe
          const double pr = __dmul_rn(si[ti][k], sj[tj][k]);
          if (kk < body)
            a[e][kk & 3] = __dadd_rn(a[e][kk & 3], pr);
          else
            tail[e] = __dadd_rn(tail[e], pr);
        }
      }
    }
    for (int e = 0; e < 4; ++e) {
      const double d = __dadd_rn(__dadd_rn(__dadd_rn(a[e][0], a[e][1]), __dadd_rn(a[e][2], a[e][3])),
                                 tail[e]);
      total[e] = __dadd_rn(total[e], d);  // g(i,j) += dot(stripe)
    }
  }
  for (int e = 0; e < 4; ++e) {
    const int64_t i = bi * GT + ti0 + 8 * e;
    if (i < n && j < n && j >= i) {
      g[i * n + j] = total[e];
      g[j * n + i] = total[e];
    }
  }
}

// New TTC column of ttc_extend: out(i, n) = dot(y_i, row), corner dot(row,row),
// history block copied.  out is (n+1) x (n+1).
__global__ void k_exact_extend(const double* g, int64_t n, const double* y, int64_t k,
                               const double* row, double* out) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n1 = n + 1;
  if (idx < n * n) {
    const int64_t i = idx / n, jj = idx % n;
    out[i * n1 + jj] = g[idx];
  }
  if (idx <= n) {
    const double v = idx < n ? ref_dot(y + idx * k, row, k) : ref_dot(row, row, k);
    out[idx * n1 + n] = v;
    out[n * n1 + idx] = v;
  }
}

// g2: thread per lag d, sequential ascending t (coalesced across the warp).
__global__ void k_exact_g2(const double* g, int64_t n, double period, double* lags,
                           double* values, int64_t* counts) {
  const int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d >= n) return;
  double acc = 0.0;
  for (int64_t t = 0; t + d < n; ++t) acc = __dadd_rn(acc, g[t * n + t + d]);
  lags[d] = __dmul_rn(static_cast<double>(d), period);
  counts[d] = n - d;
  values[d] = __ddiv_rn(acc, static_cast<double>(n - d));
}

// project_row for every (frame, coefficient): ascending m over the frame's
// nonzero pixels (compress.cpp:17 skips zeros), coeffs += xn * v.
__global__ void k_exact_project(const double* xn, int64_t n, int64_t m, const double* v,
                                int64_t k, double* coeffs) {
  const int64_t i = blockIdx.x;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * 1024;  // this block's coefficients
  __shared__ double sx[256];
  __shared__ int32_t sp[256];
  __shared__ int cnt;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // coefficients j0 + threadIdx.x + 256 * e
  for (int64_t p0 = 0; p0 < m; p0 += 256) {
    __syncthreads();
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int64_t p = p0 + threadIdx.x;
    const double xv = p < m ? xn[i * m + p] : 0.0;
    // ordered compaction: ballot prefix within warps, warp offsets in order
    const unsigned msk = __ballot_sync(0xffffffffu, xv != 0.0);
    __shared__ int wofs[8];
    if ((threadIdx.x & 31) == 0) wofs[threadIdx.x >> 5] = __popc(msk);
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < 8; ++w) {
        const int c = wofs[w];
        wofs[w] = s;
        s += c;
      }
      cnt = s;
    }
    __syncthreads();
    if (xv != 0.0) {
      const int pos = wofs[threadIdx.x >> 5] + __popc(msk & ((1u << (threadIdx.x & 31)) - 1u));
      sx[pos] = xv;
      sp[pos] = static_cast<int32_t>(p);
    }
    __syncthreads();
    for (int e = 0; e < 4; ++e) {
      const int64_t j = j0 + threadIdx.x + 256 * e;
      if (j >= k) break;
      double a = acc[e];
      for (int q = 0; q < cnt; ++q) a = __dadd_rn(a, __dmul_rn(sx[q], v[sp[q] * k + j]));
      acc[e] = a;
    }
  }
  for (int e = 0; e < 4; ++e) {
    const int64_t j = j0 + threadIdx.x + 256 * e;
    if (j < k) coeffs[i * k + j] = acc[e];
  }
}

// ttc_rel_error: the reference's single sequential pass (two chains, num
// and den, in ascending entry order -- its bits need that order).  One warp:
// 32 consecutive entries per step are loaded coalesced (4 steps in flight)
// and their products formed in parallel; every lane then runs both chains
// over the step's products, taken by shuffles in ascending order, so only
// the two dependent DADDs per entry remain on the critical path.
__global__ void __launch_bounds__(32) k_exact_relerr(const double* a, const double* b,
                                                     int64_t count, double* out) {
  const int lane = threadIdx.x;
  double num = 0.0, den = 0.0;
  for (int64_t i0 = 0; i0 < count; i0 += 128) {
    double dd[4], aa[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + 32 * u + lane;
      const double av = i < count ? a[i] : 0.0, bv = i < count ? b[i] : 0.0;
      const double d = __dadd_rn(av, -bv);
      dd[u] = __dmul_rn(d, d);
      aa[u] = __dmul_rn(av, av);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        const double pd = __shfl_sync(0xffffffffu, dd[u], l);
        const double pa = __shfl_sync(0xffffffffu, aa[u], l);
        if (i0 + 32 * u + l < count) {
          num = __dadd_rn(num, pd);
          den = __dadd_rn(den, pa);
        }
      }
  }
  if (lane == 0) out[0] = den == 0.0 ? -1.0 : sqrt(__ddiv_rn(num, den));
}

// u8 photon counts -> f64 (exact): the drop-in ships counts over PCIe at 1 B
// per pixel instead of 8 and widens them here, 16 per thread.
__global__ void k_exact_widen_u8(const uint8_t* x, int64_t count, double* out) {
  const int64_t i0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16;
  if (i0 + 16 <= count && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const uint4 w = *reinterpret_cast<const uint4*>(x + i0);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int b = 0; b < 4; ++b) out[i0 + 4 * q + b] = static_cast<double>((ws[q] >> (8 * b)) & 0xFFu);
  } else {
    for (int64_t i = i0; i < count && i < i0 + 16; ++i) out[i] = static_cast<double>(x[i]);
  }
}

}  // namespace

cudaError_t launch_exact_widen_u8(const uint8_t* x, int64_t count, double* out, cudaStream_t s) {
  if (count < 1) return cudaSuccess;
  k_exact_widen_u8<<<static_cast<unsigned>((count + 16 * 256 - 1) / (16 * 256)), 256, 0, s>>>(x, count,
                                                                                          out);
  return cudaGetLastError();
}

cudaError_t launch_exact_rownorm(const double* x, int64_t n, int64_t m, double* xn, double* norms,
                                 unsigned long long* bad, cudaStream_t s) {
  if (n < 1) return cudaSuccess;
  k_exact_rownorm<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(x, n, m, norms, bad);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !xn) return e;
  k_exact_divide<<<static_cast<unsigned>((n * m + 255) / 256), 256, 0, s>>>(x, norms, n, m, xn);
  return cudaGetLastError();
}

cudaError_t launch_exact_gram(const double* x, int64_t n, int64_t m, double* g, cudaStream_t s) {
  const unsigned nt = static_cast<unsigned>((n + GT - 1) / GT);
  k_exact_gram<<<dim3(nt, nt), GT * GT / 4, 0, s>>>(x, n, m, g);
  return cudaGetLastError();
}

cudaError_t launch_exact_extend(const double* g, int64_t n, const double* y, int64_t k,
                                const double* row, double* out, cudaStream_t s) {
  const int64_t work = n * n > n + 1 ? n * n : n + 1;
  k_exact_extend<<<static_cast<unsigned>((work + 255) / 256), 256, 0, s>>>(g, n, y, k, row, out);
  return cudaGetLastError();
}

cudaError_t launch_exact_g2(const double* g, int64_t n, double period, double* lags,
                            double* values, int64_t* counts, cudaStream_t s) {
  k_exact_g2<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(g, n, period, lags, values,
                                                                   counts);
  return cudaGetLastError();
}

cudaError_t launch_exact_project(const double* xn, int64_t n, int64_t m, const double* v,
                                 int64_t k, double* coeffs, cudaStream_t s) {
  if (n < 1 || k < 1) return cudaSuccess;
  k_exact_project<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>((k + 1023) / 1024)), 256,
                    0, s>>>(xn, n, m, v, k, coeffs);
  return cudaGetLastError();
}

cudaError_t launch_exact_relerr(const double* a, const double* b, int64_t count, double* out,
                                cudaStream_t s) {
  k_exact_relerr<<<1, 32, 0, s>>>(a, b, count, out);
  return cudaGetLastError();
}

}  // namespace xg
