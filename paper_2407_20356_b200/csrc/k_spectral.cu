// k_spectral.cu -- g2 of the compressed path without forming C~ (g2-only
// mode for series whose C~ cannot be stored: T = 65536).
//
// g2_from_ttc(ttc_compressed(Y)) (correlate.cpp:27-35, 67-85) sums, per lag
// d, C~(t, t+d) = y_t . y_{t+d} = sum_kappa y_kappa(t) y_kappa(t+d): the sum of
// the k coefficient series' autocorrelations.  Autocorrelations are products
// in the Fourier domain, so the O(T^2 k) Gram becomes O(k T log T):
//
//   * coefficient pairs become one complex series z = y_{2m} + i y_{2m+1}:
//     Re sum_t conj(z(t)) z(t+d) = r_{2m}(d) + r_{2m+1}(d), so k/2 FFTs;
//   * time is cut into blocks of B = 4096 frames, each zero-padded to
//     L = 8192 (linear, not circular, correlation); block pair (a <= b)
//     gives the lags (b - a) B + tau, tau in (-B, B), from
//     IFFT(sum_m conj(Z_{a,m}) Z_{b,m}) -- the sum over m runs in the
//     frequency domain, one inverse FFT per block pair;
//   * the lags are folded over block pairs in a fixed order (deterministic),
//     divided by the pair counts (closed form T - d, or the nonzero-frame
//     bitmask when a ring has flagged frames).
//
// Everything is f64 (the FFT's error is ~log2(L) eps of sum |y|^2, far
// inside the compressed path's 1e-5 contract; C~ itself is only
// fp32-accurate).  The FFT: radix-4 passes (+ one radix-2), 8192 points in
// padded shared memory (148 KB),
// 1024 threads, twiddles from a table built once with sincospi.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

#ifndef XG_SPT
#define XG_SPT 1024
#endif
constexpr int SPL = SPEC_L, SPLOG = 13, SPT = XG_SPT;
static_assert((1 << SPLOG) == SPL, "L must be 2^13");

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ int bitrev13(int j) { return static_cast<int>(__brev(static_cast<unsigned>(j)) >> (32 - SPLOG)); }

// Shared-memory slot of element i: one pad slot per 8 elements and one per
// 256, so the radix-4 passes' strided quads (stride 1, 4, 16 elements) and
// the bit-reversed scatter each hit all 32 banks (an unpadded layout had 2-
// to 32-way conflicts: L1 94% busy, 0.87 G conflicts per C5 launch).
__device__ __forceinline__ int pidx(int i) { return i + (i >> 3) + (i >> 8); }
constexpr int SPL_PAD = SPL + SPL / 8 + SPL / 256;

// In-place DIT over shared memory (input already in bit-reversed order):
// stages s and s + 1 fused into radix-4 passes (the two radix-2 stages'
// exact operations, half the barriers and shared-memory round trips), the
// last stage radix-2.  inverse: conjugate twiddles (no 1/L scaling here).
__device__ void fft_smem(double2* x, const double2* __restrict__ tw, bool inverse) {
  int s = 1;
  for (; s + 1 <= SPLOG; s += 2) {
    const int h = 1 << (s - 1);
    const int st1 = SPL >> s, st2 = SPL >> (s + 1);
    __syncthreads();
    for (int q = threadIdx.x; q < SPL / 4; q += SPT) {
      const int grp = q >> (s - 1), pos = q & (h - 1);
      const int i0 = (grp << (s + 1)) + pos;
      double2 w1 = __ldg(tw + pos * st1), w2a = __ldg(tw + pos * st2), w2b = __ldg(tw + (pos + h) * st2);
      if (inverse) {
        w1.y = -w1.y;
        w2a.y = -w2a.y;
        w2b.y = -w2b.y;
      }
      const double2 x0 = x[pidx(i0)], x1 = x[pidx(i0 + h)], x2 = x[pidx(i0 + 2 * h)],
                    x3 = x[pidx(i0 + 3 * h)];
      // stage s: (i0, i0 + h) and (i0 + 2h, i0 + 3h), twiddle w1
      const double2 t1 = cmul(w1, x1), t3 = cmul(w1, x3);
      const double2 a = make_double2(x0.x + t1.x, x0.y + t1.y), b = make_double2(x0.x - t1.x, x0.y - t1.y);
      const double2 c = make_double2(x2.x + t3.x, x2.y + t3.y), d = make_double2(x2.x - t3.x, x2.y - t3.y);
      // stage s + 1: (i0, i0 + 2h) twiddle w2a, (i0 + h, i0 + 3h) twiddle w2b
      const double2 tc = cmul(w2a, c), td = cmul(w2b, d);
      x[pidx(i0)] = make_double2(a.x + tc.x, a.y + tc.y);
      x[pidx(i0 + 2 * h)] = make_double2(a.x - tc.x, a.y - tc.y);
      x[pidx(i0 + h)] = make_double2(b.x + td.x, b.y + td.y);
      x[pidx(i0 + 3 * h)] = make_double2(b.x - td.x, b.y - td.y);
    }
  }
  for (; s <= SPLOG; ++s) {  // the remaining radix-2 stage
    const int half = 1 << (s - 1);
    const int step = SPL >> s;
    __syncthreads();
    for (int bf = threadIdx.x; bf < SPL / 2; bf += SPT) {
      const int grp = bf >> (s - 1), pos = bf & (half - 1);
      const int i = (grp << s) + pos, j = i + half;
      double2 w = __ldg(tw + pos * step);
      if (inverse) w.y = -w.y;
      const double2 t = cmul(w, x[pidx(j)]);
      const double2 u = x[pidx(i)];
      x[pidx(i)] = make_double2(u.x + t.x, u.y + t.y);
      x[pidx(j)] = make_double2(u.x - t.x, u.y - t.y);
    }
  }
  __syncthreads();
}

__global__ void k_spec_twiddles(double2* tw) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= SPL / 2) return;
  double sn, cs;
  sincospi(-2.0 * static_cast<double>(j) / SPL, &sn, &cs);
  tw[j] = make_double2(cs, sn);
}

// grid (pairs of coefficients m, blocks a, rings)
__global__ void __launch_bounds__(SPT) k_spec_fwd(SpecParams p) {
  extern __shared__ double2 xs[];
  const int m = blockIdx.x, a = blockIdx.y, r = blockIdx.z;
  const int c0 = 2 * m, c1 = 2 * m + 1;
  const double* y = p.y + static_cast<int64_t>(r) * p.y_ld * p.k;
  // the block's frames (strided reads of two coefficient columns, all
  // issued before any store), zero padding above B
  constexpr int PER = SPEC_B / SPT;
  double2 z[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = threadIdx.x + u * SPT;
    const int64_t t = static_cast<int64_t>(a) * SPEC_B + j;
    z[u] = make_double2(0.0, 0.0);
    if (t < p.n) {
      z[u].x = y[t * p.k + c0];
      if (c1 < p.k) z[u].y = y[t * p.k + c1];
    }
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) xs[pidx(bitrev13(threadIdx.x + u * SPT))] = z[u];
  for (int j = SPEC_B + threadIdx.x; j < SPL; j += SPT) xs[pidx(bitrev13(j))] = make_double2(0.0, 0.0);
  fft_smem(xs, p.tw, false);
  double2* out = p.spec + ((static_cast<int64_t>(r) * p.nb + a) * p.nm + m) * SPL;
  for (int j = threadIdx.x; j < SPL; j += SPT) out[j] = xs[pidx(j)];
}

// grid (block pairs, rings): the pair's cross-spectrum summed over the
// coefficient pairs, inverse FFT, real part / L -> corr[ring][pair][tau]
__global__ void __launch_bounds__(SPT) k_spec_pair(SpecParams p) {
  extern __shared__ double2 xs[];
  const int pr = blockIdx.x, r = blockIdx.y;
  // pair index -> (a, b), a <= b, pairs ordered a-major
  int a = 0, rem = pr;
  while (rem >= p.nb - a) {
    rem -= p.nb - a;
    ++a;
  }
  const int b = a + rem;
  const double2* sa = p.spec + (static_cast<int64_t>(r) * p.nb + a) * p.nm * SPL;
  const double2* sb = p.spec + (static_cast<int64_t>(r) * p.nb + b) * p.nm * SPL;
  for (int f = threadIdx.x; f < SPL; f += SPT) {
    double2 acc = make_double2(0.0, 0.0);
    for (int m = 0; m < p.nm; ++m) {  // fixed order
      const double2 u = sa[static_cast<int64_t>(m) * SPL + f], v = sb[static_cast<int64_t>(m) * SPL + f];
      acc.x += u.x * v.x + u.y * v.y;  // conj(u) v
      acc.y += u.x * v.y - u.y * v.x;
    }
    xs[pidx(bitrev13(f))] = acc;
  }
  fft_smem(xs, p.tw, true);
  double* out = p.corr + (static_cast<int64_t>(r) * p.npairs + pr) * SPL;
  for (int j = threadIdx.x; j < SPL; j += SPT) out[j] = xs[pidx(j)].x * (1.0 / SPL);
}

// grid (ceil(n / 256), rings): lag d sums the block pairs (a, a + D) with
// D in {floor(d / B), floor(d / B) + 1}, tau = d - D B, in (D, a) order
__global__ void k_spec_fold(SpecParams p) {
  const int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (d >= p.n) return;
  const double* corr = p.corr + static_cast<int64_t>(r) * p.npairs * SPL;
  double acc = 0.0;
  const int64_t d0 = d / SPEC_B;
  for (int64_t D = d0; D <= d0 + 1 && D < p.nb; ++D) {
    const int64_t tau = d - D * SPEC_B;  // in (-B, B)
    if (D == 0 && tau < 0) continue;
    const int64_t idx = tau >= 0 ? tau : SPL + tau;
    for (int64_t a = 0; a + D < p.nb; ++a) {
      const int64_t pr = a * p.nb - a * (a - 1) / 2 + D;
      acc += corr[pr * SPL + idx];
    }
  }
  // valid pairs: sum_t nz(t) nz(t+d) (k_g2_fold's count)
  int64_t cnt = 0;
  const int64_t last = p.n - 1 - d;
  if (p.zero_count[r] == 0) {
    cnt = last + 1;
  } else {
    const uint32_t* W = p.nz_bits + static_cast<int64_t>(r) * p.nz_words;
    for (int i = 0; i < p.nz_words; ++i) {
      const int64_t t0 = 32ll * i;
      if (t0 > last) break;
      const int64_t sft = t0 + d;
      const int w0 = static_cast<int>(sft >> 5), sh = static_cast<int>(sft & 31);
      const uint32_t lo = w0 < p.nz_words ? W[w0] : 0u;
      const uint32_t hi = w0 + 1 < p.nz_words ? W[w0 + 1] : 0u;
      uint32_t mm = W[i] & __funnelshift_r(lo, hi, sh);
      const int64_t lim = last - t0;
      if (lim < 31) mm &= (2u << lim) - 1u;
      cnt += __popc(mm);
    }
  }
  p.g2[r * p.g2_ld + d] = cnt > 0 ? acc / static_cast<double>(cnt) : 0.0;
  p.counts[r * p.g2_ld + d] = cnt;
}

}  // namespace

size_t spectral_scratch_bytes(int n_rings, int64_t n, int k) {
  const int64_t nb = (n + SPEC_B - 1) / SPEC_B, nm = (k + 1) / 2;
  const int64_t npairs = nb * (nb + 1) / 2;
  return static_cast<size_t>(SPL / 2) * 16 + static_cast<size_t>(n_rings) * nb * nm * SPL * 16 +
         static_cast<size_t>(n_rings) * npairs * SPL * 8;
}

cudaError_t launch_spectral_g2(SpecParams p, void* scratch, cudaStream_t s) {
  p.nb = static_cast<int32_t>((p.n + SPEC_B - 1) / SPEC_B);
  p.nm = (p.k + 1) / 2;
  p.npairs = p.nb * (p.nb + 1) / 2;
  uint8_t* base = static_cast<uint8_t*>(scratch);
  p.tw = reinterpret_cast<double2*>(base);
  p.spec = reinterpret_cast<double2*>(base + static_cast<size_t>(SPL / 2) * 16);
  p.corr = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(p.spec) +
                                     static_cast<size_t>(p.n_rings) * p.nb * p.nm * SPL * 16);
  const size_t smem = static_cast<size_t>(SPL_PAD) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(k_spec_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_spec_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_spec_twiddles<<<(SPL / 2 + 255) / 256, 256, 0, s>>>(const_cast<double2*>(p.tw));
  k_spec_fwd<<<dim3(p.nm, p.nb, p.n_rings), SPT, smem, s>>>(p);
  k_spec_pair<<<dim3(p.npairs, p.n_rings), SPT, smem, s>>>(p);
  k_spec_fold<<<dim3(static_cast<unsigned>((p.n + 255) / 256), p.n_rings), 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace xg
