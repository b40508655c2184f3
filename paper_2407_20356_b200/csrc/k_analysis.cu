// k_analysis.cu -- analysis consumers of the correlation results on the
// device: ttc_background (analysis.cpp:202-235) over the
// stored TTC tiles, and fit_kww (analysis.cpp:77-172) batched over the rings
// of a series, from the g2 curves already in HBM.  Nothing leaves the device
// but Q numbers per ring.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

// C(a, b) of the stored upper triangle (a <= b): the readback's expression
// (k_expand), so the values equal the host TTC bitwise.
__device__ __forceinline__ double bg_entry(const BgParams& p, int r, int64_t a, int64_t b,
                                           const double* inv) {
  const int64_t o = r * p.ring_stride + ttc_off(a, b, p.ld, p.nb);
  return p.cgram ? static_cast<double>(p.cgram[o])
                 : static_cast<double>(p.gram[o]) * (inv[a] * inv[b]);
}

// Pass 1 (mean) or 2 (squared deviations) over the entries with lag >
// exclusion, upper triangle only (the matrix is symmetric: every sum and
// count doubles, the ratios do not change).  Pairs with a flagged (zero-
// norm) frame are left out, as in g2.  Block b takes rows b, b + BG_BLOCKS,
// ...: fixed partition, fixed-order tree, deterministic.
__global__ void __launch_bounds__(256) k_ttc_bg(BgParams p, int pass) {
  __shared__ double rs[256];
  __shared__ long long rc[256];
  const int r = blockIdx.y;
  const double* inv = p.inv + r * p.inv_ld;
  const double mean = pass == 2 ? p.mean[r] : 0.0;
  double s = 0.0;
  long long cnt = 0;
  for (int64_t a = blockIdx.x; a < p.n; a += BG_BLOCKS) {
    if (inv[a] == 0.0) continue;
    for (int64_t b = a + p.excl + 1 + threadIdx.x; b < p.n; b += blockDim.x) {
      if (inv[b] == 0.0) continue;
      const double v = bg_entry(p, r, a, b, inv);
      if (pass == 1) {
        s += v;
        ++cnt;
      } else {
        const double d = v - mean;
        s += d * d;
      }
    }
  }
  rs[threadIdx.x] = s;
  rc[threadIdx.x] = cnt;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) {
      rs[threadIdx.x] += rs[threadIdx.x + o];
      rc[threadIdx.x] += rc[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.partial[static_cast<int64_t>(r) * BG_BLOCKS + blockIdx.x] =
        make_double2(rs[0], static_cast<double>(rc[0]));
  }
}

__global__ void k_ttc_bg_fin(BgParams p, int pass) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p.n_rings) return;
  double s = 0.0, c = 0.0;
  for (int b = 0; b < BG_BLOCKS; ++b) {
    const double2 v = p.partial[static_cast<int64_t>(r) * BG_BLOCKS + b];
    s += v.x;
    c += v.y;
  }
  if (pass == 1) {
    p.count[r] = static_cast<int64_t>(c);
    p.mean[r] = c > 0.0 ? s / c : 0.0;
  } else {
    const double n = static_cast<double>(p.count[r]);
    p.out[r] = n > 0.0 ? sqrt(s / n) : -1.0;  // -1: no entry outside the band
  }
}

// ---------------------------------------------------------------- fit_kww
// Warp butterfly sum: every lane ends with the same bits (each stage adds
// the same two operands on both partners), so the scalar logic below runs
// identically on all lanes without a broadcast.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ bool solve3(double a[3][3], const double b[3], double out[3]) {
  double m[3][4];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) m[i][j] = a[i][j];
    m[i][3] = b[i];
  }
  for (int col = 0; col < 3; ++col) {
    int pivot = col;
    for (int r = col + 1; r < 3; ++r)
      if (fabs(m[r][col]) > fabs(m[pivot][col])) pivot = r;
    if (m[pivot][col] == 0.0) return false;
    if (pivot != col)
      for (int c = 0; c < 4; ++c) {
        const double t = m[col][c];
        m[col][c] = m[pivot][c];
        m[pivot][c] = t;
      }
    for (int r = 0; r < 3; ++r) {
      if (r == col) continue;
      const double f = m[r][col] / m[col][col];
      for (int c = col; c < 4; ++c) m[r][c] -= f * m[col][c];
    }
  }
  for (int i = 0; i < 3; ++i) out[i] = m[i][3] / m[i][i];
  return true;
}

__device__ double kww_sse(const double* v, int64_t d0, int64_t np, double period, double b,
                          double c, double t0, int lane) {
  double sse = 0.0;
  for (int64_t i = lane; i < np; i += 32) {
    const double lag = static_cast<double>(d0 + i) * period;
    const double r = v[d0 + i] - (b + c * exp(-2.0 * lag / t0));
    sse += r * r;
  }
  return warp_sum(sse);
}

// One warp per ring: the reference's initialisation and damped Gauss-Newton
// verbatim (analysis.cpp:77-172), with the sums over the window's points
// split across the lanes.
__global__ void __launch_bounds__(32) k_fit_kww(KwwParams p) {
  const int r = blockIdx.x, lane = threadIdx.x;
  const double* v = p.g2 + r * p.g2_ld;
  double* out = p.out + 4 * r;
  // window: lags d * period in [min_lag, max_lag] (select_window); the lags
  // increase with d, so it is the run [d0, d1]
  // start from a guess a little below each end, settle by the exact test
  auto below = [&](double lag) -> int64_t {
    const double g = floor(lag / p.period) - 2.0;
    return !(g > 0.0) ? 0 : (g >= static_cast<double>(p.n) ? p.n : static_cast<int64_t>(g));
  };
  int64_t d0 = below(p.min_lag);
  while (d0 < p.n && !(static_cast<double>(d0) * p.period >= p.min_lag)) ++d0;
  int64_t d1 = below(p.max_lag);
  if (d1 < d0) d1 = d0;
  while (d1 < p.n && static_cast<double>(d1) * p.period <= p.max_lag) ++d1;
  const int64_t np = p.min_lag <= p.max_lag ? d1 - d0 : 0;  // points d0 .. d1 - 1
  bool finite = true;
  for (int64_t i = lane; i < np; i += 32)
    if (!isfinite(v[d0 + i])) finite = false;
  finite = __all_sync(0xffffffffu, finite);
  if (!finite || np < 5) {
    if (lane == 0) p.status[r] = 3;
    return;
  }
  // initialisation
  const int64_t tail = np / 10 > 1 ? np / 10 : 1;
  double b = 0.0;
  for (int64_t i = np - tail; i < np; ++i) b += v[d0 + i];  // sequential, as the reference
  b /= static_cast<double>(tail);
  const double c = v[d0] - b;
  if (c <= 0.0) {
    if (lane == 0) p.status[r] = 1;
    return;
  }
  const double e2 = exp(-2.0);
  double t0 = 0.0;
  for (int64_t base = 0; base < np; base += 32) {
    const int64_t i = base + lane;
    const bool hit = i < np && (v[d0 + i] - b) / c < e2;
    const uint32_t m = __ballot_sync(0xffffffffu, hit);
    if (m) {
      t0 = static_cast<double>(d0 + base + __ffs(m) - 1) * p.period;
      break;
    }
  }
  const double lag_first = static_cast<double>(d0) * p.period;
  const double lag_last = static_cast<double>(d0 + np - 1) * p.period;
  if (t0 <= 0.0) t0 = 0.5 * (lag_last - lag_first);
  if (t0 <= 0.0) t0 = lag_last > 0.0 ? lag_last : 1.0;
  // damped Gauss-Newton on (B, C, t0)
  double prm[3] = {b, c, t0};
  double sse = kww_sse(v, d0, np, p.period, prm[0], prm[1], prm[2], lane);
  double mu = 1e-3;
  bool converged = false;
  for (int iter = 0; iter < 200 && !converged; ++iter) {
    double jtj[3][3], jtr[3];
    {
      double a00 = 0, a01 = 0, a02 = 0, a11 = 0, a12 = 0, a22 = 0, r0 = 0, r1 = 0, r2 = 0;
      for (int64_t i = lane; i < np; i += 32) {
        const double t = static_cast<double>(d0 + i) * p.period;
        const double e = exp(-2.0 * t / prm[2]);
        const double res = v[d0 + i] - (prm[0] + prm[1] * e);
        const double j2 = prm[1] * e * 2.0 * t / (prm[2] * prm[2]);
        r0 += res;
        r1 += e * res;
        r2 += j2 * res;
        a00 += 1.0;
        a01 += e;
        a02 += j2;
        a11 += e * e;
        a12 += e * j2;
        a22 += j2 * j2;
      }
      jtr[0] = warp_sum(r0);
      jtr[1] = warp_sum(r1);
      jtr[2] = warp_sum(r2);
      jtj[0][0] = warp_sum(a00);
      jtj[0][1] = jtj[1][0] = warp_sum(a01);
      jtj[0][2] = jtj[2][0] = warp_sum(a02);
      jtj[1][1] = warp_sum(a11);
      jtj[1][2] = jtj[2][1] = warp_sum(a12);
      jtj[2][2] = warp_sum(a22);
    }
    bool stepped = false;
    for (int attempt = 0; attempt < 25; ++attempt) {
      double damped[3][3];
      for (int a = 0; a < 3; ++a)
        for (int q = 0; q < 3; ++q) damped[a][q] = jtj[a][q] + (a == q ? mu * (1.0 + jtj[a][a]) : 0.0);
      double step[3];
      if (!solve3(damped, jtr, step)) {
        mu *= 10.0;
        continue;
      }
      const double cand[3] = {prm[0] + step[0], prm[1] + step[1], prm[2] + step[2]};
      if (!(cand[2] > 0.0) || !isfinite(cand[2])) {
        mu *= 10.0;
        continue;
      }
      const double cand_sse = kww_sse(v, d0, np, p.period, cand[0], cand[1], cand[2], lane);
      if (cand_sse <= sse) {
        double rel = 0.0;
        for (int a = 0; a < 3; ++a) rel = fmax(rel, fabs(step[a]) / fmax(1e-30, fabs(cand[a])));
        for (int a = 0; a < 3; ++a) prm[a] = cand[a];
        sse = cand_sse;
        mu = fmax(mu / 3.0, 1e-14);
        stepped = true;
        if (rel < 1e-10) converged = true;
        break;
      }
      mu *= 10.0;
    }
    if (!stepped) converged = true;  // damping exhausted: stationary point
  }
  if (lane == 0) {
    out[0] = prm[0];
    out[1] = prm[1];
    out[2] = prm[2];
    out[3] = sqrt(sse / static_cast<double>(np));
    p.status[r] = converged ? 0 : 2;
  }
}

}  // namespace

cudaError_t launch_ttc_background(const BgParams& p, cudaStream_t s) {
  for (int pass = 1; pass <= 2; ++pass) {
    k_ttc_bg<<<dim3(BG_BLOCKS, p.n_rings), 256, 0, s>>>(p, pass);
    k_ttc_bg_fin<<<(p.n_rings + 127) / 128, 128, 0, s>>>(p, pass);
  }
  return cudaGetLastError();
}

cudaError_t launch_fit_kww(const KwwParams& p, cudaStream_t s) {
  k_fit_kww<<<p.n_rings, 32, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace xg
