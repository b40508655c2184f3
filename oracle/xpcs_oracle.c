/*
 * xpcs_oracle.c -- CPU restatement of the XPCS correlation hot path of the
 * arXiv 2407.20356 reference (`xpcsvd`), used ONLY as a test checker.
 *
 * TEST INFRASTRUCTURE.  Nothing in the product (paper_2407_20356_b200/) may
 * link, load or call this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * thing that checks (or is timed beside) the CUDA path.
 *
 * Every arithmetic routine reproduces the reference's floating-point
 * operation ORDER so that, compiled like the reference (-O3, no -march,
 * no FMA contraction), results are bitwise identical to it.  This is pinned
 * by tests/test_oracle.py against oracle/_ref (the reference compiled from
 * /root/reference by oracle/Makefile) and against tests/golden/.
 *
 * Citations are /root/reference/proj/<file>:<line>.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define XO_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ RNG --
 * Counter-based splitmix64 stream: include/xpcsvd/rng.hpp:8-22,
 * src/rng.cpp:12-44.  out(b, i) = mix(b + (i + 1) * golden). */
static const uint64_t XO_GOLDEN = 0x9E3779B97F4A7C15ULL;
static const uint64_t XO_STREAM = 0xD6E8FEB86659FD93ULL;

static inline uint64_t xo_mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

XO_API uint64_t xo_rng_substream(uint64_t base, uint64_t tag) {
  return xo_mix(base ^ (tag * XO_STREAM)); /* src/rng.cpp:20-22 */
}
XO_API uint64_t xo_rng_bits(uint64_t base, uint64_t index) {
  return xo_mix(base + (index + 1) * XO_GOLDEN); /* src/rng.cpp:24-26 */
}
XO_API double xo_rng_uniform(uint64_t base, uint64_t index) {
  /* (bits >> 11) + 1 scaled by 2^-53: never zero (src/rng.cpp:28-30). */
  return (double)((xo_rng_bits(base, index) >> 11) + 1) * 0x1.0p-53;
}
XO_API double xo_rng_normal(uint64_t base, uint64_t index) {
  /* Box-Muller on (2i, 2i+1) (src/rng.cpp:32-36). */
  const double u1 = xo_rng_uniform(base, 2 * index);
  const double u2 = xo_rng_uniform(base, 2 * index + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}
XO_API double xo_rng_exponential(uint64_t base, uint64_t index) {
  return -log(xo_rng_uniform(base, index)); /* src/rng.cpp:38-40 */
}

/* test fixture of the reference tests: tests/test_helpers.hpp:24-31
 * (positive matrix = exponential draws of substream 98). */
XO_API void xo_random_positive_matrix(int64_t rows, int64_t cols, uint64_t seed,
                                      double* out) {
  const uint64_t s = xo_rng_substream(seed, 98);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = xo_rng_exponential(s, (uint64_t)i);
}
/* tests/test_helpers.hpp:15-22 (normal draws of substream 99). */
XO_API void xo_random_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  const uint64_t s = xo_rng_substream(seed, 99);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = xo_rng_normal(s, (uint64_t)i);
}

/* --------------------------------------------------------------- linalg --
 * Fixed-order dot: four interleaved accumulators, combined
 * ((s0+s1)+(s2+s3))+tail (src/linalg.cpp:93-106). */
XO_API double xo_dot(const double* a, const double* b, int64_t n) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t k = 0;
  for (; k + 4 <= n; k += 4)
    for (int l = 0; l < 4; ++l) acc[l] += a[k + l] * b[k + l];
  double rest = 0.0;
  while (k < n) {
    rest += a[k] * b[k];
    ++k;
  }
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + rest;
}

/* X X^T, upper triangle then mirrored (src/linalg.cpp:127-156).  Entry (i,j)
 * is the ascending sum over 16384-pixel stripes of a stripe dot; the row
 * blocking and thread split of the reference never change the bits. */
#define XO_STRIPE 16384
XO_API void xo_gram(const double* x, int64_t n, int64_t m, double* g) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) {
      double s = 0.0;
      for (int64_t p0 = 0; p0 < m; p0 += XO_STRIPE) {
        const int64_t len = (m - p0 < XO_STRIPE) ? (m - p0) : XO_STRIPE;
        s += xo_dot(x + i * m + p0, x + j * m + p0, len);
      }
      g[i * n + j] = s;
      g[j * n + i] = s;
    }
}

/* Exact integer Gram of u8 counts (int64 accumulation).  Equal to xo_gram of
 * the same counts as f64 whenever the sums stay below 2^53. */
XO_API void xo_gram_u8(const uint8_t* x, int64_t n, int64_t m, int64_t* g) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) {
      int64_t s = 0;
      const uint8_t* a = x + i * m;
      const uint8_t* b = x + j * m;
      for (int64_t p = 0; p < m; ++p) s += (int64_t)a[p] * (int64_t)b[p];
      g[i * n + j] = s;
      g[j * n + i] = s;
    }
}

/* Row normalisation (src/linalg.cpp:441-456): norm = sqrt(dot(row,row)),
 * then one division per entry.  Returns -1, or the first zero row. */
XO_API int64_t xo_row_normalize(const double* x, int64_t n, int64_t m, double* out,
                                double* norms) {
  for (int64_t i = 0; i < n; ++i) {
    const double nr = sqrt(xo_dot(x + i * m, x + i * m, m));
    if (nr == 0.0) return i;
    norms[i] = nr;
    for (int64_t p = 0; p < m; ++p) out[i * m + p] = x[i * m + p] / nr;
  }
  return -1;
}

/* ------------------------------------------------------------ correlate --
 * ttc_raw = gram(row_normalize(X)) (src/correlate.cpp:19-25).  Returns -1 or
 * the zero-norm frame; -2 when n < 2 (ContractError in the reference). */
XO_API int64_t xo_ttc_raw(const double* x, int64_t n, int64_t m, double* g) {
  if (n < 2) return -2;
  double* xn = (double*)malloc(sizeof(double) * (size_t)(n * m));
  double* norms = (double*)malloc(sizeof(double) * (size_t)n);
  const int64_t bad = xo_row_normalize(x, n, m, xn, norms);
  if (bad < 0) xo_gram(xn, n, m, g);
  free(xn);
  free(norms);
  return bad;
}

/* lossless test of the reference: |g_ii - 1| <= 1e-10 (src/correlate.cpp:10-15). */
static int xo_unit_diagonal(const double* g, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (fabs(g[i * n + i] - 1.0) > 1e-10) return 0;
  return 1;
}

/* ttc_compressed = gram(Y) (src/correlate.cpp:27-35); k <= 16384 so a single
 * stripe, i.e. one plain dot per entry.  Returns the lossless flag. */
XO_API int xo_ttc_compressed(const double* y, int64_t n, int64_t k, double* g) {
  xo_gram(y, n, k, g);
  return xo_unit_diagonal(g, n);
}

/* ttc_extend (src/correlate.cpp:37-65): copy, n dots of the history rows
 * with the new row, corner = dot(new,new).  out is (n+1)x(n+1). */
XO_API int xo_ttc_extend(const double* g, int64_t n, const double* y, int64_t k,
                         const double* row, double* out) {
  const int64_t n1 = n + 1;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) out[i * n1 + j] = g[i * n + j];
  for (int64_t i = 0; i < n; ++i) {
    const double v = xo_dot(y + i * k, row, k);
    out[i * n1 + n] = v;
    out[n * n1 + i] = v;
  }
  out[n * n1 + n] = xo_dot(row, row, k);
  return xo_unit_diagonal(out, n1);
}

/* g2 (src/correlate.cpp:67-85): sequential ascending-t sum along diagonal d,
 * divided by N-d; lags d*period; counts N-d. */
XO_API void xo_g2_from_ttc(const double* g, int64_t n, double period, double* lags,
                           double* values, int64_t* counts) {
  for (int64_t d = 0; d < n; ++d) {
    double s = 0.0;
    for (int64_t t = 0; t + d < n; ++t) s += g[t * n + t + d];
    lags[d] = (double)d * period;
    counts[d] = n - d;
    values[d] = s / (double)(n - d);
  }
}

/* |G - G~|_F / |G|_F (src/correlate.cpp:87-108); -1 when |G|_F == 0. */
XO_API double xo_ttc_rel_error(const double* a, const double* b, int64_t count) {
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const double d = a[i] - b[i];
    num += d * d;
    den += a[i] * a[i];
  }
  if (den == 0.0) return -1.0;
  return sqrt(num / den);
}

/* ------------------------------------------------------------- compress --
 * project_row (src/compress.cpp:12-22): ascending pixel order, zero pixels
 * skipped, coeffs[j] += xn[m] * V(m, j). */
static void xo_project_row(const double* xn, const double* v, int64_t m, int64_t k,
                           double* coeffs) {
  for (int64_t j = 0; j < k; ++j) coeffs[j] = 0.0;
  for (int64_t p = 0; p < m; ++p) {
    const double xv = xn[p];
    if (xv == 0.0) continue;
    const double* vr = v + p * k;
    for (int64_t j = 0; j < k; ++j) coeffs[j] += xv * vr[j];
  }
}

/* compress_frame (src/compress.cpp:34-46).  Returns 0, or 1 for a zero frame. */
XO_API int xo_compress_frame(const double* frame, int64_t m, const double* v, int64_t k,
                             double* coeffs, double* norm_out) {
  const double nr = sqrt(xo_dot(frame, frame, m));
  if (nr == 0.0) return 1;
  double* xn = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t p = 0; p < m; ++p) xn[p] = frame[p] / nr;
  xo_project_row(xn, v, m, k, coeffs);
  free(xn);
  *norm_out = nr;
  return 0;
}

/* compress_series (src/compress.cpp:48-81): all norms first (first zero frame
 * reported), then each row exactly like compress_frame.  Returns -1 or the
 * zero frame index. */
XO_API int64_t xo_compress_series(const double* x, int64_t n, int64_t m, const double* v,
                                  int64_t k, double* coeffs, double* norms) {
  for (int64_t i = 0; i < n; ++i) {
    norms[i] = sqrt(xo_dot(x + i * m, x + i * m, m));
    if (norms[i] == 0.0) return i;
  }
  double* xn = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = 0; p < m; ++p) xn[p] = x[i * m + p] / norms[i];
    xo_project_row(xn, v, m, k, coeffs + i * k);
  }
  free(xn);
  return -1;
}

/* ---------------------------------------------------------------- model --
 * apply_mask (src/model.cpp:42-59): pure column gather in mask order. */
XO_API void xo_apply_mask(const double* x, int64_t n, int64_t m_full, const int64_t* idx,
                          int64_t m_q, double* out) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m_q; ++j) out[i * m_q + j] = x[i * m_full + idx[j]];
}

/* ---------------------------------------------- synthetic speckle data --
 * The BASELINE generator; the reference has no Poisson
 * sampler or per-pixel rate, so this extends gen_relaxation
 * (src/synth.cpp:54-90) on top of CounterRng:
 *   ring(p) = min(Q-1, floor(r Q / r_max)), r = |p - c|, c = ((W-1)/2,(H-1)/2),
 *             r_max = corner distance;
 *   field f_t = rho f_{t-1} + sqrt(1-rho^2) eps_t, complex eps with
 *             E|eps|^2 = 1 (Re, Im ~ N(0, 1/2)), f_0 = eps_0 (stationary);
 *   rho(p) = exp(-Gamma(p)): gamma_mode 0 -> Gamma = a * r^2,
 *             gamma_mode 1 -> Gamma = a * 10^(3 q / (Q-1)) (per ring);
 *   counts = Poisson(mu |f|^2) by CDF inversion of a uniform, clipped to 255.
 * Streams: substream 1 = Re eps, 2 = Im eps, 3 = Poisson uniform; index
 * t*M + p.  The GPU generator (csrc/synth.cu) follows the same recipe but
 * libm differs, so parity always feeds the bytes produced HERE to both sides. */
XO_API void xo_ring_map(int64_t h, int64_t w, int64_t q, int32_t* ring, double* radius) {
  const double cy = 0.5 * (double)(h - 1), cx = 0.5 * (double)(w - 1);
  const double rmax = sqrt(cx * cx + cy * cy);
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      const double dy = (double)y - cy, dx = (double)x - cx;
      const double r = sqrt(dx * dx + dy * dy);
      int64_t b = (int64_t)floor(r * (double)q / rmax);
      if (b > q - 1) b = q - 1;
      ring[y * w + x] = (int32_t)b;
      if (radius) radius[y * w + x] = r;
    }
}

static inline uint8_t xo_poisson(double lam, double u) {
  /* CDF inversion: smallest k with F(k) >= u. */
  double p = exp(-lam), f = p;
  int k = 0;
  while (u > f && k < 255) {
    ++k;
    p *= lam / (double)k;
    f += p;
    if (p == 0.0 && f < u) { /* tail underflow: stop at the current k */
      break;
    }
  }
  return (uint8_t)k;
}

/* Same generator restricted to a pixel subset (every pixel is an independent
 * chain indexed by t*M + p): out is t_frames x n_pix, column j = pixel pix[j]. */
XO_API void xo_gen_speckle_pixels(int64_t t_frames, int64_t h, int64_t w, int64_t q, double mu,
                                  int gamma_mode, double gamma_a, uint64_t seed,
                                  const int64_t* pix, int64_t n_pix, uint8_t* out) {
  const int64_t m = h * w;
  const double cy = 0.5 * (double)(h - 1), cx = 0.5 * (double)(w - 1);
  const double rmax = sqrt(cx * cx + cy * cy);
  const uint64_t s_re = xo_rng_substream(seed, 1);
  const uint64_t s_im = xo_rng_substream(seed, 2);
  const uint64_t s_po = xo_rng_substream(seed, 3);
  const double half = sqrt(0.5);
  for (int64_t j = 0; j < n_pix; ++j) {
    const int64_t p = pix[j];
    const double dy = (double)(p / w) - cy, dx = (double)(p % w) - cx;
    const double r = sqrt(dx * dx + dy * dy);
    int64_t b = (int64_t)floor(r * (double)q / rmax);
    if (b > q - 1) b = q - 1;
    const double gam = gamma_mode == 0
                           ? gamma_a * r * r
                           : gamma_a * pow(10.0, 3.0 * (double)b / (double)(q > 1 ? q - 1 : 1));
    const double rho = exp(-gam);
    double fr = 0.0, fi = 0.0;
    for (int64_t t = 0; t < t_frames; ++t) {
      const uint64_t idx = (uint64_t)(t * m + p);
      const double er = half * xo_rng_normal(s_re, idx);
      const double ei = half * xo_rng_normal(s_im, idx);
      if (t == 0) {
        fr = er;
        fi = ei;
      } else {
        const double c = sqrt(1.0 - rho * rho);
        fr = rho * fr + c * er;
        fi = rho * fi + c * ei;
      }
      out[t * n_pix + j] = xo_poisson(mu * (fr * fr + fi * fi), xo_rng_uniform(s_po, idx));
    }
  }
}

XO_API void xo_gen_speckle(int64_t t_frames, int64_t h, int64_t w, int64_t q, double mu,
                           int gamma_mode, double gamma_a, uint64_t seed, uint8_t* out) {
  const int64_t m = h * w;
  int32_t* ring = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
  double* radius = (double*)malloc(sizeof(double) * (size_t)m);
  double* rho = (double*)malloc(sizeof(double) * (size_t)m);
  double* fre = (double*)malloc(sizeof(double) * (size_t)m);
  double* fim = (double*)malloc(sizeof(double) * (size_t)m);
  xo_ring_map(h, w, q, ring, radius);
  const uint64_t s_re = xo_rng_substream(seed, 1);
  const uint64_t s_im = xo_rng_substream(seed, 2);
  const uint64_t s_po = xo_rng_substream(seed, 3);
  const double half = sqrt(0.5);
  for (int64_t p = 0; p < m; ++p) {
    double gam;
    if (gamma_mode == 0)
      gam = gamma_a * radius[p] * radius[p];
    else
      gam = gamma_a * pow(10.0, 3.0 * (double)ring[p] / (double)(q > 1 ? q - 1 : 1));
    rho[p] = exp(-gam);
  }
  for (int64_t t = 0; t < t_frames; ++t) {
    for (int64_t p = 0; p < m; ++p) {
      const uint64_t idx = (uint64_t)(t * m + p);
      const double er = half * xo_rng_normal(s_re, idx);
      const double ei = half * xo_rng_normal(s_im, idx);
      if (t == 0) {
        fre[p] = er;
        fim[p] = ei;
      } else {
        const double r = rho[p], c = sqrt(1.0 - r * r);
        fre[p] = r * fre[p] + c * er;
        fim[p] = r * fim[p] + c * ei;
      }
      const double lam = mu * (fre[p] * fre[p] + fim[p] * fim[p]);
      out[t * m + p] = xo_poisson(lam, xo_rng_uniform(s_po, idx));
    }
  }
  free(ring);
  free(radius);
  free(rho);
  free(fre);
  free(fim);
}
