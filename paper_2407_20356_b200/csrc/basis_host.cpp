// basis_host.cpp -- rank-k encoding basis V_K of NON-COUNT f64 training rows
// (host, f64): the untimed setup of the compressed path for data the device
// builder cannot take.  Photon counts (the detector's data) are factorised on
// the device by K9 (k_basis.cu, xg_series_build_basis), which the xpcsvd
// surface routes them to; this file is never on the correlation path.
//
// Follows the reference's Gram-trick SVD (SPEC.md core-linalg gram_svd;
// src/linalg.cpp:184-439) and encoder (src/encoder.cpp:13-60):
//   Xn = row_normalize(X); S = Xn Xn^T; S = U diag(lambda) U^T by cyclic Jacobi
//   with the graded threshold |s_pq| <= tol sqrt(|s_pp s_qq|); W = Xn^T U;
//   sigma_j = |W_j| (measured, not sqrt(lambda)); rank = #{sigma > 1e-12
//   sigma_max}; two modified Gram-Schmidt passes over the kept columns;
//   sign fix: the largest-magnitude entry of every column is positive.
// It is not bit-identical to the reference (different summation order);
// parity is V within 1e-10 after the shared sign convention, pinned in
// tests/test_host.py (test_basis_builder_*).  Rings are independent and
// built on separate threads.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "../../include/xpcs_b200.h"

namespace {

struct Svd {
  int status = XG_OK;
  int64_t bad = -1;      // zero-norm row / achievable rank payload
  std::vector<double> v;  // m x r (row-major)
  std::vector<double> sigma;
  int64_t r = 0;
};

// Cyclic Jacobi on a symmetric n x n matrix (upper triangle), eigenvectors
// accumulated in u (n x n, columns).
void jacobi(std::vector<double>& a, std::vector<double>& u, int64_t n) {
  u.assign(static_cast<size_t>(n * n), 0.0);
  for (int64_t i = 0; i < n; ++i) u[i * n + i] = 1.0;
  double tol = 1e-15;
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool any = false;
    for (int64_t p = 0; p + 1 < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double app = a[p * n + p], aqq = a[q * n + q];
        if (std::fabs(apq) <= tol * std::sqrt(std::fabs(app) * std::fabs(aqq))) continue;
        any = true;
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        a[p * n + p] = app - t * apq;
        a[q * n + q] = aqq + t * apq;
        a[p * n + q] = 0.0;
        // rotate the remaining upper-triangle entries of rows/cols p and q
        for (int64_t k = 0; k < n; ++k) {
          if (k == p || k == q) continue;
          double& akp = k < p ? a[k * n + p] : a[p * n + k];
          double& akq = k < q ? a[k * n + q] : a[q * n + k];
          const double x = akp, y = akq;
          akp = cs * x - sn * y;
          akq = sn * x + cs * y;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double x = u[k * n + p], y = u[k * n + q];
          u[k * n + p] = cs * x - sn * y;
          u[k * n + q] = sn * x + cs * y;
        }
      }
    if (!any) break;
    if (sweep >= 40 && sweep % 10 == 0) tol *= 100.0;
  }
}

Svd gram_svd(const double* x, int64_t n, int64_t m, double rel_tol) {
  Svd out;
  // row normalisation
  std::vector<double> xn(static_cast<size_t>(n * m));
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t p = 0; p < m; ++p) s += x[i * m + p] * x[i * m + p];
    const double nr = std::sqrt(s);
    if (nr == 0.0) {
      out.status = XG_ERR_NORMALIZATION;
      out.bad = i;
      return out;
    }
    for (int64_t p = 0; p < m; ++p) xn[i * m + p] = x[i * m + p] / nr;
  }
  // Gram (upper triangle)
  std::vector<double> a(static_cast<size_t>(n * n), 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) {
      double s = 0.0;
      const double* xi = &xn[i * m];
      const double* xj = &xn[j * m];
      for (int64_t p = 0; p < m; ++p) s += xi[p] * xj[p];
      a[i * n + j] = s;
    }
  std::vector<double> u;
  jacobi(a, u, n);
  // W = Xn^T U  (m x n), sigma_j = |W_j|
  std::vector<double> w(static_cast<size_t>(m * n), 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = 0; p < m; ++p) {
      const double xv = xn[i * m + p];
      if (xv == 0.0) continue;
      double* wr = &w[p * n];
      const double* ur = &u[i * n];
      for (int64_t j = 0; j < n; ++j) wr[j] += xv * ur[j];
    }
  std::vector<double> nrm(n, 0.0);
  for (int64_t p = 0; p < m; ++p)
    for (int64_t j = 0; j < n; ++j) nrm[j] += w[p * n + j] * w[p * n + j];
  for (auto& v : nrm) v = std::sqrt(v);
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t i, int64_t j) { return nrm[i] > nrm[j]; });
  const double smax = nrm[order[0]];
  if (smax == 0.0) {
    out.status = XG_ERR_RANK;
    out.bad = 0;
    return out;
  }
  int64_t r = 0;
  while (r < n && nrm[order[r]] > rel_tol * smax) ++r;
  // kept columns as contiguous vectors, two MGS passes
  std::vector<double> vt(static_cast<size_t>(r * m));
  for (int64_t j = 0; j < r; ++j)
    for (int64_t p = 0; p < m; ++p) vt[j * m + p] = w[p * n + order[j]];
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t j = 0; j < r; ++j) {
      double* vj = &vt[j * m];
      for (int64_t i = 0; i < j; ++i) {
        const double* vi = &vt[i * m];
        double d = 0.0;
        for (int64_t p = 0; p < m; ++p) d += vi[p] * vj[p];
        for (int64_t p = 0; p < m; ++p) vj[p] -= d * vi[p];
      }
      double s = 0.0;
      for (int64_t p = 0; p < m; ++p) s += vj[p] * vj[p];
      s = std::sqrt(s);
      if (s == 0.0) {
        out.status = XG_ERR_RANK;
        out.bad = j;
        return out;
      }
      for (int64_t p = 0; p < m; ++p) vj[p] /= s;
    }
  // sign convention: largest-magnitude entry positive
  for (int64_t j = 0; j < r; ++j) {
    double* vj = &vt[j * m];
    int64_t arg = 0;
    double best = -1.0;
    for (int64_t p = 0; p < m; ++p)
      if (std::fabs(vj[p]) > best) {
        best = std::fabs(vj[p]);
        arg = p;
      }
    if (vj[arg] < 0.0)
      for (int64_t p = 0; p < m; ++p) vj[p] = -vj[p];
  }
  out.r = r;
  out.v.resize(static_cast<size_t>(m * r));
  for (int64_t p = 0; p < m; ++p)
    for (int64_t j = 0; j < r; ++j) out.v[p * r + j] = vt[j * m + p];
  out.sigma.resize(r);
  for (int64_t j = 0; j < r; ++j) out.sigma[j] = nrm[order[j]];
  return out;
}

}  // namespace

extern "C" {

XG_API uint64_t xg_content_hash(const double* v, int64_t m, int64_t k, int32_t mode) {
  uint64_t h = 0xCBF29CE484222325ULL;
  auto feed = [&](const unsigned char* p, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      h ^= p[i];
      h *= 0x100000001B3ULL;
    }
  };
  auto feed_u64 = [&](uint64_t x) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(x >> (8 * i));
    feed(b, 8);
  };
  feed(reinterpret_cast<const unsigned char*>("XENC"), 4);
  const unsigned char md = static_cast<unsigned char>(mode);
  feed(&md, 1);
  feed_u64(static_cast<uint64_t>(m));
  feed_u64(static_cast<uint64_t>(k));
  for (int64_t i = 0; i < m * k; ++i) {
    uint64_t bits;
    std::memcpy(&bits, v + i, 8);
    feed_u64(bits);
  }
  return h;
}

// build_online_from_frames (encoder.cpp:53-60) / build_offline (k = 0: full
// numerical rank) for one ring: training frames x (n x m, f64, mask order).
XG_API int xg_build_basis(const double* x, int64_t n, int64_t m, int32_t k, double* v_out,
                          double* sigma_out, int64_t* rank_out) {
  if (!x || !rank_out || n < 2 || m < 1 || k < 0) return XG_ERR_CONTRACT;
  Svd s = gram_svd(x, n, m, 1e-12);
  *rank_out = s.status == XG_OK ? s.r : s.bad;
  if (s.status != XG_OK) return s.status;
  const int64_t kk = k == 0 ? s.r : k;
  if (kk > s.r) return XG_ERR_RANK;  // achievable rank in *rank_out
  if (v_out)
    for (int64_t p = 0; p < m; ++p)
      for (int64_t j = 0; j < kk; ++j) v_out[p * kk + j] = s.v[p * s.r + j];
  if (sigma_out)
    for (int64_t j = 0; j < s.r; ++j) sigma_out[j] = s.sigma[j];
  return XG_OK;
}

// All rings of a layout-free batch at once, one thread per ring:
// x_ring[r] is n x m_ring[r]; v_ring[r] receives m_ring[r] x k.
XG_API int xg_build_basis_batch(int32_t n_rings, const double* const* x_ring, int64_t n,
                                const int64_t* m_ring, int32_t k, double* const* v_ring,
                                int32_t threads, int64_t* rank_out) {
  std::vector<int> st(n_rings, XG_OK);
  const int nt = std::max(1, threads > 0 ? threads : (int)std::thread::hardware_concurrency());
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; ++w)
    pool.emplace_back([&, w] {
      for (int32_t r = w; r < n_rings; r += nt)
        st[r] = xg_build_basis(x_ring[r], n, m_ring[r], k, v_ring[r], nullptr, &rank_out[r]);
    });
  for (auto& t : pool) t.join();
  for (int32_t r = 0; r < n_rings; ++r)
    if (st[r] != XG_OK) return st[r];
  return XG_OK;
}

}  // extern "C"
