// xg_exact_api.cu -- reference-facing f64 entry points of the C ABI.
//
// One call per reference function, same arguments (row-major f64 host
// buffers), same validation and error taxonomy, and the reference's exact
// floating-point operation order on the device (k_exact.cu), so results are
// the reference's bits.  These are the entries a drop-in xpcs::correlate /
// xpcs::compress built on this library calls; the u8 batch /
// stream API is the high-throughput path for photon counts.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <vector>

#include "../../include/xpcs_b200.h"
#include "xg_kernels.h"

using namespace xg;

namespace {

// Device buffers of the one-shot entries: a per-thread pool of grow-only
// slots (the entries are called in loops by the reference's code -- e.g.
// ttc_extend once per frame -- so no cudaMalloc/cudaFree per call).
struct Pool {
  void* p[8] = {};
  size_t cap[8] = {};
  int device = -1;
  ~Pool() {
    for (void* q : p)
      if (q) cudaFree(q);
  }
};
thread_local Pool g_pool;
thread_local int g_slot = 0;  // next slot of the current entry

template <class T>
struct DBuf {
  T* p = nullptr;
  cudaError_t alloc(size_t n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_pool.device != dev) {  // buffers belong to one device
      for (int i = 0; i < 8; ++i) {
        if (g_pool.p[i]) cudaFree(g_pool.p[i]);
        g_pool.p[i] = nullptr;
        g_pool.cap[i] = 0;
      }
      g_pool.device = dev;
    }
    const int s = g_slot++ & 7;
    const size_t bytes = (n ? n : 1) * sizeof(T);
    if (g_pool.cap[s] < bytes) {
      if (g_pool.p[s]) cudaFree(g_pool.p[s]);
      g_pool.p[s] = nullptr;
      g_pool.cap[s] = 0;
      const cudaError_t e = cudaMalloc(&g_pool.p[s], bytes);
      if (e != cudaSuccess) return e;
      g_pool.cap[s] = bytes;
    }
    p = static_cast<T*>(g_pool.p[s]);
    return cudaSuccess;
  }
};
// every entry starts allocating at slot 0
struct SlotScope {
  SlotScope() { g_slot = 0; }
};

thread_local char g_err[256];
thread_local int64_t g_payload = -1;

int err(int code, const char* msg, int64_t payload = -1) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  g_payload = payload;
  return code;
}

#define XG_TRY(expr)                                                   \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) return err(XG_ERR_CUDA, cudaGetErrorString(_e)); \
  } while (0)

bool finite_all(const double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

}  // namespace

extern "C" {

XG_API const char* xg_f64_last_error(void) { return g_err; }
XG_API int64_t xg_f64_last_payload(void) { return g_payload; }

// ttc_raw (correlate.cpp:19-25): gram(row_normalize(X)).
XG_API int xg_f64_ttc_raw(const double* x, int64_t n, int64_t m, double* out) {
  SlotScope slots_;
  if (!x || !out) return XG_ERR_INVALID;
  if (n < 1 || m < 1) return err(XG_ERR_CONTRACT, "matrix dimensions must be at least 1x1");
  if (n < 2) return err(XG_ERR_CONTRACT, "ttc_raw: need at least 2 frames");
  if (!finite_all(x, n * m)) return err(XG_ERR_CONTRACT, "non-finite matrix entry");
  for (int64_t i = 0; i < n * m; ++i)
    if (x[i] < 0.0) return err(XG_ERR_CONTRACT, "negative intensity in frame series");
  DBuf<double> dx, dxn, dn, dg;
  DBuf<unsigned long long> dbad;
  XG_TRY(dx.alloc(n * m));
  XG_TRY(dxn.alloc(n * m));
  XG_TRY(dn.alloc(n));
  XG_TRY(dg.alloc(n * n));
  XG_TRY(dbad.alloc(1));
  XG_TRY(cudaMemcpy(dx.p, x, n * m * 8, cudaMemcpyHostToDevice));
  XG_TRY(cudaMemset(dbad.p, 0xFF, 8));
  XG_TRY(launch_exact_rownorm(dx.p, n, m, dxn.p, dn.p, dbad.p, 0));
  unsigned long long bad = 0;
  XG_TRY(cudaMemcpy(&bad, dbad.p, 8, cudaMemcpyDeviceToHost));
  if (bad != ULLONG_MAX)
    return err(XG_ERR_NORMALIZATION, "row_normalize: frame has zero norm", (int64_t)bad);
  XG_TRY(launch_exact_gram(dxn.p, n, m, dg.p, 0));
  XG_TRY(cudaMemcpy(out, dg.p, n * n * 8, cudaMemcpyDeviceToHost));
  return XG_OK;
}

// ttc_compressed (correlate.cpp:27-35): gram(Y); lossless = |diag - 1| <= 1e-10.
XG_API int xg_f64_ttc_compressed(const double* y, int64_t n, int64_t k, double* out,
                                 int* lossless) {
  SlotScope slots_;
  if (!y || !out) return XG_ERR_INVALID;
  if (n < 2) return err(XG_ERR_CONTRACT, "ttc_compressed: need at least 2 frames");
  if (k < 1) return err(XG_ERR_CONTRACT, "compressed series needs k >= 1");
  DBuf<double> dy, dg;
  XG_TRY(dy.alloc(n * k));
  XG_TRY(dg.alloc(n * n));
  XG_TRY(cudaMemcpy(dy.p, y, n * k * 8, cudaMemcpyHostToDevice));
  XG_TRY(launch_exact_gram(dy.p, n, k, dg.p, 0));
  XG_TRY(cudaMemcpy(out, dg.p, n * n * 8, cudaMemcpyDeviceToHost));
  if (lossless) {
    *lossless = 1;
    for (int64_t i = 0; i < n; ++i)
      if (std::fabs(out[i * n + i] - 1.0) > 1e-10) *lossless = 0;
  }
  return XG_OK;
}

// ttc_extend (correlate.cpp:37-65): out is (n+1) x (n+1).
XG_API int xg_f64_ttc_extend(const double* g, int64_t n, const double* y, int64_t k,
                             const double* row, double* out, int* lossless) {
  SlotScope slots_;
  if (!g || !y || !row || !out) return XG_ERR_INVALID;
  if (k < 1) return err(XG_ERR_SHAPE, "ttc_extend: new row length does not match k");
  DBuf<double> dg, dy, dr, dout;
  const int64_t n1 = n + 1;
  XG_TRY(dg.alloc(n * n));
  XG_TRY(dy.alloc(n * k));
  XG_TRY(dr.alloc(k));
  XG_TRY(dout.alloc(n1 * n1));
  if (n > 0) {
    XG_TRY(cudaMemcpy(dg.p, g, n * n * 8, cudaMemcpyHostToDevice));
    XG_TRY(cudaMemcpy(dy.p, y, n * k * 8, cudaMemcpyHostToDevice));
  }
  XG_TRY(cudaMemcpy(dr.p, row, k * 8, cudaMemcpyHostToDevice));
  XG_TRY(launch_exact_extend(dg.p, n, dy.p, k, dr.p, dout.p, 0));
  XG_TRY(cudaMemcpy(out, dout.p, n1 * n1 * 8, cudaMemcpyDeviceToHost));
  if (lossless) {
    *lossless = 1;
    for (int64_t i = 0; i < n1; ++i)
      if (std::fabs(out[i * n1 + i] - 1.0) > 1e-10) *lossless = 0;
  }
  return XG_OK;
}

// g2_from_ttc (correlate.cpp:67-85).
XG_API int xg_f64_g2_from_ttc(const double* g, int64_t n, double period, double* lags,
                              double* values, int64_t* counts) {
  SlotScope slots_;
  if (!g || !lags || !values || !counts) return XG_ERR_INVALID;
  if (n < 2) return err(XG_ERR_CONTRACT, "g2_from_ttc: need at least 2 frames");
  if (!(period > 0.0)) return err(XG_ERR_CONTRACT, "g2_from_ttc: frame_period must be positive");
  DBuf<double> dg, dl, dv;
  DBuf<int64_t> dc;
  XG_TRY(dg.alloc(n * n));
  XG_TRY(dl.alloc(n));
  XG_TRY(dv.alloc(n));
  XG_TRY(dc.alloc(n));
  XG_TRY(cudaMemcpy(dg.p, g, n * n * 8, cudaMemcpyHostToDevice));
  XG_TRY(launch_exact_g2(dg.p, n, period, dl.p, dv.p, dc.p, 0));
  XG_TRY(cudaMemcpy(lags, dl.p, n * 8, cudaMemcpyDeviceToHost));
  XG_TRY(cudaMemcpy(values, dv.p, n * 8, cudaMemcpyDeviceToHost));
  XG_TRY(cudaMemcpy(counts, dc.p, n * 8, cudaMemcpyDeviceToHost));
  return XG_OK;
}

// compress_series (compress.cpp:48-81): all norms first (first zero frame
// reported), then every row like compress_frame.  v is m x k.
namespace {
int compress_series_impl(const double* x, const uint8_t* x8, int64_t n, int64_t m,
                         const double* v, int64_t k, double* coeffs, double* norms);
}  // namespace

XG_API int xg_f64_compress_series(const double* x, int64_t n, int64_t m, const double* v,
                                  int64_t k, double* coeffs, double* norms) {
  SlotScope slots_;
  if (!x || !v || !coeffs || !norms) return XG_ERR_INVALID;
  if (k < 1) return err(XG_ERR_CONTRACT, "compress: k must be >= 1");
  if (n == 0) return XG_OK;  // an empty store (compress.cpp:48-81 loops over no frames)
  return compress_series_impl(x, nullptr, n, m, v, k, coeffs, norms);
}

// The same over photon counts the caller packed to u8 (integer counts in
// [0, 255], what the drop-in's compress_series detects): 1 B per pixel over
// PCIe, widened to f64 on the device, then the identical kernels -- the
// coefficients and norms are those of xg_f64_compress_series on the same
// values, bit for bit.
XG_API int xg_f64_compress_series_u8(const uint8_t* x, int64_t n, int64_t m, const double* v,
                                     int64_t k, double* coeffs, double* norms) {
  SlotScope slots_;
  if (!x || !v || !coeffs || !norms) return XG_ERR_INVALID;
  if (k < 1) return err(XG_ERR_CONTRACT, "compress: k must be >= 1");
  if (n == 0) return XG_OK;
  return compress_series_impl(nullptr, x, n, m, v, k, coeffs, norms);
}

namespace {
int compress_series_impl(const double* x, const uint8_t* x8, int64_t n, int64_t m,
                         const double* v, int64_t k, double* coeffs, double* norms) {
  DBuf<double> dx, dxn, dn, dv, dc;
  DBuf<unsigned long long> dbad;
  DBuf<uint8_t> d8;
  XG_TRY(dx.alloc(n * m));
  XG_TRY(dxn.alloc(n * m));
  XG_TRY(dn.alloc(n));
  XG_TRY(dv.alloc(m * k));
  XG_TRY(dc.alloc(n * k));
  XG_TRY(dbad.alloc(1));
  if (x8) {
    XG_TRY(d8.alloc(n * m));
    XG_TRY(cudaMemcpy(d8.p, x8, n * m, cudaMemcpyHostToDevice));
    XG_TRY(launch_exact_widen_u8(d8.p, n * m, dx.p, 0));
  } else {
    XG_TRY(cudaMemcpy(dx.p, x, n * m * 8, cudaMemcpyHostToDevice));
  }
  XG_TRY(cudaMemcpy(dv.p, v, m * k * 8, cudaMemcpyHostToDevice));
  XG_TRY(cudaMemset(dbad.p, 0xFF, 8));
  XG_TRY(launch_exact_rownorm(dx.p, n, m, dxn.p, dn.p, dbad.p, 0));
  unsigned long long bad = 0;
  XG_TRY(cudaMemcpy(&bad, dbad.p, 8, cudaMemcpyDeviceToHost));
  if (bad != ULLONG_MAX)
    return err(XG_ERR_NORMALIZATION, "compress_series: frame has zero norm", (int64_t)bad);
  XG_TRY(launch_exact_project(dxn.p, n, m, dv.p, k, dc.p, 0));
  XG_TRY(cudaMemcpy(coeffs, dc.p, n * k * 8, cudaMemcpyDeviceToHost));
  XG_TRY(cudaMemcpy(norms, dn.p, n * 8, cudaMemcpyDeviceToHost));
  return XG_OK;
}
}  // namespace

// compress_frame (compress.cpp:34-46).
XG_API int xg_f64_compress_frame(const double* frame, int64_t m, const double* v, int64_t k,
                                 double* coeffs, double* norm) {
  SlotScope slots_;
  if (!frame || !v || !coeffs || !norm) return XG_ERR_INVALID;
  const int rc = xg_f64_compress_series(frame, 1, m, v, k, coeffs, norm);
  if (rc == XG_ERR_NORMALIZATION)
    return err(XG_ERR_NORMALIZATION, "compress_frame: frame has zero norm", 0);
  return rc;
}

// ttc_rel_error (correlate.cpp:87-108) over count = N*N entries.
XG_API int xg_f64_ttc_rel_error(const double* a, const double* b, int64_t count, double* out) {
  SlotScope slots_;
  if (!a || !b || !out) return XG_ERR_INVALID;
  DBuf<double> da, db, dr;
  XG_TRY(da.alloc(count));
  XG_TRY(db.alloc(count));
  XG_TRY(dr.alloc(1));
  XG_TRY(cudaMemcpy(da.p, a, count * 8, cudaMemcpyHostToDevice));
  XG_TRY(cudaMemcpy(db.p, b, count * 8, cudaMemcpyHostToDevice));
  XG_TRY(launch_exact_relerr(da.p, db.p, count, dr.p, 0));
  XG_TRY(cudaMemcpy(out, dr.p, 8, cudaMemcpyDeviceToHost));
  if (*out < 0.0) return err(XG_ERR_CONTRACT, "ttc_rel_error: reference TTC is all zero");
  return XG_OK;
}

}  // extern "C"
