// k_basis.cu -- K9: the encoding basis V_K built on the device (setup of the
// compressed path; the reference's gram_svd, src/linalg.cpp:279-439, called
// by encoder_from_rows, src/encoder.cpp:13-28).
//
//   S = G / (|x_i| |x_j|)       G = the exact int32 Gram of the training frames (K2)
//   S = U diag(l) U^T           parallel-order two-sided Jacobi (this file)
//   W = Xn^T U                  f64 GEMM over the ring-major u8 frames (this file)
//   sigma_j = |W_j|, rank, 2x orthonormalisation (Gram on the device, the k x k
//   Cholesky on the host), sign fix -- orchestrated in xg_api.cu.
//
// Jacobi.  The reference sweeps the pairs (p, q) cyclically by rows
// (linalg.cpp:184-230), one rotation at a time.  Here a sweep is n-1 steps of
// the round-robin ("circle") ordering: every step rotates n/2 disjoint pairs at
// once, so one step is one elementwise pass over A and V.  The rotation of a
// pair uses the reference's formulas and threshold verbatim (theta, t, c, s;
// skip when a_pq == 0 or |a_pq| <= tol sqrt(|a_pp a_qq|); a_pp - t a_pq,
// a_qq + t a_pq, a_pq = 0).  A is held in a "slot" layout: at step s the pair
// k occupies slots (2k, 2k+1), so a pair's 2 x 2 block is contiguous, and
// each step writes its output straight into the next step's slot layout.
// Only the upper pair blocks are computed; each is written with its mirror,
// so A stays bitwise symmetric.
#include <cuda_runtime.h>

#include <cstdint>

#include "xg_kernels.h"

namespace xg {

namespace {

constexpr int PT = 16;  // pairs per tile edge (32 x 32 elements)

struct Rot {
  double c, s, t;
  int rot;
};

// The reference's rotation of pair (p, q) (linalg.cpp:191-205).
__device__ __forceinline__ Rot pair_rotation(const double* a, int np, int pair, double tol) {
  const int p = 2 * pair, q = p + 1;
  const double apq = a[(int64_t)p * np + q];
  Rot r{1.0, 0.0, 0.0, 0};
  if (apq == 0.0) return r;
  const double app = a[(int64_t)p * np + p], aqq = a[(int64_t)q * np + q];
  const double scale = sqrt(fabs(app) * fabs(aqq));
  if (fabs(apq) <= tol * scale) return r;
  const double theta = (aqq - app) / (2.0 * apq);
  const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
  r.c = 1.0 / sqrt(t * t + 1.0);
  r.s = t * r.c;
  r.t = t;
  r.rot = 1;
  return r;
}

// grid.x: [0, nA) upper pair tiles of A, then [nA, nA + nV) tiles of V.
__global__ void __launch_bounds__(256) k_jacobi_step(JacParams p) {
  const int ring = blockIdx.y;
  JacState& st = p.state[ring];
  if (!st.active) return;
  const int np = p.np, half = np >> 1;
  const int ntp = (half + PT - 1) / PT;
  const int nA = ntp * (ntp + 1) / 2;
  const int64_t rs = (int64_t)np * np;
  const double* a = p.a_in + ring * rs;
  const double tol = st.tol;
  const int s = p.step, s1 = (p.step + 1) % (np - 1);
  __shared__ Rot rot_r[PT], rot_c[PT];
  __shared__ int ns_r[2 * PT], ns_c[2 * PT];
  const int tid = threadIdx.x;
  int bx = blockIdx.x;
  if (bx < nA) {
    // upper tile (ti, tj), ti <= tj
    int ti = 0;
    while (bx >= ntp - ti) {
      bx -= ntp - ti;
      ++ti;
    }
    const int tj = ti + bx;
    if (tid < 2 * PT) {
      const int which = tid / PT, l = tid % PT;
      const int pair = (which ? tj : ti) * PT + l;
      if (pair < half) {
        const Rot r = pair_rotation(a, np, pair, tol);
        if (which) {
          rot_c[l] = r;
        } else {
          rot_r[l] = r;
          if (r.rot && ti == tj) st.rotated = 1;  // each pair flagged once (diagonal tile)
        }
        int* ns = which ? ns_c : ns_r;
        ns[2 * l] = index_slot(slot_index(2 * pair, s, np), s1, np);
        ns[2 * l + 1] = index_slot(slot_index(2 * pair + 1, s, np), s1, np);
      }
    }
    __syncthreads();
    const int la = tid / PT, lb = tid % PT;
    const int pa = ti * PT + la, pb = tj * PT + lb;
    if (pa >= half || pb >= half || pa > pb) return;
    double* o = p.a_out + ring * rs;
    const int r0 = 2 * pa, c0 = 2 * pb;
    const double2 top = *reinterpret_cast<const double2*>(a + (int64_t)r0 * np + c0);
    const double2 bot = *reinterpret_cast<const double2*>(a + (int64_t)(r0 + 1) * np + c0);
    const int np0 = ns_r[2 * la], nq0 = ns_r[2 * la + 1];
    const int np1 = ns_c[2 * lb], nq1 = ns_c[2 * lb + 1];
    if (pa == pb) {
      const Rot r = rot_r[la];
      double y00 = top.x, y11 = bot.y, y01 = top.y;
      if (r.rot) {
        y00 = top.x - r.t * top.y;
        y11 = bot.y + r.t * top.y;
        y01 = 0.0;
      }
      o[(int64_t)np0 * np + np0] = y00;
      o[(int64_t)nq0 * np + nq0] = y11;
      o[(int64_t)np0 * np + nq0] = y01;
      o[(int64_t)nq0 * np + np0] = y01;
      return;
    }
    const Rot ra = rot_r[la], rb = rot_c[lb];
    // rows (reference: a(p,k) = c a_pk - s a_qk, a(q,k) = s a_pk + c a_qk), then columns
    const double r00 = ra.c * top.x - ra.s * bot.x, r01 = ra.c * top.y - ra.s * bot.y;
    const double r10 = ra.s * top.x + ra.c * bot.x, r11 = ra.s * top.y + ra.c * bot.y;
    const double y00 = rb.c * r00 - rb.s * r01, y01 = rb.s * r00 + rb.c * r01;
    const double y10 = rb.c * r10 - rb.s * r11, y11 = rb.s * r10 + rb.c * r11;
    o[(int64_t)np0 * np + np1] = y00;
    o[(int64_t)np0 * np + nq1] = y01;
    o[(int64_t)nq0 * np + np1] = y10;
    o[(int64_t)nq0 * np + nq1] = y11;
    o[(int64_t)np1 * np + np0] = y00;
    o[(int64_t)nq1 * np + np0] = y01;
    o[(int64_t)np1 * np + nq0] = y10;
    o[(int64_t)nq1 * np + nq0] = y11;
    return;
  }
  // V tile: 16 coordinate rows x 16 pairs (columns 2b, 2b+1)
  bx -= nA;
  const int tb = bx % ntp, tk = bx / ntp;
  if (tid < PT) {
    const int pair = tb * PT + tid;
    if (pair < half) {
      rot_c[tid] = pair_rotation(a, np, pair, tol);
      ns_c[2 * tid] = index_slot(slot_index(2 * pair, s, np), s1, np);
      ns_c[2 * tid + 1] = index_slot(slot_index(2 * pair + 1, s, np), s1, np);
    }
  }
  __syncthreads();
  const int lk = tid / PT, lb = tid % PT;
  const int krow = tk * PT + lk, pb = tb * PT + lb;
  if (krow >= np || pb >= half) return;
  const double2 v = *reinterpret_cast<const double2*>(p.v_in + ring * rs + (int64_t)krow * np + 2 * pb);
  const Rot rb = rot_c[lb];
  double* vo = p.v_out + ring * rs + (int64_t)krow * np;
  // reference: v(k,p) = c v_kp - s v_kq, v(k,q) = s v_kp + c v_kq
  vo[ns_c[2 * lb]] = rb.c * v.x - rb.s * v.y;
  vo[ns_c[2 * lb + 1]] = rb.s * v.x + rb.c * v.y;
}

// S in the slot layout of step 0 + V = I (columns in slots).  Pad indices
// (>= n) are zero rows/columns: their pairs never rotate (a_pq == 0).
__global__ void k_basis_s(BasisSParams p) {
  const int ring = blockIdx.z;
  const int np = p.np;
  const int si = blockIdx.y * 16 + threadIdx.y, sj = blockIdx.x * 16 + threadIdx.x;
  if (si >= np || sj >= np) return;
  const int i = slot_index(si, 0, np), j = slot_index(sj, 0, np);
  const int64_t rs = (int64_t)np * np;
  double v = 0.0;
  if (i < p.n && j < p.n) {
    const int a = min(i, j), b = max(i, j);
    if (p.s64) {
      v = p.s64[(int64_t)ring * p.n * p.n + (int64_t)a * p.n + b];
    } else {
      const int32_t g = p.gram[(int64_t)ring * p.ring_stride + ttc_off(a, b, p.ld, p.nb)];
      const double* inv = p.inv + ring * p.inv_ld;
      v = static_cast<double>(g) * inv[a] * inv[b];
    }
  }
  p.a[ring * rs + (int64_t)si * np + sj] = v;
  // V: row = coordinate si, column = slot sj holding index j
  p.v[ring * rs + (int64_t)si * np + sj] = (si == j) ? 1.0 : 0.0;
}

__global__ void k_jacobi_diag(const double* const* a_ring, double* eig, int np) {
  const int ring = blockIdx.y;
  const int sl = blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= np) return;
  const double* a = a_ring[ring];
  eig[(int64_t)ring * np + slot_index(sl, 0, np)] = a[(int64_t)sl * np + sl];
}

// ------------------------------------------------------------ f64 GEMMs
constexpr int GM = 64, GN = 128, GK = 16;

template <bool B_U8>
__global__ void __launch_bounds__(256) k_dgemm_nn(const DGemmRing* rings) {
  const DGemmRing d = rings[blockIdx.z];
  const int m0 = blockIdx.y * GM, n0 = blockIdx.x * GN;
  if (m0 >= d.m || n0 >= d.n) return;
  __shared__ double as[GK][GM];
  __shared__ double bs[GK][GN];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  double acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < d.k; k0 += GK) {
    // A tile: 64 rows x 16 k (4 per thread), stored k-major
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + 256 * e, r = idx / GK, kk = idx % GK;
      const int gm = m0 + r, gk = k0 + kk;
      as[kk][r] = (gm < d.m && gk < d.k) ? d.a[(int64_t)gm * d.lda + gk] : 0.0;
    }
    // B tile: 16 k x 128 n (8 per thread)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = tid + 256 * e, kk = idx / GN, c = idx % GN;
      const int gk = k0 + kk, gn = n0 + c;
      double v = 0.0;
      if (gk < d.k && gn < d.n) {
        if (B_U8)
          v = static_cast<double>(static_cast<const uint8_t*>(d.b)[(int64_t)gk * d.ldb + gn]);
        else
          v = static_cast<const double*>(d.b)[(int64_t)gk * d.ldb + gn];
      }
      bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      double av[4], bv[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = as[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) bv[j] = bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= d.m) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn < d.n) d.c[(int64_t)gm * d.ldc + gn] = acc[i][j];
    }
  }
}

// Gram partial of one K chunk: P[i][j] = sum_{p in chunk} A[i][p] A[j][p] over
// the upper 64 x 64 tiles (ti <= tj); grid.x = tile pair, grid.y = chunk.
constexpr int SM_T = 64;
__global__ void __launch_bounds__(256) k_dsyrk(const DGemmRing* rings, double* partial,
                                               int64_t part_stride) {
  const DGemmRing d = rings[blockIdx.z];
  const int nt = (d.m + SM_T - 1) / SM_T;
  int bx = blockIdx.x, ti = 0;
  while (ti < nt && bx >= nt - ti) {
    bx -= nt - ti;
    ++ti;
  }
  if (ti >= nt) return;
  const int tj = ti + bx;
  const int64_t p0 = (int64_t)blockIdx.y * SYRK_CHUNK;
  if (p0 >= d.n) return;
  const int64_t p1 = min((int64_t)d.n, p0 + SYRK_CHUNK);
  __shared__ double as[GK][SM_T + 1];
  __shared__ double bs[GK][SM_T + 1];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int i0 = ti * SM_T, j0 = tj * SM_T;
  for (int64_t k0 = p0; k0 < p1; k0 += GK) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + 256 * e, r = idx / GK, kk = idx % GK;
      const int64_t gk = k0 + kk;
      const bool kin = gk < p1;
      as[kk][r] = (i0 + r < d.m && kin) ? d.a[(int64_t)(i0 + r) * d.lda + gk] : 0.0;
      bs[kk][r] = (j0 + r < d.m && kin) ? d.a[(int64_t)(j0 + r) * d.lda + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = as[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* out = partial + blockIdx.z * part_stride + (int64_t)blockIdx.y * d.m * d.m;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = i0 + ty + 16 * i;
    if (gi >= d.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = j0 + tx + 16 * j;
      if (gj < d.m) out[(int64_t)gi * d.m + gj] = acc[i][j];
    }
  }
}

// C[i][j] (i <= j, the upper tiles written by k_dsyrk) = sum over chunks in
// ascending order; ldc = m.
__global__ void k_dsyrk_sum(const DGemmRing* rings, const double* partial, int64_t part_stride) {
  const DGemmRing d = rings[blockIdx.z];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)d.m * d.m) return;
  const int i = e / d.m, j = e % d.m;
  if (i / SM_T > j / SM_T) return;  // lower tiles are never written
  const int nch = (d.n + SYRK_CHUNK - 1) / SYRK_CHUNK;
  const double* src = partial + blockIdx.z * part_stride + e;
  double acc = 0.0;
  for (int c = 0; c < nch; ++c) acc += src[(int64_t)c * d.m * d.m];
  d.c[(int64_t)i * d.ldc + j] = acc;
}

// out[j] = sum_p A[j][p]^2, block per row, fixed-order tree.
__global__ void k_row_norm2(const DGemmRing* rings, double* out, int64_t out_ld) {
  const DGemmRing d = rings[blockIdx.y];
  const int j = blockIdx.x;
  if (j >= d.m) return;
  const double* row = d.a + (int64_t)j * d.lda;
  double acc = 0.0;
  for (int p = threadIdx.x; p < d.n; p += blockDim.x) acc = fma(row[p], row[p], acc);
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.y * out_ld + j] = red[0];
}

__global__ void k_gather_rows(const DGemmRing* rings, const int32_t* idx, const double* scale,
                              int64_t ld_idx) {
  const DGemmRing d = rings[blockIdx.z];
  const int j = blockIdx.y;
  if (j >= d.m) return;
  const int src = idx[blockIdx.z * ld_idx + j];
  const double sc = scale[blockIdx.z * ld_idx + j];
  const double* a = d.a + (int64_t)src * d.lda;
  double* c = d.c + (int64_t)j * d.ldc;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < d.n; p += gridDim.x * blockDim.x)
    c[p] = a[p] * sc;
}

}  // namespace

cudaError_t launch_jacobi_step(const JacParams& p, int n_rings, cudaStream_t s) {
  const int half = p.np / 2, ntp = (half + PT - 1) / PT;
  const int nA = ntp * (ntp + 1) / 2;
  const int nV = ntp * ((p.np + PT - 1) / PT);
  k_jacobi_step<<<dim3(nA + nV, n_rings), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_basis_s(const BasisSParams& p, int n_rings, cudaStream_t s) {
  const int nb = (p.np + 15) / 16;
  k_basis_s<<<dim3(nb, nb, n_rings), dim3(16, 16), 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_jacobi_diag(const double* const* a_ring, double* eig, int np, int n_rings,
                               cudaStream_t s) {
  k_jacobi_diag<<<dim3((np + 127) / 128, n_rings), 128, 0, s>>>(a_ring, eig, np);
  return cudaGetLastError();
}

cudaError_t launch_dgemm_nn(const DGemmRing* d_rings, int n_rings, int max_m, int max_n,
                            bool b_u8, cudaStream_t s) {
  const dim3 grid((max_n + GN - 1) / GN, (max_m + GM - 1) / GM, n_rings);
  if (b_u8)
    k_dgemm_nn<true><<<grid, 256, 0, s>>>(d_rings);
  else
    k_dgemm_nn<false><<<grid, 256, 0, s>>>(d_rings);
  return cudaGetLastError();
}

cudaError_t launch_dsyrk(const DGemmRing* d_rings, int n_rings, int max_m, int max_chunks,
                         double* partial, int64_t part_stride, cudaStream_t s) {
  const int nt = (max_m + SM_T - 1) / SM_T;
  k_dsyrk<<<dim3(nt * (nt + 1) / 2, max_chunks, n_rings), 256, 0, s>>>(d_rings, partial,
                                                                        part_stride);
  return cudaGetLastError();
}

cudaError_t launch_dsyrk_sum(const DGemmRing* d_rings, int n_rings, int max_m, int max_chunks,
                             const double* partial, int64_t part_stride, cudaStream_t s) {
  (void)max_chunks;
  const int64_t e = (int64_t)max_m * max_m;
  k_dsyrk_sum<<<dim3((unsigned)((e + 255) / 256), 1, n_rings), 256, 0, s>>>(d_rings, partial,
                                                                            part_stride);
  return cudaGetLastError();
}

cudaError_t launch_row_norm2(const DGemmRing* d_rings, int n_rings, int max_m, double* out,
                             int64_t out_ld, cudaStream_t s) {
  k_row_norm2<<<dim3(max_m, n_rings), 256, 0, s>>>(d_rings, out, out_ld);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const DGemmRing* d_rings, const int32_t* idx, const double* scale,
                               int64_t ld_idx, int n_rings, int max_m, int max_n, cudaStream_t s) {
  const int bx = (max_n + 255) / 256 < 64 ? (max_n + 255) / 256 : 64;
  k_gather_rows<<<dim3(bx, max_m, n_rings), 256, 0, s>>>(d_rings, idx, scale, ld_idx);
  return cudaGetLastError();
}

}  // namespace xg
