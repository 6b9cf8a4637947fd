// Per-matrix kernels of the hexmc hot path on sm_100a.
//
//  * fused_smem_kernel: one CTA per (mask, k) Bloch matrix, everything in shared memory
//    (N <= HX_SMEM_MAX_N): compaction -> assembly -> tridiagonalisation -> bisection -> IDOS.
//  * global_solve_kernel: same pipeline with the matrix in an HBM workspace slice (any N; also the
//    general (H, S) pencil via Cholesky).  The large-N two-stage path lives in hx_band.cu.
//  * finalize_kernel: prefix-sum of the integer full-weight counts + fixed-point transition sums
//    -> per-mask IDOS curves (qoi.py:96-102: values = counts / area, weights 1/nk).
#include <cuda_runtime.h>
#include <stdint.h>

#include "hx_dense.cuh"
#include "hx_kernels.cuh"

namespace hx {

__device__ __forceinline__ void emit_eigs_and_idos(const CellDev& c, const GridDev& g, const double* lam, int d,
                                                   int* diff_row, unsigned long long* trans_row, double* eig_out,
                                                   int N, int* st, bool sharp) {
  // pencil map; the commuting map is monotone (decreasing when t - s*eps0 < 0)
  const bool rev = (c.pencil == 1) && (c.t - c.s * c.eps0 < 0.0);
  bool bad = false;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const double E = pencil_map(c, lam[i]);
    bad |= !isfinite(E);
    if (sharp) sharp_state(g, E, diff_row);
    else idos_state(g, E, diff_row, trans_row);
    if (eig_out) eig_out[rev ? d - 1 - i : i] = E;
  }
  if (eig_out)
    for (int i = d + threadIdx.x; i < N; i += blockDim.x) eig_out[i] = __longlong_as_double(0x7ff8000000000000ll);
  if (bad) atomicMax(st, 2);
}

// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fused_smem_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                         const uint64_t* __restrict__ masks, GridDev g, int* diff,
                                                         unsigned long long* trans, double* eigs, int* status,
                                                         int sharp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = c.N;
  const int ld = N | 1;  // odd row stride: conflict-free column walks
  const int64_t mat = blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  double* R = reinterpret_cast<double*>(smem_raw);
  double2* v = reinterpret_cast<double2*>(R + (((size_t)N * ld + 1) & ~(size_t)1));
  double2* y = v + N;
  double* diag = reinterpret_cast<double*>(y + N);
  double* e2 = diag + N;
  double* lam = e2 + N;
  double* red = lam + N;                                   // 96
  int* new_idx = reinterpret_cast<int*>(red + 96);         // N
  int* cnt = new_idx + N;                                  // ceil(N/32)

  int* st = status + mat;
  if (threadIdx.x == 0) *st = 0;
  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (d == 0) {
    if (threadIdx.x == 0) *st = 3;
    if (eigs)
      for (int i = threadIdx.x; i < N; i += blockDim.x) eigs[mat * N + i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  assemble_packed(c, new_idx, d, kpts[kk], R, ld);
  tridiag_packed(R, ld, d, diag, e2, v, y, red);
  bisect_all(diag, e2, d, lam, red);
  emit_eigs_and_idos(c, g, lam, d, diff + mk * (g.npts + 1), trans + mk * g.npts, eigs ? eigs + mat * N : nullptr, N,
                     st, sharp != 0);
}

size_t fused_smem_bytes(int N) {
  const int ld = N | 1;
  return (((size_t)N * ld + 1) & ~(size_t)1) * 8 + (size_t)N * 16 * 2 + (size_t)N * 8 * 3 + 96 * 8 + (size_t)N * 4 + ((N + 31) / 32) * 4 + 16;
}

// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) global_solve_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                           const uint64_t* __restrict__ masks, GridDev g, int* diff,
                                                           unsigned long long* trans, double* eigs, int* status,
                                                           int64_t mat0, unsigned char* ws, size_t ws_stride,
                                                           int sharp) {
  __shared__ double red[96];
  __shared__ int cnt[(HX_MAX_N + 31) / 32];
  const int N = c.N;
  const int64_t mat = mat0 + blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  unsigned char* w = ws + (size_t)blockIdx.x * ws_stride;
  double2* A = reinterpret_cast<double2*>(w);
  double2* B = A + (size_t)N * N;
  const bool general = c.pencil == 2;
  double2* v = general ? B + (size_t)N * N : B;
  double2* y = v + N;
  double* diag = reinterpret_cast<double*>(y + N);
  double* e2 = diag + N;
  double* lam = e2 + N;
  int* new_idx = reinterpret_cast<int*>(lam + N);

  int* st = status + mat;
  if (threadIdx.x == 0) *st = 0;
  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (d == 0) {
    if (threadIdx.x == 0) *st = 3;
    if (eigs)
      for (int i = threadIdx.x; i < N; i += blockDim.x) eigs[mat * N + i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const double2 k = kpts[kk];
  assemble_full(c, new_idx, d, k, A, N, false);
  if (general) {
    assemble_full(c, new_idx, d, k, B, N, true);
    if (!chol_reduce_full(A, B, N, d, red)) {
      if (threadIdx.x == 0) *st = 1;
      if (eigs)
        for (int i = threadIdx.x; i < N; i += blockDim.x) eigs[mat * N + i] = __longlong_as_double(0x7ff8000000000000ll);
      return;
    }
  }
  tridiag_full(A, N, d, diag, e2, v, y, red);
  bisect_all(diag, e2, d, lam, red);
  emit_eigs_and_idos(c, g, lam, d, diff + mk * (g.npts + 1), trans + mk * g.npts, eigs ? eigs + mat * N : nullptr, N,
                     st, sharp != 0);
}

// Dense H(k), S(k) per (mask, k) into caller buffers (column-major N x N complex, leading d x d
// block valid, rest zero): assemble_bloch (tbmodel.py:277-293) on the device.
__global__ void __launch_bounds__(256) assemble_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                       const uint64_t* __restrict__ masks, double2* H, double2* S,
                                                       int* dims) {
  __shared__ int cnt[(HX_MAX_N + 31) / 32];
  extern __shared__ int new_idx[];
  const int N = c.N;
  const int64_t mat = blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  double2* h = H + mat * (int64_t)N * N;
  double2* s = S ? S + mat * (int64_t)N * N : nullptr;
  for (int64_t p = threadIdx.x; p < (int64_t)N * N; p += blockDim.x) {
    h[p] = make_double2(0.0, 0.0);
    if (s) s[p] = make_double2(0.0, 0.0);
  }
  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (threadIdx.x == 0 && kk == 0) dims[mk] = d;
  if (d == 0) return;
  const double2 k = kpts[kk];
  assemble_full(c, new_idx, d, k, h, N, false);
  if (!s) return;
  if (c.pencil == 2) {
    assemble_full(c, new_idx, d, k, s, N, true);
  } else if (c.pencil == 1) {
    // h holds T: S = I + s T, H = eps0 I + t T
    for (int64_t p = threadIdx.x; p < (int64_t)d * d; p += blockDim.x) {
      const int col = (int)(p / d), row = (int)(p - (int64_t)col * d);
      const double2 tv = h[row + (int64_t)col * N];
      const double dg = row == col ? 1.0 : 0.0;
      s[row + (int64_t)col * N] = make_double2(dg + c.s * tv.x, c.s * tv.y);
      h[row + (int64_t)col * N] = make_double2(dg * c.eps0 + c.t * tv.x, c.t * tv.y);
    }
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) s[i + (int64_t)i * N] = make_double2(1.0, 0.0);
  }
}

size_t global_ws_stride(int N, bool general) {
  size_t b = (size_t)N * N * 16 * (general ? 2 : 1) + (size_t)N * 16 * 2 + (size_t)N * 8 * 3 + (size_t)N * 4;
  return (b + 255) & ~(size_t)255;
}

// ------------------------------------------------------------------------------------------------
// curves[mk][m] = (sum_{m' <= m} diff[mk][m'] + trans[mk][m] * 2^-shift) * inv_nk / area
__global__ void finalize_kernel(const int* diff, const unsigned long long* trans, int64_t nmasks, GridDev g,
                                double inv_nk, double inv_area, double* curves) {
  const int64_t mk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (mk >= nmasks) return;
  const int lane = threadIdx.x & 31;
  const int* dr = diff + mk * (g.npts + 1);
  const unsigned long long* tr = trans + mk * g.npts;
  const double sc = ldexp(1.0, -g.shift);
  long long carry = 0;
  for (int base = 0; base < g.npts; base += 32) {
    const int m = base + lane;
    long long x = m < g.npts ? dr[m] : 0;
    // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    const long long cnt = carry + x;
    if (m < g.npts) {
      const double frac = (double)(long long)tr[m] * sc;
      curves[mk * g.npts + m] = ((double)cnt + frac) * inv_nk * inv_area;
    }
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

}  // namespace hx
