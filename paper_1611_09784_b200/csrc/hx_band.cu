// Large-N path: batched two-stage Hermitian tridiagonalisation on sm_100a.
//
// Stage 1 (dense -> band of width BW=32), per panel step k0 for every matrix of the batch:
//   panel_qr_kernel    Householder QR of the m x BW panel below the band (m = N - k0 - BW):
//                      V (explicit, unit lower trapezoidal), T (zlarft forward/columnwise), R into A.
//   xv_kernel<1>       Y = A22 V T                  (hx_gemm.cuh: DMMA f64 tensor cores, cp.async pipeline)
//   w_z/w_m/w_rows     W = Y - 1/2 V (T^H V^H Y)         (row-parallel)
//   her2k_kernel       A22 -= W V^H + V W^H          (hx_gemm.cuh; lower tiles computed, upper mirrored)
// so that A22 <- Q^H A22 Q with Q = I - V T V^H (the blocked two-sided update of zhetrd/zhe2hb).
// Stage 2 (band -> tridiagonal): bulge_chase_pipe_kernel (hx_chase.cuh), pipelined Householder bulge chasing.
// Then Sturm bisection + the reference IDOS functional (hx_dense.cuh) per matrix.
//
// Vacancies: kept dofs are compacted to the leading d x d block and the tail is exactly zero, so
// every reflector acting on it is the identity; bisection runs on the leading d x d tridiagonal.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "hx_band.cuh"
#include "hx_dense.cuh"
#include "hx_dmma.cuh"
#include "hx_gemm.cuh"
#include "hx_kernels.cuh"
#include "hx_chase.cuh"
#include "hx_panel.cuh"

namespace hx {

constexpr int BW = 32;  // band width of stage 1

static std::string g_band_err;
const char* band_last_error() { return g_band_err.c_str(); }

#define BAND_CUDA(call)                                             \
  do {                                                              \
    cudaError_t e_ = (call);                                        \
    if (e_ != cudaSuccess) {                                        \
      g_band_err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      return -1;                                                    \
    }                                                               \
  } while (0)

struct BandWs {
  // per-matrix layout inside one workspace slab (offsets in double2 units)
  size_t a_off, v_off, x_off, t_off, z_off, m_off, dg_off;  // dg: diag + e2 (2N doubles = N double2)
  size_t b_off;                              // general pencil: S (then its Cholesky factor L), N x N
  size_t stride;                             // per matrix, double2 units
  static BandWs make(int N, bool general = false) {
    BandWs w;
    w.a_off = 0;
    w.v_off = (size_t)N * N;
    w.x_off = w.v_off + (size_t)N * BW;
    w.t_off = w.x_off + (size_t)N * BW;
    w.z_off = w.t_off + (size_t)BW * BW;
    w.m_off = w.z_off + (size_t)16 * BW * BW;
    w.dg_off = w.m_off + (size_t)BW * BW;
    w.b_off = w.dg_off + (size_t)N + 16;
    w.stride = w.b_off + (general ? (size_t)N * N : 0);
    w.stride = (w.stride + 15) & ~(size_t)15;
    return w;
  }
};

__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// ------------------------------------------------------------------------------------------------
// Panel QR: one CTA per matrix.
__global__ void __launch_bounds__(256) panel_qr_kernel(double2* ws, BandWs L, int N, int k0) {
  __shared__ double red[96];
  __shared__ double2 sred[8][BW];
  __shared__ double2 s[BW];
  __shared__ double2 Ts[BW][BW + 1];
  double2* base = ws + (size_t)blockIdx.x * L.stride;
  const int lda = N;
  const int m = N - k0 - BW;
  double2* P = base + L.a_off + (size_t)k0 * lda + k0 + BW;  // P[i + c*lda], i < m, c < BW
  double2* V = base + L.v_off;                                 // V[i + c*N]
  double2* T = base + L.t_off;
  const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = bd >> 5;
  for (int p = tid; p < BW * (BW + 1); p += bd) (&Ts[0][0])[p] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int j = 0; j < BW; ++j) {
    if (j >= m) {
      for (int i = tid; i < m; i += bd) V[i + (size_t)j * N] = make_double2(0.0, 0.0);
      __syncthreads();
      continue;
    }
    double part = 0.0;
    for (int i = j + tid; i < m; i += bd) {
      const double2 x = P[i + (size_t)j * lda];
      part += x.x * x.x + x.y * x.y;
    }
    const double sig2 = block_sum(part, red);
    const double2 alpha = P[j + (size_t)j * lda];
    const Reflector h = make_reflector(alpha, sig2);
    const double tau = h.tau;
    // explicit V column j; R diagonal beta into the panel, zeros below it
    for (int i = tid; i < m; i += bd) {
      double2 vi;
      if (i < j) vi = make_double2(0.0, 0.0);
      else if (i == j) vi = make_double2(1.0, 0.0);
      else vi = tau == 0.0 ? make_double2(0.0, 0.0) : cmul(P[i + (size_t)j * lda], h.scale);
      V[i + (size_t)j * N] = vi;
    }
    // dots s_c = v^H col_c, col_c = P[:,c] (c > j) or V[:,c] (c < j); rows i >= j (own rows, no sync needed)
    double2 acc[BW];
#pragma unroll
    for (int c = 0; c < BW; ++c) acc[c] = make_double2(0.0, 0.0);
    if (tau != 0.0) {
      for (int i = tid; i < m; i += bd) {
        if (i < j) continue;
        const double2 vi = V[i + (size_t)j * N];
#pragma unroll
        for (int c = 0; c < BW; ++c) {
          if (c == j) continue;
          const double2 x = c > j ? P[i + (size_t)c * lda] : V[i + (size_t)c * N];
          acc[c].x += vi.x * x.x + vi.y * x.y;
          acc[c].y += vi.x * x.y - vi.y * x.x;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < BW; ++c) {
      acc[c].x = warp_sum(acc[c].x);
      acc[c].y = warp_sum(acc[c].y);
    }
    __syncthreads();
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < BW; ++c) sred[warp][c] = acc[c];
    }
    __syncthreads();
    if (tid < BW) {
      double2 t = make_double2(0.0, 0.0);
      for (int w = 0; w < nw; ++w) {
        t.x += sred[w][tid].x;
        t.y += sred[w][tid].y;
      }
      s[tid] = t;
    }
    if (tid == 0) {
      if (tau != 0.0) {
        const double sg = sqrt(sig2);
        const double aa = hypot(alpha.x, alpha.y);
        const double2 ph = aa > 0.0 ? make_double2(alpha.x / aa, alpha.y / aa) : make_double2(1.0, 0.0);
        P[j + (size_t)j * lda] = make_double2(-ph.x * sg, -ph.y * sg);
      }
    }
    __syncthreads();
    // zero below R's diagonal in column j; update the remaining panel columns: col_c -= tau v s_c
    if (tau != 0.0) {
      for (int i = j + 1 + tid; i < m; i += bd) P[i + (size_t)j * lda] = make_double2(0.0, 0.0);
      for (int i = j + tid; i < m; i += bd) {
        const double2 vi = V[i + (size_t)j * N];
        const double2 tv = make_double2(tau * vi.x, tau * vi.y);
        for (int c = j + 1; c < BW; ++c) {
          const double2 sc = s[c];
          double2 x = P[i + (size_t)c * lda];
          x.x -= tv.x * sc.x - tv.y * sc.y;
          x.y -= tv.x * sc.y + tv.y * sc.x;
          P[i + (size_t)c * lda] = x;
        }
      }
    }
    // T column j: T[j][j] = tau ; T[0:j, j] = -tau T[0:j,0:j] conj(s[0:j])
    if (tid < j) {
      double2 t = make_double2(0.0, 0.0);
      for (int l = tid; l < j; ++l) t = make_double2(t.x + (Ts[tid][l].x * s[l].x + Ts[tid][l].y * s[l].y),
                                                      t.y + (Ts[tid][l].y * s[l].x - Ts[tid][l].x * s[l].y));
      Ts[tid][j] = make_double2(-tau * t.x, -tau * t.y);
    }
    if (tid == 0) Ts[j][j] = make_double2(tau, 0.0);
    __syncthreads();
  }
  for (int p = tid; p < BW * BW; p += bd) {
    const int r = p % BW, c = p / BW;
    T[r + c * BW] = Ts[r][c];
  }
}

// ------------------------------------------------------------------------------------------------
// With Y = X T = A22 V T (xv_kernel's epilogue): W = Y - 1/2 V M, M = T^H (V^H Y), in three row-parallel
// steps (W overwrites Y):
//   w_z_kernel    partial Z_s = V[rows_s]^H Y[rows_s] for nsplit row ranges of every matrix
//   w_m_kernel    Z = sum_s Z_s (fixed order), M/2 = T^H Z / 2             (one small CTA per matrix)
//   w_rows_kernel W[rows] = Y[rows] - V[rows] (M/2)                        (32-row tiles)
constexpr int W_SPLIT_MAX = 16;

__global__ void __launch_bounds__(256) w_z_kernel(double2* ws, BandWs L, int N, int k0, int nsplit) {
  __shared__ double2 Vt[32][BW + 1];
  __shared__ double2 Xt[32][BW + 1];
  double2* base = ws + (size_t)blockIdx.y * L.stride;
  const int m = N - k0 - BW;
  const double2* V = base + L.v_off;
  const double2* X = base + L.x_off;
  const int per = ((m + nsplit - 1) / nsplit + 31) & ~31;
  const int ra = blockIdx.x * per, rb = min(m, ra + per);
  const int tid = threadIdx.x, oc = tid & 31, orow = tid >> 5;
  double2 z[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) z[q] = make_double2(0.0, 0.0);
  for (int r0 = ra; r0 < rb; r0 += 32) {
    __syncthreads();
    for (int p = tid; p < 32 * BW; p += 256) {
      const int rr = p & 31, c = p >> 5;
      const bool ok = r0 + rr < rb;
      Vt[rr][c] = ok ? V[r0 + rr + (size_t)c * N] : make_double2(0.0, 0.0);
      Xt[rr][c] = ok ? X[r0 + rr + (size_t)c * N] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      const double2 x = Xt[rr][oc];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = Vt[rr][orow + 8 * q];
        z[q].x += v.x * x.x + v.y * x.y;  // conj(v) * x
        z[q].y += v.x * x.y - v.y * x.x;
      }
    }
  }
  double2* zp = base + L.z_off + (size_t)blockIdx.x * BW * BW;
#pragma unroll
  for (int q = 0; q < 4; ++q) zp[(orow + 8 * q) * BW + oc] = z[q];
}

__global__ void __launch_bounds__(256) w_m_kernel(double2* ws, BandWs L, int nsplit) {
  __shared__ double2 Zs[BW][BW];
  __shared__ double2 Tsh[BW][BW];
  double2* base = ws + (size_t)blockIdx.x * L.stride;
  const double2* T = base + L.t_off;
  const double2* zp = base + L.z_off;
  const int tid = threadIdx.x, oc = tid & 31, orow = tid >> 5;
  for (int p = tid; p < BW * BW; p += 256) Tsh[p % BW][p / BW] = T[p];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = orow + 8 * q;
    double2 t = make_double2(0.0, 0.0);
    for (int s = 0; s < nsplit; ++s) {
      const double2 u = zp[(size_t)s * BW * BW + r * BW + oc];
      t = make_double2(t.x + u.x, t.y + u.y);
    }
    Zs[r][oc] = t;
  }
  __syncthreads();
  double2* mh = base + L.m_off;
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // M/2 = T^H Ms / 2
    const int r = orow + 8 * q;
    double2 t = make_double2(0.0, 0.0);
    for (int l = 0; l < BW; ++l) {
      const double2 a = cconj(Tsh[l][r]), b = Zs[l][oc];
      t.x += a.x * b.x - a.y * b.y;
      t.y += a.x * b.y + a.y * b.x;
    }
    mh[r * BW + oc] = make_double2(0.5 * t.x, 0.5 * t.y);
  }
}

__global__ void __launch_bounds__(256) w_rows_kernel(double2* ws, BandWs L, int N, int k0) {
  extern __shared__ double2 wsm[];
  double2 (*Tsh)[BW] = reinterpret_cast<double2 (*)[BW]>(wsm);
  double2 (*Mh)[BW] = reinterpret_cast<double2 (*)[BW]>(wsm + BW * BW);
  double2 (*Xt)[BW + 1] = reinterpret_cast<double2 (*)[BW + 1]>(wsm + 2 * BW * BW);
  double2 (*Vt)[BW + 1] = reinterpret_cast<double2 (*)[BW + 1]>(wsm + 2 * BW * BW + 32 * (BW + 1));
  double2* base = ws + (size_t)blockIdx.y * L.stride;
  const int m = N - k0 - BW;
  const double2* V = base + L.v_off;
  double2* X = base + L.x_off;
  const double2* T = base + L.t_off;
  const double2* mh = base + L.m_off;
  const int tid = threadIdx.x, oc = tid & 31, orow = tid >> 5;
  const int r0 = blockIdx.x * 32;
  for (int p = tid; p < BW * BW; p += 256) {
    Tsh[p % BW][p / BW] = T[p];
    Mh[p / BW][p % BW] = mh[p];
  }
  for (int p = tid; p < 32 * BW; p += 256) {
    const int rr = p & 31, c = p >> 5;
    const bool ok = r0 + rr < m;
    Vt[rr][c] = ok ? V[r0 + rr + (size_t)c * N] : make_double2(0.0, 0.0);
    Xt[rr][c] = ok ? X[r0 + rr + (size_t)c * N] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 z[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rr = orow + 8 * q;
    double2 t = Xt[rr][oc];
#pragma unroll 8
    for (int l = 0; l < BW; ++l) {
      const double2 v = Vt[rr][l], mm = Mh[l][oc];
      t.x -= v.x * mm.x - v.y * mm.y;
      t.y -= v.x * mm.y + v.y * mm.x;
    }
    z[q] = t;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rr = orow + 8 * q;
    if (r0 + rr < m) X[r0 + rr + (size_t)oc * N] = z[q];
  }
}

// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) band_assemble_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                            const uint64_t* __restrict__ masks, int64_t mat0,
                                                            double2* ws, BandWs L, int* dims, int* status) {
  __shared__ int cnt[(HX_MAX_N + 31) / 32];
  extern __shared__ int new_idx[];
  const int N = c.N;
  const int64_t mat = mat0 + blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  double2* A = ws + (size_t)blockIdx.x * L.stride + L.a_off;
  for (int64_t p = threadIdx.x; p < (int64_t)N * N; p += blockDim.x) A[p] = make_double2(0.0, 0.0);
  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (threadIdx.x == 0) {
    dims[blockIdx.x] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  if (d == 0) return;
  assemble_full(c, new_idx, d, kpts[kk], A, N, false);
}

__global__ void __launch_bounds__(256) band_copy_kernel(const double2* __restrict__ src, int64_t mat0, int N, double2* ws,
                                                        BandWs L, int* dims, int* status) {
  double2* A = ws + (size_t)blockIdx.x * L.stride + L.a_off;
  const double2* a = src + (size_t)(mat0 + blockIdx.x) * N * N;
  for (int64_t p = threadIdx.x; p < (int64_t)N * N; p += blockDim.x) A[p] = a[p];
  if (threadIdx.x == 0) {
    dims[blockIdx.x] = N;
    status[mat0 + blockIdx.x] = 0;
  }
}

// ------------------------------------------------------------------------------------------------
// General pencil (overlap tables, zhegv in the reference: spectrum.py:106-108): S = L L^H (Cholesky), then the
// standard problem L^-1 H L^-H goes through the same two-stage reduction.  Blocked with 32-wide blocks:
//   chol_panel_kernel     L11 = chol(S11) in shared memory, L21 = S21 L11^-H (one row per thread)
//   rank_update_kernel    S22 -= L21 L21^H                              (DMMA, hx_gemm.cuh)
//   trsm_rows_kernel      A[k0:k0+32, :] = L11^-1 A[k0:k0+32, :], its conjugate transpose into X (N x 32)
//   rank_update_kernel    A[k0+32:, :] -= L21 A[k0:k0+32, :]             (M -= U W^H, W = X)
// run twice with an in-place conjugate transpose between (L^-1 H, then L^-1 (L^-1 H)^H = L^-1 H L^-H).
// Vacancies: the kept d x d block is assembled in place and S's tail diagonal is 1, so L = diag(L11, I) and
// the tail of L^-1 H L^-H stays exactly zero.  A non-positive (or non-finite) Cholesky pivot marks the matrix
// HX_ST_NOT_PD (the reference's SolverError "overlap matrix not positive definite", spectrum.py:109-117) and is
// replaced by 1 so the batch runs on.
__global__ void __launch_bounds__(256) band_assemble_general_kernel(CellDev c, const double2* __restrict__ kpts,
                                                                    int nk, const uint64_t* __restrict__ masks,
                                                                    int64_t mat0, double2* ws, BandWs L, int* dims,
                                                                    int* status) {
  __shared__ int cnt[(HX_MAX_N + 31) / 32];
  extern __shared__ int new_idx[];
  const int N = c.N;
  const int64_t mat = mat0 + blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  double2* A = ws + (size_t)blockIdx.x * L.stride + L.a_off;
  double2* B = ws + (size_t)blockIdx.x * L.stride + L.b_off;
  for (int64_t p = threadIdx.x; p < (int64_t)N * N; p += blockDim.x) {
    A[p] = make_double2(0.0, 0.0);
    B[p] = make_double2(0.0, 0.0);
  }
  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (threadIdx.x == 0) {
    dims[blockIdx.x] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  for (int i = d + threadIdx.x; i < N; i += blockDim.x) B[i + (int64_t)i * N] = make_double2(1.0, 0.0);
  if (d == 0) return;
  assemble_full(c, new_idx, d, kpts[kk], A, N, false);
  assemble_full(c, new_idx, d, kpts[kk], B, N, true);
}

// One CTA per matrix: Cholesky of the 32 x 32 diagonal block at k0 (lower), then L21 = S21 L11^-H.
__global__ void __launch_bounds__(256) chol_panel_kernel(double2* ws, BandWs L, int N, int k0, int* status,
                                                         int64_t mat0) {
  __shared__ double2 Ls[BW][BW + 1];
  __shared__ int bad;
  double2* B = ws + (size_t)blockIdx.x * L.stride + L.b_off;
  const int tid = threadIdx.x;
  const int nb = min(BW, N - k0);
  if (tid == 0) bad = 0;
  for (int p = tid; p < BW * BW; p += blockDim.x) {
    const int r = p % BW, cc = p / BW;
    Ls[r][cc] = (r < nb && cc < nb && r >= cc) ? B[k0 + r + (size_t)(k0 + cc) * N] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      double pv = Ls[j][j].x;
      if (!(pv > 0.0) || !isfinite(pv)) {
        bad = 1;
        pv = 1.0;
      }
      Ls[j][j] = make_double2(sqrt(pv), 0.0);
    }
    __syncthreads();
    const double inv = 1.0 / Ls[j][j].x;
    if (tid > j && tid < nb) Ls[tid][j] = make_double2(Ls[tid][j].x * inv, Ls[tid][j].y * inv);
    __syncthreads();
    // trailing: Ls[r][cc] -= Ls[r][j] conj(Ls[cc][j]), j < cc <= r
    for (int p = tid; p < BW * BW; p += blockDim.x) {
      const int r = p % BW, cc = p / BW;
      if (cc > j && r >= cc && r < nb) {
        const double2 a = Ls[r][j], b = Ls[cc][j];
        Ls[r][cc].x -= a.x * b.x + a.y * b.y;
        Ls[r][cc].y -= a.y * b.x - a.x * b.y;
      }
    }
    __syncthreads();
  }
  if (bad && tid == 0) status[mat0 + blockIdx.x] = 1;  // HX_ST_NOT_PD
  for (int p = tid; p < BW * BW; p += blockDim.x) {
    const int r = p % BW, cc = p / BW;
    if (r < nb && cc < nb) B[k0 + r + (size_t)(k0 + cc) * N] = r >= cc ? Ls[r][cc] : make_double2(0.0, 0.0);
  }
  // rows below: x L11^H = b  ->  x_j = (b_j - sum_{l<j} x_l conj(L_jl)) / L_jj
  for (int r = k0 + nb + tid; r < N; r += blockDim.x) {
    double2 x[BW];
#pragma unroll
    for (int j = 0; j < BW; ++j) x[j] = j < nb ? B[r + (size_t)(k0 + j) * N] : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < BW; ++j) {
      if (j >= nb) break;
      double2 t = x[j];
      for (int l = 0; l < j; ++l) {
        const double2 a = x[l], b = Ls[j][l];  // x_l conj(L_jl)
        t.x -= a.x * b.x + a.y * b.y;
        t.y -= a.y * b.x - a.x * b.y;
      }
      const double inv = 1.0 / Ls[j][j].x;
      x[j] = make_double2(t.x * inv, t.y * inv);
    }
#pragma unroll
    for (int j = 0; j < BW; ++j)
      if (j < nb) B[r + (size_t)(k0 + j) * N] = x[j];
  }
}

// Rows [k0, k0+32) of A <- L11^-1 (those rows), and X[c][i] = conj(new A[k0+i][c]) (N x 32, ld N).  CTA = 32
// columns x 32 rows staged through shared memory; one thread per column runs the forward substitution.
__global__ void __launch_bounds__(256) trsm_rows_kernel(double2* ws, BandWs L, int N, int k0) {
  __shared__ double2 Ls[BW][BW + 1];
  __shared__ double2 As[BW][BW + 1];  // As[i][c]
  double2* base = ws + (size_t)blockIdx.y * L.stride;
  const double2* B = base + L.b_off;
  double2* A = base + L.a_off;
  double2* X = base + L.x_off;
  const int tid = threadIdx.x, c0 = blockIdx.x * BW;
  const int nb = min(BW, N - k0), nc = min(BW, N - c0);
  for (int p = tid; p < BW * BW; p += blockDim.x) {
    const int i = p % BW, cc = p / BW;
    Ls[i][cc] = (i < nb && cc < nb) ? B[k0 + i + (size_t)(k0 + cc) * N] : make_double2(0.0, 0.0);
    As[i][cc] = (i < nb && cc < nc) ? A[k0 + i + (size_t)(c0 + cc) * N] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (tid < nc) {
    for (int i = 0; i < nb; ++i) {
      double2 t = As[i][tid];
      for (int l = 0; l < i; ++l) {
        const double2 a = Ls[i][l], b = As[l][tid];
        t.x -= a.x * b.x - a.y * b.y;
        t.y -= a.x * b.y + a.y * b.x;
      }
      const double inv = 1.0 / Ls[i][i].x;
      As[i][tid] = make_double2(t.x * inv, t.y * inv);
    }
  }
  __syncthreads();
  for (int p = tid; p < BW * BW; p += blockDim.x) {
    const int i = p % BW, cc = p / BW;
    if (i < nb && cc < nc) A[k0 + i + (size_t)(c0 + cc) * N] = As[i][cc];
  }
  for (int p = tid; p < BW * BW; p += blockDim.x) {
    const int cc = p % BW, i = p / BW;  // X[c0 + cc][i], coalesced over cc
    if (cc < nc) X[c0 + cc + (size_t)i * N] = i < nb ? cconj(As[i][cc]) : make_double2(0.0, 0.0);
  }
}

// In-place A <- A^H (N x N): one CTA per 32 x 32 tile pair (ti <= tj).
__global__ void __launch_bounds__(256) conj_transpose_kernel(double2* ws, BandWs L, int N) {
  __shared__ double2 P[BW][BW + 1], Q[BW][BW + 1];
  double2* A = ws + (size_t)blockIdx.y * L.stride + L.a_off;
  const int nt = (N + BW - 1) / BW;
  int t = blockIdx.x, ti = 0;
  while (t >= nt - ti) {
    t -= nt - ti;
    ++ti;
  }
  const int tj = ti + t;
  const int tid = threadIdx.x;
  for (int p = tid; p < BW * BW; p += blockDim.x) {
    const int r = p % BW, cc = p / BW;
    const int gr = ti * BW + r, gc = tj * BW + cc;
    P[r][cc] = (gr < N && gc < N) ? A[gr + (size_t)gc * N] : make_double2(0.0, 0.0);
    const int hr = tj * BW + r, hc = ti * BW + cc;
    Q[r][cc] = (hr < N && hc < N) ? A[hr + (size_t)hc * N] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int p = tid; p < BW * BW; p += blockDim.x) {
    const int r = p % BW, cc = p / BW;
    const int gr = ti * BW + r, gc = tj * BW + cc;
    if (gr < N && gc < N) A[gr + (size_t)gc * N] = cconj(Q[cc][r]);
    const int hr = tj * BW + r, hc = ti * BW + cc;
    if (hr < N && hc < N) A[hr + (size_t)hc * N] = cconj(P[cc][r]);
  }
}

// A <- L^-1 A for the whole batch (the rows-then-update sweep of the file comment).
static void band_trsm_left(double2* ws, const BandWs& L, int N, int64_t cnt, cudaStream_t st) {
  const SlabGeom G{L.stride, N, L.a_off};
  for (int k0 = 0; k0 < N; k0 += BW) {
    trsm_rows_kernel<<<dim3((unsigned)((N + BW - 1) / BW), (unsigned)cnt), 256, 0, st>>>(ws, L, N, k0);
    const int m = N - k0 - BW;
    if (m > 0)
      rank_update_kernel<64><<<dim3((unsigned)((m + RU_T - 1) / RU_T), (unsigned)((N + 63) / 64), (unsigned)cnt), 256,
                               ru_smem<64>(), st>>>(ws, G, k0 + BW, 0, m, N, L.b_off + (size_t)k0 * N + k0 + BW,
                                                    L.x_off);
    count_launch(m > 0 ? 2 : 1);
  }
}

// Standard form L^-1 H L^-H of the staged pencils (status of non-PD overlaps set by chol_panel_kernel).
static int band_reduce_pencil(double2* ws, const BandWs& L, int N, int64_t cnt, int* status, int64_t mat0,
                              cudaStream_t st) {
  const SlabGeom GB{L.stride, N, L.b_off};
  for (int k0 = 0; k0 < N; k0 += BW) {
    chol_panel_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, L, N, k0, status, mat0);
    const int m = N - k0 - BW;
    if (m > 0)
      rank_update_kernel<64><<<dim3((unsigned)((m + RU_T - 1) / RU_T), (unsigned)((m + 63) / 64), (unsigned)cnt), 256,
                               ru_smem<64>(), st>>>(ws, GB, k0 + BW, k0 + BW, m, m,
                                                    L.b_off + (size_t)k0 * N + k0 + BW,
                                                    L.b_off + (size_t)k0 * N + k0 + BW);
    count_launch(m > 0 ? 2 : 1);
  }
  band_trsm_left(ws, L, N, cnt, st);
  const int nt = (N + BW - 1) / BW;
  conj_transpose_kernel<<<dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)cnt), 256, 0, st>>>(ws, L, N);
  count_launch();
  band_trsm_left(ws, L, N, cnt, st);
  BAND_CUDA(cudaGetLastError());
  return 0;
}

// ------------------------------------------------------------------------------------------------

constexpr size_t W_ROWS_SMEM = (size_t)(2 * BW * BW + 64 * (BW + 1)) * sizeof(double2);

void band_init_attributes() {
  set_smem_attr(w_rows_kernel, (int)W_ROWS_SMEM);
  cudaFuncSetAttribute(panel_qr_reg_kernel<16, 8, 32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  set_smem_attr(band_assemble_kernel, 64 * 1024);
  set_smem_attr(band_assemble_general_kernel, 64 * 1024);
  set_smem_attr(rank_update_kernel<64>, (int)ru_smem<64>());
  set_smem_attr(her2k_kernel<false>, (int)HK_SMEM);
  set_smem_attr(her2k_kernel<true>, (int)HK_SMEM);
  set_smem_attr(xv_kernel<0>, (int)XV_SMEM);
  set_smem_attr(xv_kernel<1>, (int)XV_SMEM);
#define HCHASE_ATTR(NW)                                                                           \
  set_smem_attr(bulge_chase_pipe_kernel<NW, BW, false>, chase_smem_bytes<NW, BW, false>())
  HCHASE_ATTR(1);
  HCHASE_ATTR(2);
  HCHASE_ATTR(3);
  HCHASE_ATTR(6);
  HCHASE_ATTR(11);
#undef HCHASE_ATTR
  set_smem_attr(herm_chase_r_kernel<1>, (int)herm_chase_r_smem<1>());
  set_smem_attr(herm_chase_r_kernel<2>, (int)herm_chase_r_smem<2>());
  set_smem_attr(herm_chase_r_kernel<4>, (int)herm_chase_r_smem<4>());
  set_smem_attr(herm_chase_r_kernel<8>, (int)herm_chase_r_smem<8>());
}

bool band_path_supported(int N) { return N > HX_SMEM_MAX_N && N <= HX_MAX_N; }

template <int CL, int GR, int RPT>
static void launch_panel(double2* ws, const PanelArgs& a, int64_t cnt, cudaStream_t st) {
  const int r = (a.m + CL - 1) / CL;
  panel_qr_reg_kernel<CL, GR, RPT><<<dim3((unsigned)CL, (unsigned)cnt), 32 * GR, 0, st>>>(ws, a, r);
}

// Panel QR with the panel in registers (hx_panel.cuh): the smallest configuration whose CTA (or
// cluster of 2..16 CTAs of 256 rows) holds all m rows; false if the panel is taller than 4096 rows.
// (Clusters of 128-row CTAs measured 1.5-2x slower than 256-row CTAs: two cluster barriers per column.)
bool launch_cluster_panel(double2* ws, const PanelArgs& a, int64_t cnt, cudaStream_t st) {
  const int m = a.m;
  if (m <= 32) launch_panel<1, 8, 4>(ws, a, cnt, st);
  else if (m <= 64) launch_panel<1, 8, 8>(ws, a, cnt, st);
  else if (m <= 128) launch_panel<1, 16, 8>(ws, a, cnt, st);
  else if (m <= 256) launch_panel<1, 16, 16>(ws, a, cnt, st);
  else if (m <= 512) launch_panel<2, 16, 16>(ws, a, cnt, st);
  else if (m <= 1024) launch_panel<4, 16, 16>(ws, a, cnt, st);
  else if (m <= 2048) launch_panel<8, 16, 16>(ws, a, cnt, st);
  else if (m <= 4096) launch_panel<16, 8, 32>(ws, a, cnt, st);
  else return false;
  return true;
}

// Stage 1 + 2 for `cnt` matrices already staged in the workspace.
static int band_reduce(double2* ws, const BandWs& L, int N, int64_t cnt, const int* dims, cudaStream_t st) {
  const bool herk_3m = opt("HX_HERK_3M", 0) != 0;
  for (int k0 = 0; N - k0 - BW > 0; k0 += BW) {
    const int m = N - k0 - BW;
    // register-resident panel QR; panels taller than 4096 rows use the L2-resident single-CTA kernel
    PanelArgs pa{L.stride, L.a_off, N, k0 + BW, k0, m, 0, L.v_off, N, L.t_off};
    if (!launch_cluster_panel(ws, pa, cnt, st))
      panel_qr_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, L, N, k0);
    const SlabGeom G{L.stride, N, L.a_off};
    // Y = A22 V T; op(A)[i][k] = conj(A[k0+BW+k][k0+BW+i]) = A22[i][k] (Hermitian, column-contiguous reads)
    xv_kernel<1><<<dim3((unsigned)((m + XV_TM - 1) / XV_TM), (unsigned)cnt), 128, XV_SMEM, st>>>(
        ws, G, k0 + BW, k0 + BW, m, m, L.v_off, L.x_off, L.t_off);
    const int nsplit = std::min(W_SPLIT_MAX, std::max(1, (m + 127) / 128));
    w_z_kernel<<<dim3((unsigned)nsplit, (unsigned)cnt), 256, 0, st>>>(ws, L, N, k0, nsplit);
    w_m_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, L, nsplit);
    w_rows_kernel<<<dim3((unsigned)((m + 31) / 32), (unsigned)cnt), 256, W_ROWS_SMEM, st>>>(ws, L, N, k0);
    count_launch(2);
    const unsigned tt = (unsigned)((m + RU_T - 1) / RU_T);
    if (herk_3m)
      her2k_kernel<true><<<dim3(tt * (tt + 1) / 2, (unsigned)cnt), 256, HK_SMEM, st>>>(ws, G, k0 + BW, m, L.x_off,
                                                                                        L.v_off);
    else
      her2k_kernel<false><<<dim3(tt * (tt + 1) / 2, (unsigned)cnt), 256, HK_SMEM, st>>>(ws, G, k0 + BW, m, L.x_off,
                                                                                         L.v_off);
    count_launch(4);
    BAND_CUDA(cudaGetLastError());
  }
  // warps per matrix: enough sweeps in flight to fill ~12 warps per SM across the batch (single-tile
  // variant: 19 KB of shared memory per warp)
  // at least 3 sweeps in flight per matrix: the many-matrix launches (c3 level 2: ~1900 matrices) ran one
  // warp per matrix with its sweeps fully serialised (c3 levels 2 / 3: 521 -> 446 / 1487 -> 1412 ms);
  // HX_HCHASE_MIN_NW overrides
  const int min_nw = (int)opt("HX_HCHASE_MIN_NW", 3);
  const int64_t want = std::max<int64_t>(min_nw, (148 * 12 + cnt - 1) / cnt);
  if (opt("HX_HCHASE_REG", 1) != 0) {
    // compact band (in the V / X panels' space: N x 64 double2) + register-row chase
    herm_band_extract_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, L.stride, L.a_off, L.v_off, N, dims);
    const int rnw = (int)opt("HX_HCHASE_RNW", 0);
    // warps (sweeps in flight) per matrix by the launch size: 242 registers per thread keep 8 warps per SM
    // resident, so the launch is split 8 x 1 / 4 x 2 / 2 x 4 (warps x CTAs per SM); measured on c3: 128 x N = 2816:
    // 8 warps 119 ms (shared-memory-tile kernel 177 ms); 1844 x N = 704: 8 / 4 / 2 warps 109 / 99 / 114 ms
    // (151 ms); 3072 x N = 352: 23 / 13 / 9.7 ms
    const int nw = rnw > 0 ? rnw : (cnt <= 300 ? 8 : (cnt <= 2400 ? 4 : 2));
#define HCHASE_R(NW)                                                                                       \
  herm_chase_r_kernel<NW><<<(unsigned)cnt, NW * 32, herm_chase_r_smem<NW>(), st>>>(ws, L.stride, L.v_off,   \
                                                                                   L.dg_off, N, dims)
    if (nw >= 8) HCHASE_R(8);
    else if (nw >= 4) HCHASE_R(4);
    else if (nw >= 2) HCHASE_R(2);
    else HCHASE_R(1);
#undef HCHASE_R
    count_launch(2);
    BAND_CUDA(cudaGetLastError());
    return 0;
  }
#define HCHASE(NW)                                                                                \
  bulge_chase_pipe_kernel<NW, BW, false><<<(unsigned)cnt, NW * 32, chase_smem_bytes<NW, BW, false>(), st>>>( \
      ws, L.stride, L.a_off, L.dg_off, N, dims)
  if (want >= 11) HCHASE(11);
  else if (want >= 6) HCHASE(6);
  else if (want >= 3) HCHASE(3);
  else if (want >= 2) HCHASE(2);
  else HCHASE(1);
#undef HCHASE
  count_launch(1);
  BAND_CUDA(cudaGetLastError());
  return 0;
}

HermSlab herm_slab(int n) {
  const BandWs L = BandWs::make(n);
  // scratch: the V and X panels (adjacent, n x 64 double2), free until the first panel QR
  return HermSlab{L.a_off, L.v_off, (size_t)2 * n * BW, L.dg_off, L.stride};
}

int herm_reduce(double2* ws, int n, int64_t cnt, const int* dims, cudaStream_t st) {
  NvtxRange nvtx_red("Hermitian two-stage reduce n=%d cnt=%lld", n, (long long)cnt);
  return band_reduce(ws, BandWs::make(n), n, cnt, dims, st);
}

int band_eval(const CellDev& c, const double2* kp, int nk, const uint64_t* masks, int64_t nmasks, const GridDev& g,
              int* diff, unsigned long long* trans, double* eigs, int* status, int sharp, size_t ws_budget,
              const Alloc& alloc, cudaStream_t st, RefineItem* refine, unsigned long long* refine_count) {
  const int N = c.N;
  const bool general = c.pencil == 2;  // HX_PENCIL_GENERAL
  const BandWs L = BandWs::make(N, general);
  const size_t per = L.stride * sizeof(double2) + sizeof(int) + (size_t)N * 8;
  const int64_t nmat = nmasks * nk;
  int64_t chunk = std::max<int64_t>(1, (int64_t)(ws_budget / per));
  chunk = std::min<int64_t>(chunk, nmat);
  chunk = std::min<int64_t>(chunk, 65535);
  unsigned char* buf = static_cast<unsigned char*>(alloc(per * (size_t)chunk + 256));
  if (!buf) {
    g_band_err = "workspace allocation failed";
    return -1;
  }
  double2* ws = reinterpret_cast<double2*>(buf);
  int* dims = reinterpret_cast<int*>(buf + L.stride * sizeof(double2) * chunk);
  const size_t smem = (size_t)N * sizeof(int);
  for (int64_t m0 = 0; m0 < nmat; m0 += chunk) {
    const int64_t cnt = std::min(chunk, nmat - m0);
    if (general) {
      band_assemble_general_kernel<<<(unsigned)cnt, 256, smem, st>>>(c, kp, nk, masks, m0, ws, L, dims, status);
      count_launch();
      BAND_CUDA(cudaGetLastError());
      if (band_reduce_pencil(ws, L, N, cnt, status, m0, st)) return -1;
    } else {
      band_assemble_kernel<<<(unsigned)cnt, 256, smem, st>>>(c, kp, nk, masks, m0, ws, L, dims, status);
      count_launch();
      BAND_CUDA(cudaGetLastError());
    }
    if (band_reduce(ws, L, N, cnt, dims, st)) return -1;
    launch_eig_idos(c, nk, g, m0, cnt, reinterpret_cast<const double*>(ws + L.dg_off), L.stride * 2, dims, diff,
                    trans, eigs, status, sharp, st, refine, refine_count);
    BAND_CUDA(cudaGetLastError());
  }
  return 0;
}

__global__ void __launch_bounds__(256) band_copy_b_kernel(const double2* __restrict__ src, int64_t mat0, int N,
                                                          double2* ws, BandWs L) {
  double2* B = ws + (size_t)blockIdx.x * L.stride + L.b_off;
  const double2* b = src + (size_t)(mat0 + blockIdx.x) * N * N;
  for (int64_t p = threadIdx.x; p < (int64_t)N * N; p += blockDim.x) B[p] = b[p];
}

int band_eigvalsh(int n, int64_t batch, const double2* A, const double2* Bm, double* eigs, int* status,
                  size_t ws_budget, const Alloc& alloc, cudaStream_t st) {
  const bool general = Bm != nullptr;
  const BandWs L = BandWs::make(n, general);
  const size_t per = L.stride * sizeof(double2) + sizeof(int) + (size_t)n * 8;
  int64_t chunk = std::max<int64_t>(1, (int64_t)(ws_budget / per));
  chunk = std::min<int64_t>(std::min<int64_t>(chunk, batch), 65535);
  unsigned char* buf = static_cast<unsigned char*>(alloc(per * (size_t)chunk + 256));
  if (!buf) {
    g_band_err = "workspace allocation failed";
    return -1;
  }
  double2* ws = reinterpret_cast<double2*>(buf);
  int* dims = reinterpret_cast<int*>(buf + L.stride * sizeof(double2) * chunk);
  CellDev c{};
  c.N = n;
  c.pencil = 0;
  GridDev g{};
  for (int64_t m0 = 0; m0 < batch; m0 += chunk) {
    const int64_t cnt = std::min(chunk, batch - m0);
    band_copy_kernel<<<(unsigned)cnt, 256, 0, st>>>(A, m0, n, ws, L, dims, status);
    count_launch();
    BAND_CUDA(cudaGetLastError());
    if (general) {  // S = L L^H, then the standard problem L^-1 A L^-H (zhegv, spectrum.py:106-108)
      band_copy_b_kernel<<<(unsigned)cnt, 256, 0, st>>>(Bm, m0, n, ws, L);
      count_launch();
      if (band_reduce_pencil(ws, L, n, cnt, status, m0, st)) return -1;
    }
    if (band_reduce(ws, L, n, cnt, dims, st)) return -1;
    launch_eig_idos(c, 1, g, m0, cnt, reinterpret_cast<const double*>(ws + L.dg_off), L.stride * 2, dims, nullptr,
                    nullptr, eigs, status, 0, st);
    BAND_CUDA(cudaGetLastError());
  }
  return 0;
}

}  // namespace hx
