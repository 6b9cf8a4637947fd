// Stage 1 of the bipartite banded tier in REAL arithmetic and REAL storage, for real batches (periodic
// gauge at time-reversal-invariant k, hx_capi batch_is_real) with S % 4 == 0.
//
// The complex-storage path (hx_gemm.cuh with RE = true) already issues one real DMMA per fragment product,
// but the matrix still moves through HBM as double2 - the rank-32 updates and the xv products are DRAM
// bound, so half of every byte they move is a zero imaginary part.  Here the S x S block C, the
// Householder vectors V, the products X / Z and the T factors are plain doubles (leading dimension S):
//   panel_qr_real_kernel    m x 32 panel QR (column panel, or transposed row panel), reflectors real
//   xv_real_kernel<MODE>    X = (op(A) V) T, op(A) = A (MODE 0) or A^T (MODE 1), DMMA m8n8k4
//   rank_update_real_kernel M -= U W^T, DMMA m8n8k4
//   bd_band_extract_real_kernel  upper band(32) of C into the compact band of the real bulge chase
// Every range of stage 1 ends at row / column S and starts at a multiple of 32, and S % 4 == 0, so the
// 16-byte cp.async copies (two doubles) never straddle a range boundary and are always 16-byte aligned.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include "hx_bulk.cuh"
#include "hx_dense.cuh"
#include "hx_dmma.cuh"
#include "hx_gemm.cuh"
#include "hx_panel.cuh"

namespace hx {

struct RSlab {
  size_t stride;  // per-matrix slab (double units)
  int ld;         // leading dimension of the matrix and of the tall-skinny blocks
  size_t m_off;   // matrix offset inside the slab (doubles)
};

// mode 0: P[i][j] = M[r0 + i][c0 + j] (column panel);  mode 1: P[i][j] = M[r0 + j][c0 + i] (row panel,
// transposed).  Offsets in doubles.
struct RPanelArgs {
  size_t stride;
  size_t m_off;
  int ld;
  int r0, c0;
  int m;
  int mode;
  size_t v_off;
  int ldv;
  size_t t_off;
};

__device__ __forceinline__ double* rpanel_elem(double* M, const RPanelArgs& a, int i, int j) {
  return a.mode == 0 ? M + (size_t)(a.c0 + j) * a.ld + a.r0 + i : M + (size_t)(a.c0 + i) * a.ld + a.r0 + j;
}

__device__ __forceinline__ double lds_fresh_d(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

template <int RPT>
__device__ __forceinline__ double pick_row_d(const double (&x)[RPT], int r) {
  double out = 0.0;
#pragma unroll
  for (int k = 0; k < RPT; ++k)
    if (k == r) out = x[k];
  return out;
}

struct RPanelSlots {
  double sig2;
  double alpha;
  double dots[32];
};

// T[l][jt] = -tau_jt sum_{l'=l}^{jt-1} T[l][l'] w[l'] (dlarft forward/columnwise), T[jt][jt] = tau_jt.
template <int GR>
__device__ __forceinline__ void build_t_column_real(double (*Ts)[33], const double* w, const double* tauS, int jt) {
  const int tid = threadIdx.x, l = tid / GR, part = tid % GR;
  double t = 0.0;
  if (l < jt)
#pragma unroll 1
    for (int lp = l + part; lp < jt; lp += GR) t = fma(Ts[l][lp], w[lp], t);
  t = group_sum<GR>(t);
  if (jt >= 0) {
    const double tj = tauS[jt];
    if (part == 0 && l < jt) Ts[l][jt] = -tj * t;
    if (tid == 0) Ts[jt][jt] = tj;
  }
}

// Register-resident real panel QR: the layout and schedule of panel_qr_reg_kernel (hx_panel.cuh) - thread
// (c, g) owns column c, rows g + GR r (r < RPT) in registers; one CTA barrier per column; clusters of CL
// CTAs combine the norm and the 32 dot products through DSMEM in fixed rank order - on doubles.
template <int CL, int GR, int RPT>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(32 * GR)
    panel_qr_real_kernel(double* ws, RPanelArgs a, int R) {
  constexpr int BWc = 32, NT = 32 * GR, CPW = 32 / GR;
  __shared__ __align__(16) double vbuf[2][GR * RPT];
  __shared__ double wbuf[2][BWc];
  __shared__ double Ts[BWc][BWc + 1];
  __shared__ double tauS[BWc];
  __shared__ RPanelSlots slot;

  const int tid = threadIdx.x, lane = tid & 31;
  const int c = (tid >> 5) * CPW + lane / GR, g = lane % GR;
  int rank = 0;
  if constexpr (CL > 1) rank = (int)cgx::this_cluster().block_rank();
  double* base = ws + (size_t)blockIdx.y * a.stride;
  double* M = base + a.m_off;
  double* V = base + a.v_off;
  const int m = a.m;
  const int r0 = rank * R;
  const int rows = max(0, min(R, m - r0));

  for (int p = tid; p < BWc * (BWc + 1); p += NT) (&Ts[0][0])[p] = 0.0;
  double x[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int li = g + GR * r;
    x[r] = li < rows ? *rpanel_elem(M, a, r0 + li, c) : 0.0;
  }

  const int jmax = min(BWc, m);
#pragma unroll 1
  for (int j = 0; j < jmax; ++j) {
    const int buf = j & 1;
    const int jl = j - r0;
    const bool own_row = jl >= 0 && jl < rows;
    double sig2 = 0.0, alpha = 0.0;
    if ((tid >> 5) == j / CPW) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (g + GR * r >= jl) sig2 = fma(x[r], x[r], sig2);
      alpha = pick_row_d(x, jl / GR);
    }
    sig2 = group_sum<GR>(sig2);
    alpha = __shfl_sync(0xffffffffu, alpha, (lane & ~(GR - 1)) | (jl & (GR - 1)));
    if (!own_row) alpha = 0.0;
    if constexpr (CL > 1) {
      if (c == j && g == 0) {
        slot.sig2 = sig2;
        if (own_row) slot.alpha = alpha;
      }
      cgx::cluster_group cluster = cgx::this_cluster();
      cluster.sync();
      if (c == j) {
        sig2 = 0.0;
        for (int q = 0; q < CL; ++q) sig2 += cluster.map_shared_rank(&slot, q)->sig2;
        alpha = cluster.map_shared_rank(&slot, j / R)->alpha;
      }
    }
    if (c == j) {
      const QuickReflector h = quick_reflector(make_double2(alpha, 0.0), sig2);
      const double beta = h.beta.x, scale = h.scale.x;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int li = g + GR * r;
        double v;
        if (li < jl) {
          v = 0.0;
        } else if (li == jl) {
          v = 1.0;
          x[r] = h.tau == 0.0 ? x[r] : beta;
        } else {
          v = x[r] * scale;
          x[r] = v;
        }
        vbuf[buf][li] = v;
      }
      if (g == 0) tauS[j] = h.tau;
    }
    __syncthreads();
    const double tau = tauS[j];
    double s;
    {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int r = 0; r < RPT; r += 2) {
        s0 = fma(vbuf[buf][g + GR * r], x[r], s0);
        if (r + 1 < RPT) s1 = fma(vbuf[buf][g + GR * (r + 1)], x[r + 1], s1);
      }
      s = group_sum<GR>(s0 + s1);
    }
    if constexpr (CL > 1) {
      cgx::cluster_group cluster = cgx::this_cluster();
      if (g == 0) slot.dots[c] = s;
      cluster.sync();
      s = 0.0;
      for (int q = 0; q < CL; ++q) s += cluster.map_shared_rank(&slot, q)->dots[c];
    }
    if (c > j && tau != 0.0) {
      const double q = tau * s;
#pragma unroll
      for (int r = 0; r < RPT; ++r) x[r] = fma(-q, lds_fresh_d(&vbuf[buf][g + GR * r]), x[r]);
    }
    if (g == 0 && c < j) wbuf[buf][c] = s;  // V_c^T v_j
    build_t_column_real<GR>(Ts, wbuf[(j - 1) & 1], tauS, j - 1);
  }
  __syncthreads();
  build_t_column_real<GR>(Ts, wbuf[(jmax - 1) & 1], tauS, jmax - 1);
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int li = g + GR * r;
    if (li < rows) {
      const int gi = r0 + li;
      *rpanel_elem(M, a, gi, c) = gi <= c ? x[r] : 0.0;
      V[gi + (size_t)c * a.ldv] = (c >= jmax || gi < c) ? 0.0 : (gi == c ? 1.0 : x[r]);
    }
  }
  __syncthreads();
  if (rank == 0) {
    double* T = base + a.t_off;
    for (int p = tid; p < BWc * BWc; p += NT) T[(p % BWc) + (p / BWc) * BWc] = Ts[p % BWc][p / BWc];
  }
  if constexpr (CL > 1) cgx::this_cluster().sync();
}

// ------------------------------------------------------------------------------------------------
// X[rows x 32] = (op(A) V) T, op(A)[i][k] = M[ar0+i][ac0+k] (MODE 0) or M[ar0+k][ac0+i] (MODE 1).
// 64-row tiles, 4 warps x (16 x 32), K in chunks of 32 through a 3-stage cp.async pipeline.  Shared
// layouts (ld = 4 mod 16 doubles: conflict-free fragment loads):
//   MODE 0: As[k][i] (i contiguous, ld 68);  MODE 1: As[i][k] (k contiguous, ld 36);  Vs[n][k] (ld 36).
constexpr int RXV_TM = 64, RXV_TK = 32, RXV_ST = 3;
constexpr int RXV_LD0 = RXV_TM + 4, RXV_LD1 = RXV_TK + 4, RXV_LDV = RXV_TK + 4;
constexpr int RXV_A = RXV_TK * RXV_LD0 > RXV_TM * RXV_LD1 ? RXV_TK * RXV_LD0 : RXV_TM * RXV_LD1;
constexpr size_t RXV_SMEM = (size_t)RXV_ST * (RXV_A + GBW * RXV_LDV) * sizeof(double);
static_assert((size_t)(RXV_TM + GBW) * (GBW + 4) * sizeof(double) <= RXV_SMEM, "real xv epilogue tile does not fit");

// UPD (fused schedule): before a chunk of op(A) enters the product it receives the pending rank-32 update of
// the other side, op(A)[i][k] -= sum_l R[i][l] S[k][l] (R: the CTA's 64 rows, in registers as DMMA A
// fragments; S: the chunk's 32 rows, staged with the chunk), and the updated chunk is written back to M -
// one pass over the trailing matrix instead of a rank update (read + write) followed by this product (read).
//   MODE 0: M[ar0+i][ac0+k] -= R[i] . S[k];   MODE 1: M[ar0+k][ac0+i] -= S[k] . R[i]
// R[i][l] = base[r_off + i0 + i + l*ld], S[k][l] = base[s_off + k + l*ld].
constexpr int RXV_LDS = RXV_TK + 4;  // Ss[l][k]
constexpr size_t RXV_SMEM_UPD = RXV_SMEM + (size_t)RXV_ST * GBW * RXV_LDS * sizeof(double);

template <int MODE, bool UPD = false>
__global__ void __launch_bounds__(128) xv_real_kernel(double* ws, RSlab g, int ar0, int ac0, int rows, int K,
                                                      size_t v_off, size_t x_off, size_t t_off, size_t r_off = 0,
                                                      size_t s_off = 0) {
  extern __shared__ __align__(16) double rxv_sm[];
  double* As = rxv_sm;
  double* Vs = rxv_sm + RXV_ST * RXV_A;
  double* Ss = Vs + RXV_ST * GBW * RXV_LDV;  // UPD: [RXV_ST][GBW (l)][RXV_LDS (k)]
  double* base = ws + (size_t)blockIdx.y * g.stride;
  const int ld = g.ld;
  double* M = base + g.m_off;
  const double* V = base + v_off;
  double* X = base + x_off;
  const int i0 = blockIdx.x * RXV_TM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunks = (K + RXV_TK - 1) / RXV_TK;
  auto load_chunk = [&](int ch, int stg) {
    const int kk = ch * RXV_TK;
    double* A = As + stg * RXV_A;
    if (MODE == 1) {  // (i, k) at M[(ac0+i)*ld + ar0 + k]: pairs along k
#pragma unroll
      for (int q = 0; q < RXV_TM * RXV_TK / 256; ++q) {
        const int p = tid + 128 * q, kc = 2 * (p & 15), r = p >> 4;
        const int gi = i0 + r, gk = kk + kc;
        const bool ok = gi < rows && gk < K;
        cp_async16_zfill(A + r * RXV_LD1 + kc, M + (ok ? (size_t)(ac0 + gi) * ld + ar0 + gk : 0), ok);
      }
    } else {  // (i, k) at M[(ac0+k)*ld + ar0 + i]: pairs along i
#pragma unroll
      for (int q = 0; q < RXV_TM * RXV_TK / 256; ++q) {
        const int p = tid + 128 * q, r = 2 * (p & 31), kc = p >> 5;
        const int gi = i0 + r, gk = kk + kc;
        const bool ok = gi < rows && gk < K;
        cp_async16_zfill(A + kc * RXV_LD0 + r, M + (ok ? (size_t)(ac0 + gk) * ld + ar0 + gi : 0), ok);
      }
    }
    double* Vt = Vs + stg * GBW * RXV_LDV;
#pragma unroll
    for (int q = 0; q < GBW * RXV_TK / 256; ++q) {
      const int p = tid + 128 * q, kc = 2 * (p & 15), n = p >> 4;
      const int gk = kk + kc;
      const bool ok = gk < K;
      cp_async16_zfill(Vt + n * RXV_LDV + kc, V + (ok ? gk + (size_t)n * ld : 0), ok);
    }
    if (UPD) {
      double* St = Ss + stg * GBW * RXV_LDS;
      const double* Sg = base + s_off;
#pragma unroll
      for (int q = 0; q < GBW * RXV_TK / 256; ++q) {
        const int p = tid + 128 * q, kc = 2 * (p & 15), l = p >> 4;
        const int gk = kk + kc;
        const bool ok = gk < K;
        cp_async16_zfill(St + l * RXV_LDS + kc, Sg + (ok ? gk + (size_t)l * ld : 0), ok);
      }
    }
  };
  // UPD: this warp's 16 rows of R as DMMA A fragments (row 16 warp + 8 rt + lane/4, column 4 k4 + lane%4)
  double rf[2][GBW / 4];
  if (UPD) {
    const double* Rg = base + r_off;
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int k4 = 0; k4 < GBW / 4; ++k4) {
        const int r = i0 + 16 * warp + 8 * rt + (lane >> 2);
        rf[rt][k4] = r < rows ? -Rg[r + (size_t)(4 * k4 + (lane & 3)) * ld] : 0.0;
      }
  }
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int stg = 0; stg < RXV_ST - 1; ++stg) {
    if (stg < nchunks) load_chunk(stg, stg);
    cp_async_commit();
  }
  for (int ch = 0; ch < nchunks; ++ch) {
    cp_async_wait<RXV_ST - 2>();
    __syncthreads();
    {
      const int nx = ch + RXV_ST - 1;
      if (nx < nchunks) load_chunk(nx, nx % RXV_ST);
      cp_async_commit();
    }
    const int stg = ch % RXV_ST;
    double* A = As + stg * RXV_A;
    const double* Vt = Vs + stg * GBW * RXV_LDV;
    if (UPD) {
      // op(A)[rows of this warp][32 columns of the chunk] -= R S^T (K = 32), in place + back to M
      const double* St = Ss + stg * GBW * RXV_LDS;
      const int kk = ch * RXV_TK;
      double u[2][4][2];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) {
          const int r = 16 * warp + 8 * rt + (lane >> 2), c = 8 * ct + 2 * (lane & 3);
          u[rt][ct][0] = MODE == 1 ? A[r * RXV_LD1 + c] : A[c * RXV_LD0 + r];
          u[rt][ct][1] = MODE == 1 ? A[r * RXV_LD1 + c + 1] : A[(c + 1) * RXV_LD0 + r];
        }
#pragma unroll
      for (int k4 = 0; k4 < GBW / 4; ++k4) {
        const int lc = 4 * k4 + (lane & 3);
        double b[4];
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) b[ct] = St[lc * RXV_LDS + 8 * ct + (lane >> 2)];
#pragma unroll
        for (int rt = 0; rt < 2; ++rt)
#pragma unroll
          for (int ct = 0; ct < 4; ++ct) dmma(u[rt][ct][0], u[rt][ct][1], rf[rt][k4], b[ct]);
      }
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) {
          const int r = 16 * warp + 8 * rt + (lane >> 2), c = 8 * ct + 2 * (lane & 3);
          if (MODE == 1) {
            A[r * RXV_LD1 + c] = u[rt][ct][0];
            A[r * RXV_LD1 + c + 1] = u[rt][ct][1];
          } else {
            A[c * RXV_LD0 + r] = u[rt][ct][0];
            A[(c + 1) * RXV_LD0 + r] = u[rt][ct][1];
          }
          const int gi = i0 + r, gk = kk + c;
          if (gi < rows && gk < K) {  // K even, gk even: gk + 1 < K too
            if (MODE == 1) {
              *reinterpret_cast<double2*>(M + (size_t)(ac0 + gi) * ld + ar0 + gk) =
                  make_double2(u[rt][ct][0], u[rt][ct][1]);
            } else {
              M[(size_t)(ac0 + gk) * ld + ar0 + gi] = u[rt][ct][0];
              M[(size_t)(ac0 + gk + 1) * ld + ar0 + gi] = u[rt][ct][1];
            }
          }
        }
      __syncwarp();  // the product below reads only this warp's rows of the chunk
    }
#pragma unroll
    for (int k4 = 0; k4 < RXV_TK / 4; ++k4) {
      const int kc = 4 * k4 + (lane & 3);
      double a[2], b[4];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) {
        const int r = 16 * warp + 8 * rt + (lane >> 2);
        a[rt] = MODE == 1 ? A[r * RXV_LD1 + kc] : A[kc * RXV_LD0 + r];
      }
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) b[ct] = Vt[(8 * ct + (lane >> 2)) * RXV_LDV + kc];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) dmma(acc[rt][ct][0], acc[rt][ct][1], a[rt], b[ct]);
    }
  }
  // ---- epilogue: X <- (op(A) V) T on the tile in shared memory
  cp_async_wait<0>();
  __syncthreads();
  constexpr int XL = GBW + 4;
  double* Xs = rxv_sm;               // [RXV_TM][XL]
  double* Ts = rxv_sm + RXV_TM * XL;  // [n][k] = T[k][n]
  const double* T = base + t_off;
  for (int p = tid; p < GBW * GBW; p += 128) Ts[(p / GBW) * XL + (p % GBW)] = T[p];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = 16 * warp + 8 * rt + (lane >> 2), cc = 8 * ct + 2 * (lane & 3);
      Xs[r * XL + cc] = acc[rt][ct][0];
      Xs[r * XL + cc + 1] = acc[rt][ct][1];
      acc[rt][ct][0] = acc[rt][ct][1] = 0.0;
    }
  __syncthreads();
#pragma unroll
  for (int k4 = 0; k4 < GBW / 4; ++k4) {
    const int kc = 4 * k4 + (lane & 3);
    double a[2], b[4];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) a[rt] = Xs[(16 * warp + 8 * rt + (lane >> 2)) * XL + kc];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) b[ct] = Ts[(8 * ct + (lane >> 2)) * XL + kc];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) dmma(acc[rt][ct][0], acc[rt][ct][1], a[rt], b[ct]);
  }
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = i0 + 16 * warp + 8 * rt + (lane >> 2), cc = 8 * ct + 2 * (lane & 3);
      if (r < rows) {
        X[r + (size_t)cc * ld] = acc[rt][ct][0];
        X[r + (size_t)(cc + 1) * ld] = acc[rt][ct][1];
      }
    }
}

// ------------------------------------------------------------------------------------------------
// M[mr0:mr0+m, mc0:mc0+n] -= U W^T, U [m x 32], W [n x 32] (ld): RT x 64 tiles (RT = 64 or 128), 8 warps
// (4 x 2) of (RT/4) x 32, U and W staged once by cp.async as Us[k][r] / Ws[k][c] (ld = 4 mod 16 doubles),
// the C tile read straight into the DMMA accumulators.
constexpr int RRU_TN = 64;
template <int RT, bool SYM2 = false>
constexpr size_t rru_smem() {
  return (size_t)(SYM2 ? 2 : 1) * GBW * ((RT + 4) + (RRU_TN + 4)) * sizeof(double);
}

// SYM2: the symmetric rank-2k update M -= U W^T + W U^T in ONE pass over M (the Gram path's G22 -= W V^T + V W^T):
// the k index runs over 64, [U | W] against [W | U].
template <int RT, bool SYM2 = false>
__global__ void __launch_bounds__(256) rank_update_real_kernel(double* ws, RSlab g, int mr0, int mc0, int m, int n,
                                                               size_t u_off, size_t w_off, int tri = 0) {
  constexpr int LU = RT + 4, LW = RRU_TN + 4, RF = RT / 32;  // row fragments per warp
  constexpr int KK = SYM2 ? 2 * GBW : GBW;
  extern __shared__ __align__(16) double rru_sm[];
  double* Us = rru_sm;            // [KK][LU]
  double* Ws = rru_sm + KK * LU;  // [KK][LW]
  double* base = ws + (size_t)blockIdx.z * g.stride;
  const int ld = g.ld;
  double* M = base + g.m_off + (size_t)mc0 * ld + mr0;
  const double* U = base + u_off;
  const double* W = base + w_off;
  const int I0 = blockIdx.x * RT, J0 = blockIdx.y * RRU_TN;
  // SYM2 with tri (square symmetric block, mr0 == mc0, RT == RRU_TN): only the tiles on and below the diagonal are
  // computed; every element (r, c), r >= c, is stored at (r, c) AND mirrored to (c, r) - half the DMMA work of the
  // two-triangle update and an exactly symmetric matrix
  const bool mirror = SYM2 && tri;
  if (mirror && blockIdx.y > blockIdx.x) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
#pragma unroll
  for (int q = 0; q < RT * GBW / 512; ++q) {
    const int p = tid + 256 * q, r = 2 * (p % (RT / 2)), k = p / (RT / 2);
    const bool ok = I0 + r < m;
    cp_async16_zfill(Us + k * LU + r, U + (ok ? I0 + r + (size_t)k * ld : 0), ok);
    if constexpr (SYM2) cp_async16_zfill(Us + (GBW + k) * LU + r, W + (ok ? I0 + r + (size_t)k * ld : 0), ok);
  }
#pragma unroll
  for (int q = 0; q < RRU_TN * GBW / 512; ++q) {
    const int p = tid + 256 * q, r = 2 * (p & 31), k = p >> 5;
    const bool ok = J0 + r < n;
    cp_async16_zfill(Ws + k * LW + r, W + (ok ? J0 + r + (size_t)k * ld : 0), ok);
    if constexpr (SYM2) cp_async16_zfill(Ws + (GBW + k) * LW + r, U + (ok ? J0 + r + (size_t)k * ld : 0), ok);
  }
  cp_async_commit();
  double acc[RF][4][2];
#pragma unroll
  for (int rt = 0; rt < RF; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = I0 + (RT / 4) * wr + 8 * rt + (lane >> 2);
      const int cc = J0 + 32 * wc + 8 * ct + 2 * (lane & 3);
      const bool okr = r < m;
      acc[rt][ct][0] = okr && cc < n ? M[r + (size_t)cc * ld] : 0.0;
      acc[rt][ct][1] = okr && cc + 1 < n ? M[r + (size_t)(cc + 1) * ld] : 0.0;
    }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int k4 = 0; k4 < KK / 4; ++k4) {
    const int kc = 4 * k4 + (lane & 3);
    double au[RF], bw[4];
#pragma unroll
    for (int rt = 0; rt < RF; ++rt) au[rt] = -Us[kc * LU + (RT / 4) * wr + 8 * rt + (lane >> 2)];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) bw[ct] = Ws[kc * LW + 32 * wc + 8 * ct + (lane >> 2)];
#pragma unroll
    for (int rt = 0; rt < RF; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) dmma(acc[rt][ct][0], acc[rt][ct][1], au[rt], bw[ct]);
  }
#pragma unroll
  for (int rt = 0; rt < RF; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = I0 + (RT / 4) * wr + 8 * rt + (lane >> 2);
      const int cc = J0 + 32 * wc + 8 * ct + 2 * (lane & 3);
      if (mirror) {
        if (r < m && cc < n && r >= cc) {
          M[r + (size_t)cc * ld] = acc[rt][ct][0];
          if (r > cc) M[cc + (size_t)r * ld] = acc[rt][ct][0];
        }
        if (r < m && cc + 1 < n && r >= cc + 1) {
          M[r + (size_t)(cc + 1) * ld] = acc[rt][ct][1];
          if (r > cc + 1) M[cc + 1 + (size_t)r * ld] = acc[rt][ct][1];
        }
        continue;
      }
      if (r < m && cc < n) M[r + (size_t)cc * ld] = acc[rt][ct][0];
      if (r < m && cc + 1 < n) M[r + (size_t)(cc + 1) * ld] = acc[rt][ct][1];
    }
}

// ------------------------------------------------------------------------------------------------
// Persistent, double-buffered variant of rank_update_real_kernel<64> on the bulk-copy engine
// (HX_RU_BULK=1; off by default - measured 3.2x slower, see bd_reduce_real): each CTA walks the 64 x 64 tiles (all matrices of the batch) with a stride of
// gridDim.x; the C tile, the 64 x 32 U rows and the 64 x 32 W rows of the NEXT tile are in flight as bulk
// copies (one per tile column, completing on the stage's mbarrier) while the current tile runs its DMMAs, and
// the updated tile leaves through bulk stores.  The rank update is HBM-bound (C read and written once per
// update, 3.7-4.0 TB/s with the load-compute-store kernel); this keeps ~2 tiles per SM in flight.
constexpr int RBU_T = 64, RBU_LD = 68;  // tile, shared leading dimension (doubles; 2-way = minimal fragment reads)
struct RBulkStage {
  double M[RBU_T * RBU_LD];
  double U[GBW * RBU_LD];
  double W[GBW * RBU_LD];
};
constexpr size_t rru_bulk_smem() { return 2 * sizeof(RBulkStage) + 128; }

__global__ void __launch_bounds__(256, 1) rank_update_real_bulk_kernel(double* ws, RSlab g, int mr0, int mc0, int m,
                                                                        int n, size_t u_off, size_t w_off, int tiles_i,
                                                                        int tiles_j, int64_t ntiles) {
  extern __shared__ __align__(128) unsigned char rbu_raw[];
  RBulkStage* stg = reinterpret_cast<RBulkStage*>(rbu_raw);
  __shared__ __align__(8) uint64_t full[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
  const int ld = g.ld;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  const int64_t per_mat = (int64_t)tiles_i * tiles_j;
  auto tile_of = [&](int64_t t, double*& base, int& I0, int& J0) {
    const int64_t b = t / per_mat;
    const int r = (int)(t - b * per_mat);
    I0 = (r % tiles_i) * RBU_T;
    J0 = (r / tiles_i) * RBU_T;
    base = ws + (size_t)b * g.stride;
  };
  // warp 0: arm stage s and issue the bulk loads of tile t (one copy per column)
  auto issue = [&](int64_t t, int s) {
    double* base;
    int I0, J0;
    tile_of(t, base, I0, J0);
    const int rows = min(RBU_T, m - I0), cols = min(RBU_T, n - J0);
    if (lane == 0) mbar_arrive_expect_tx(&full[s], (unsigned)(8 * rows * (cols + GBW) + 8 * cols * GBW));
    __syncwarp();
    const double* Mg = base + g.m_off + (size_t)(mc0 + J0) * ld + mr0 + I0;
    for (int c = lane; c < cols; c += 32) bulk_g2s(stg[s].M + c * RBU_LD, Mg + (size_t)c * ld, 8u * rows, &full[s]);
    bulk_g2s(stg[s].U + lane * RBU_LD, base + u_off + I0 + (size_t)lane * ld, 8u * rows, &full[s]);
    bulk_g2s(stg[s].W + lane * RBU_LD, base + w_off + J0 + (size_t)lane * ld, 8u * cols, &full[s]);
  };
  const int64_t t0 = blockIdx.x, step = gridDim.x;
  if (warp == 0) {
    if (t0 < ntiles) issue(t0, 0);
    if (t0 + step < ntiles) issue(t0 + step, 1);
  }
  unsigned phase0 = 0, phase1 = 0;
  int s = 0;
  for (int64_t t = t0; t < ntiles; t += step, s ^= 1) {
    mbar_wait(&full[s], s ? phase1 : phase0);
    if (s) phase1 ^= 1u;
    else phase0 ^= 1u;
    RBulkStage& S = stg[s];
    double acc[2][4][2];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) {
        const int r = 16 * wr + 8 * rt + (lane >> 2), cc = 32 * wc + 8 * ct + 2 * (lane & 3);
        acc[rt][ct][0] = S.M[cc * RBU_LD + r];
        acc[rt][ct][1] = S.M[(cc + 1) * RBU_LD + r];
      }
#pragma unroll
    for (int k4 = 0; k4 < GBW / 4; ++k4) {
      const int kc = 4 * k4 + (lane & 3);
      double au[2], bw[4];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) au[rt] = -S.U[kc * RBU_LD + 16 * wr + 8 * rt + (lane >> 2)];
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) bw[ct] = S.W[kc * RBU_LD + 32 * wc + 8 * ct + (lane >> 2)];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) dmma(acc[rt][ct][0], acc[rt][ct][1], au[rt], bw[ct]);
    }
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) {
        const int r = 16 * wr + 8 * rt + (lane >> 2), cc = 32 * wc + 8 * ct + 2 * (lane & 3);
        S.M[cc * RBU_LD + r] = acc[rt][ct][0];
        S.M[(cc + 1) * RBU_LD + r] = acc[rt][ct][1];
      }
    fence_proxy_async_smem();
    __syncthreads();
    if (warp == 0) {
      double* base;
      int I0, J0;
      tile_of(t, base, I0, J0);
      const int rows = min(RBU_T, m - I0), cols = min(RBU_T, n - J0);
      double* Mg = base + g.m_off + (size_t)(mc0 + J0) * ld + mr0 + I0;
      for (int c = lane; c < cols; c += 32) bulk_s2g(Mg + (size_t)c * ld, S.M + c * RBU_LD, 8u * rows);
      bulk_commit();
      const int64_t tn = t + 2 * step;
      if (tn < ntiles) {
        bulk_wait_read0();  // this lane's stores have read the stage
        __syncwarp();       // ... and every other lane's
        issue(tn, s);
      }
    }
  }
  if (warp == 0) bulk_wait0();
}

// ------------------------------------------------------------------------------------------------
// The rank update on the TMA engine (HX_RU_TMA=1; off by default - measured 0.125 vs 0.091 ms per launch against
// the cp.async kernel, see bd_reduce_real; for the trailing updates that end at row and column S): a persistent CTA per SM walks the 64 x 64 tiles of every matrix of the batch; the C tile moves by
// cp.async.bulk.tensor (UTMALDG / UTMASTG) as four 16-row x 64-column boxes of a 3-D tensor map (rows, columns,
// matrix) with the 128-byte swizzle - element (r, c) of box b at 1024 b + 16 c + 2 ((r % 16) / 2 ^ c % 8) +
// r % 2 doubles, so the DMMA accumulator fragments read and write it with the minimal two wavefronts - and the
// loads of the next tile (its C boxes on the stage's mbarrier, its U / W rows by cp.async) are in flight while
// the current tile runs its DMMAs; the updated tile leaves through TMA stores.  Rows / columns past S are
// zero-filled on load and dropped on store by the tensor map.
constexpr int RTU_LD = 68;  // U / W rows: [k][row], ld 68 (conflict-free fragments)
struct __align__(1024) RTmaStage {
  double M[4 * 1024];            // 4 swizzled boxes of 16 rows x 64 columns
  double U[GBW * RTU_LD];
  double W[GBW * RTU_LD];
};
constexpr int RTMA_ST = 3;  // stages in flight per CTA (one CTA per SM)
constexpr size_t rru_tma_smem() { return RTMA_ST * sizeof(RTmaStage) + 1024; }

__device__ __forceinline__ int rtma_idx(int r, int c) {
  return (r >> 4) * 1024 + c * 16 + ((((r & 15) >> 1) ^ (c & 7)) << 1) + (r & 1);
}

__global__ void __launch_bounds__(256, 1) rank_update_real_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                       double* ws, RSlab g, int mr0, int mc0, int m,
                                                                       int n, size_t u_off, size_t w_off, int tiles_i,
                                                                       int tiles_j, int64_t ntiles) {
  extern __shared__ unsigned char rtma_raw[];
  RTmaStage* stg = reinterpret_cast<RTmaStage*>((reinterpret_cast<uintptr_t>(rtma_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[RTMA_ST];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
  const int ld = g.ld;
  if (tid == 0) {
    for (int q = 0; q < RTMA_ST; ++q) mbar_init(&full[q], 1);
    mbar_init_fence();
  }
  __syncthreads();
  const int64_t per_mat = (int64_t)tiles_i * tiles_j;
  auto coords = [&](int64_t t, int& b, int& I0, int& J0) {
    b = (int)(t / per_mat);
    const int r = (int)(t - (int64_t)b * per_mat);
    I0 = (r % tiles_i) * 64;
    J0 = (r / tiles_i) * 64;
  };
  // stage s <- tile t: C boxes by TMA (thread 0), U / W rows by cp.async (all threads, one commit group)
  auto issue = [&](int64_t t, int s) {
    if (t < ntiles) {
      int b, I0, J0;
      coords(t, b, I0, J0);
      if (tid == 0) {
        mbar_arrive_expect_tx(&full[s], 4u * 8192u);
#pragma unroll
        for (int q = 0; q < 4; ++q) tma_load_3d(stg[s].M + q * 1024, &tmap, mr0 + I0 + 16 * q, mc0 + J0, b, &full[s]);
      }
      const double* base = ws + (size_t)b * g.stride;
      const double* U = base + u_off;
      const double* W = base + w_off;
#pragma unroll
      for (int q = 0; q < 64 * GBW / 512; ++q) {
        const int p = tid + 256 * q, r = 2 * (p & 31), k = p >> 5;
        const bool oku = I0 + r < m, okw = J0 + r < n;
        cp_async16_zfill(stg[s].U + k * RTU_LD + r, U + (oku ? I0 + r + (size_t)k * ld : 0), oku);
        cp_async16_zfill(stg[s].W + k * RTU_LD + r, W + (okw ? J0 + r + (size_t)k * ld : 0), okw);
      }
    }
    cp_async_commit();
  };
  const int64_t t0 = blockIdx.x, step = gridDim.x;
#pragma unroll
  for (int q = 0; q < RTMA_ST; ++q) issue(t0 + q * step, q);
  unsigned phases = 0;  // bit q: parity of stage q's next completion
  int s = 0;
  for (int64_t t = t0; t < ntiles; t += step, s = (s + 1 == RTMA_ST ? 0 : s + 1)) {
    cp_async_wait<RTMA_ST - 1>();  // this stage's U / W (the later stages' groups may still be in flight)
    mbar_wait(&full[s], (phases >> s) & 1u);
    phases ^= 1u << s;
    __syncthreads();
    RTmaStage& S = stg[s];
    double acc[2][4][2];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) {
        const int r = 16 * wr + 8 * rt + (lane >> 2), cc = 32 * wc + 8 * ct + 2 * (lane & 3);
        acc[rt][ct][0] = S.M[rtma_idx(r, cc)];
        acc[rt][ct][1] = S.M[rtma_idx(r, cc + 1)];
      }
#pragma unroll
    for (int k4 = 0; k4 < GBW / 4; ++k4) {
      const int kc = 4 * k4 + (lane & 3);
      double au[2], bw[4];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) au[rt] = -S.U[kc * RTU_LD + 16 * wr + 8 * rt + (lane >> 2)];
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) bw[ct] = S.W[kc * RTU_LD + 32 * wc + 8 * ct + (lane >> 2)];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) dmma(acc[rt][ct][0], acc[rt][ct][1], au[rt], bw[ct]);
    }
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) {
        const int r = 16 * wr + 8 * rt + (lane >> 2), cc = 32 * wc + 8 * ct + 2 * (lane & 3);
        S.M[rtma_idx(r, cc)] = acc[rt][ct][0];
        S.M[rtma_idx(r, cc + 1)] = acc[rt][ct][1];
      }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      int b, I0, J0;
      coords(t, b, I0, J0);
#pragma unroll
      for (int q = 0; q < 4; ++q) tma_store_3d(&tmap, mr0 + I0 + 16 * q, mc0 + J0, b, S.M + q * 1024);
      bulk_commit();
      bulk_wait_read0();  // the stage's C boxes have been read out before they are refilled
    }
    __syncthreads();
    issue(t + RTMA_ST * step, s);
  }
  cp_async_wait<0>();
  if (tid == 0) bulk_wait0();
}

}  // namespace hx
