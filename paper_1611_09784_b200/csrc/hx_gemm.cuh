// Batched complex128 GEMM kernels of stage 1 (both banded tiers), FP64 DMMA m8n8k4 on sm_100a:
//   xv_kernel<MODE>      X = (op(A) V) T  - tall-skinny product with the block reflector's T in the epilogue
//   rank_update_kernel   M -= U W^H       - the trailing update of one side
//   her2k_kernel         A -= W V^H + V W^H on lower tiles, conjugate mirror above the diagonal
// Operands live in per-matrix workspace slabs: matrix b of the batch at ws + b * stride, the matrix
// itself at m_off (column-major, leading dimension ld), tall-skinny blocks (V, X, W: rows x 32) with the
// same leading dimension.
#pragma once
#include <cuda_runtime.h>
#include <type_traits>
#include <stdint.h>

#include "hx_dmma.cuh"

namespace hx {

constexpr int GBW = 32;  // block reflector width (band width of stage 1)

struct SlabGeom {
  size_t stride;  // per-matrix slab (double2 units)
  int ld;         // leading dimension of the matrix and of the tall-skinny blocks
  size_t m_off;   // matrix offset inside the slab
};

__device__ __forceinline__ double2 gconj(double2 a) { return make_double2(a.x, -a.y); }

// ------------------------------------------------------------------------------------------------
// Asynchronous 16-byte global -> shared copy; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// X[rows x GBW] = op(A) V, op(A)[i][k] = M[ar0+i][ac0+k] (MODE 0) or conj(M[ar0+k][ac0+i]) (MODE 1),
// V [K x GBW] (ld S).  64-row tiles, 4 warps x (16 x 32), DMMA m8n8k4 f64, K in chunks of 16 through a
// 3-stage cp.async pipeline.  Shared layouts keep the fragment loads conflict-free:
//   MODE 0: As[k][i] (i contiguous, the matrix's column direction), ld 66 (= 2 mod 8 in 16 B units)
//   MODE 1: As[i][k] (k contiguous), ld 20 (= 4 mod 8); the conjugate is applied at fragment load.
constexpr int XV_TM = 64, XV_TK = 16, XV_ST = 3;
constexpr int XV_LD0 = XV_TM + 2, XV_LD1 = XV_TK + 4, XV_LDV = XV_TK + 4;
constexpr int XV_A_ELEMS = XV_TK * XV_LD0 > XV_TM * XV_LD1 ? XV_TK * XV_LD0 : XV_TM * XV_LD1;
constexpr size_t XV_SMEM = (size_t)XV_ST * (XV_A_ELEMS + GBW * XV_LDV) * sizeof(double2);
constexpr int XV_LDS = GBW + 4;  // S chunk rows (k) x 32 (l), 4 (mod 8)
constexpr size_t XV_SMEM_UPD = XV_SMEM + (size_t)XV_ST * XV_TK * XV_LDS * sizeof(double2);
static_assert((size_t)(XV_TM + GBW) * (GBW + 4) * sizeof(double2) <= XV_SMEM, "xv epilogue tile does not fit");

// UPD: before a chunk of op(A) enters the product it receives the pending rank-32 update of the other
// side, op(A) -= R S^H (R: the CTA's 64 rows, resident in registers; S: the chunk's 16 rows, staged with
// the chunk), and the updated chunk is written back to M - one pass over the trailing matrix instead of
// a separate rank update (read + write) followed by this product (read).  In matrix terms:
//   MODE 0: M[ar0+i][ac0+k] -= R[i] conj(S[k]);   MODE 1: M[ar0+k][ac0+i] -= S[k] conj(R[i]).
// R[i][l] = base[r_off + i0 + i + l*ld], S[k][l] = base[s_off + k + l*ld].
template <int MODE, bool UPD = false, bool RE = false>
__global__ void __launch_bounds__(128) xv_kernel(double2* ws, SlabGeom g, int ar0, int ac0, int rows, int K,
                                                 size_t v_off, size_t x_off, size_t t_off, size_t r_off = 0,
                                                 size_t s_off = 0) {
  extern __shared__ __align__(16) double2 xv_sm[];
  double2* As = xv_sm;                         // [XV_ST][XV_A_ELEMS]
  double2* Vs = xv_sm + XV_ST * XV_A_ELEMS;    // [XV_ST][GBW][XV_LDV]
  double2* Ss = Vs + XV_ST * GBW * XV_LDV;     // UPD: [XV_ST][XV_TK][XV_LDS]
  double2* base = ws + (size_t)blockIdx.y * g.stride;
  const int ld = g.ld;
  double2* M = base + g.m_off;
  const double2* V = base + v_off;
  double2* X = base + x_off;
  const int i0 = blockIdx.x * XV_TM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunks = (K + XV_TK - 1) / XV_TK;
  auto load_chunk = [&](int ch, int stg) {
    const int kk = ch * XV_TK;
    double2* A = As + stg * XV_A_ELEMS;
    if (MODE == 1) {
      // element (i, k) at M[(ac0+i)*ld + ar0 + k]: 16 consecutive k per row i
#pragma unroll
      for (int q = 0; q < XV_TM * XV_TK / 128; ++q) {
        const int p = tid + 128 * q, kc = p & (XV_TK - 1), r = p >> 4;
        const int gi = i0 + r, gk = kk + kc;
        const bool ok = gi < rows && gk < K;
        cp_async16_zfill(A + r * XV_LD1 + kc, M + (ok ? (size_t)(ac0 + gi) * ld + ar0 + gk : 0), ok);
      }
    } else {
      // element (i, k) at M[(ac0+k)*ld + ar0 + i]: 64 consecutive i per column k
#pragma unroll
      for (int q = 0; q < XV_TM * XV_TK / 128; ++q) {
        const int p = tid + 128 * q, r = p & (XV_TM - 1), kc = p >> 6;
        const int gi = i0 + r, gk = kk + kc;
        const bool ok = gi < rows && gk < K;
        cp_async16_zfill(A + kc * XV_LD0 + r, M + (ok ? (size_t)(ac0 + gk) * ld + ar0 + gi : 0), ok);
      }
    }
    double2* Vt = Vs + stg * GBW * XV_LDV;
#pragma unroll
    for (int q = 0; q < GBW * XV_TK / 128; ++q) {
      const int p = tid + 128 * q, kc = p & (XV_TK - 1), n = p >> 4;
      const int gk = kk + kc;
      const bool ok = gk < K;
      cp_async16_zfill(Vt + n * XV_LDV + kc, V + (ok ? gk + (size_t)n * ld : 0), ok);
    }
    if (UPD) {
      double2* St = Ss + stg * XV_TK * XV_LDS;
      const double2* Sg = base + s_off;
#pragma unroll
      for (int q = 0; q < GBW * XV_TK / 128; ++q) {
        const int p = tid + 128 * q, kc = p & (XV_TK - 1), l = p >> 4;
        const int gk = kk + kc;
        const bool ok = gk < K;
        cp_async16_zfill(St + kc * XV_LDS + l, Sg + (ok ? gk + (size_t)l * ld : 0), ok);
      }
    }
  };
  // UPD: this warp's 16 rows of R as DMMA A fragments (row 16 warp + 8 rt + lane/4, column 4 k4 + lane%4)
  double2 rf[2][GBW / 4];
  if (UPD) {
    const double2* Rg = base + r_off;
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int k4 = 0; k4 < GBW / 4; ++k4) {
        const int r = i0 + 16 * warp + 8 * rt + (lane >> 2);
        rf[rt][k4] = r < rows ? Rg[r + (size_t)(4 * k4 + (lane & 3)) * ld] : make_double2(0.0, 0.0);
      }
  }
  CTile3 acc[2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b].zero();
#pragma unroll
  for (int stg = 0; stg < XV_ST - 1; ++stg) {
    if (stg < nchunks) load_chunk(stg, stg);
    cp_async_commit();
  }
  for (int ch = 0; ch < nchunks; ++ch) {
    cp_async_wait<XV_ST - 2>();
    __syncthreads();
    {  // prefetch chunk ch + ST - 1 into the stage freed at iteration ch - 1
      const int nx = ch + XV_ST - 1;
      if (nx < nchunks) load_chunk(nx, nx % XV_ST);
      cp_async_commit();
    }
    const int stg = ch % XV_ST;
    double2* A = As + stg * XV_A_ELEMS;
    const double2* Vt = Vs + stg * GBW * XV_LDV;
    if (UPD) {
      // op(A)[rows of this warp][16 columns of the chunk] -= R S^H (K = 32), in place + back to M
      const double2* St = Ss + stg * XV_TK * XV_LDS;
      const int kk = ch * XV_TK;
      CTile3 u[2][2];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 2; ++ct) {
          const int r = 16 * warp + 8 * rt + (lane >> 2), c = 8 * ct + 2 * (lane & 3);
          const double2 z0 = MODE == 1 ? A[r * XV_LD1 + c] : A[c * XV_LD0 + r];
          const double2 z1 = MODE == 1 ? A[r * XV_LD1 + c + 1] : A[(c + 1) * XV_LD0 + r];
          // op(A) holds conj(M) in MODE 1: update the conjugates (A - R S^H)
          u[rt][ct].re0 = z0.x;
          u[rt][ct].im0 = MODE == 1 ? -z0.y : z0.y;
          u[rt][ct].re1 = z1.x;
          u[rt][ct].im1 = MODE == 1 ? -z1.y : z1.y;
          u[rt][ct].begin();
        }
#pragma unroll
      for (int k4 = 0; k4 < GBW / 4; ++k4) {
        const int lc = 4 * k4 + (lane & 3);
        double2 b[2];
#pragma unroll
        for (int ct = 0; ct < 2; ++ct) b[ct] = gconj(St[(8 * ct + (lane >> 2)) * XV_LDS + lc]);
#pragma unroll
        for (int rt = 0; rt < 2; ++rt)
#pragma unroll
          for (int ct = 0; ct < 2; ++ct) u[rt][ct].mac(-rf[rt][k4].x, -rf[rt][k4].y, b[ct].x, b[ct].y);
      }
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 2; ++ct) {
          u[rt][ct].end();
          const int r = 16 * warp + 8 * rt + (lane >> 2), c = 8 * ct + 2 * (lane & 3);
          const double2 n0 = make_double2(u[rt][ct].re0, MODE == 1 ? -u[rt][ct].im0 : u[rt][ct].im0);
          const double2 n1 = make_double2(u[rt][ct].re1, MODE == 1 ? -u[rt][ct].im1 : u[rt][ct].im1);
          if (MODE == 1) {
            A[r * XV_LD1 + c] = n0;
            A[r * XV_LD1 + c + 1] = n1;
          } else {
            A[c * XV_LD0 + r] = n0;
            A[(c + 1) * XV_LD0 + r] = n1;
          }
          const int gi = i0 + r, gk = kk + c;
          if (gi < rows) {
            if (MODE == 1) {  // M[ar0 + k][ac0 + i] = conj(op(A)) = n (the tile holds raw M values)
              double2* mp = M + (size_t)(ac0 + gi) * ld + ar0 + gk;
              if (gk < K) mp[0] = n0;
              if (gk + 1 < K) mp[1] = n1;
            } else {
              if (gk < K) M[(size_t)(ac0 + gk) * ld + ar0 + gi] = n0;
              if (gk + 1 < K) M[(size_t)(ac0 + gk + 1) * ld + ar0 + gi] = n1;
            }
          }
        }
      __syncwarp();  // the product below reads only this warp's rows of the chunk
    }
#pragma unroll
    for (int k4 = 0; k4 < XV_TK / 4; ++k4) {
      const int kc = 4 * k4 + (lane & 3);
      double2 a[2], b[4];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) {
        const int r = 16 * warp + 8 * rt + (lane >> 2);
        a[rt] = MODE == 1 ? A[r * XV_LD1 + kc] : A[kc * XV_LD0 + r];
        if (MODE == 1) a[rt].y = -a[rt].y;
      }
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) b[ct] = Vt[(8 * ct + (lane >> 2)) * XV_LDV + kc];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) cmac<RE>(acc[rt][ct], a[rt].x, a[rt].y, b[ct].x, b[ct].y);
    }
  }
  // ---- epilogue: X <- (op(A) V) T with T (GBW x GBW, column-major) - the block reflector's T factor,
  //      applied on the tile in shared memory (DMMA), saving a pass over X
  cp_async_wait<0>();
  __syncthreads();
  constexpr int XL = GBW + 4;  // 4 (mod 8): conflict-free fragments
  double2* Xs = xv_sm;        // [XV_TM][XL]   (reuses the pipeline stages)
  double2* Ts = xv_sm + XV_TM * XL;  // [GBW (n)][XL (k)] = T[k][n]
  const double2* T = base + t_off;
  for (int p = tid; p < GBW * GBW; p += 128) Ts[(p / GBW) * XL + (p % GBW)] = T[p];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = 16 * warp + 8 * rt + (lane >> 2);
      const int cc = 8 * ct + 2 * (lane & 3);
      cend<RE>(acc[rt][ct]);
      Xs[r * XL + cc] = make_double2(acc[rt][ct].re0, acc[rt][ct].im0);
      Xs[r * XL + cc + 1] = make_double2(acc[rt][ct].re1, acc[rt][ct].im1);
      acc[rt][ct].zero();
    }
  __syncthreads();
#pragma unroll
  for (int k4 = 0; k4 < GBW / 4; ++k4) {
    const int kc = 4 * k4 + (lane & 3);
    double2 a[2], b[4];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) a[rt] = Xs[(16 * warp + 8 * rt + (lane >> 2)) * XL + kc];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) b[ct] = Ts[(8 * ct + (lane >> 2)) * XL + kc];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) cmac<RE>(acc[rt][ct], a[rt].x, a[rt].y, b[ct].x, b[ct].y);
  }
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = i0 + 16 * warp + 8 * rt + (lane >> 2);
      const int cc = 8 * ct + 2 * (lane & 3);
      cend<RE>(acc[rt][ct]);
      if (r < rows) {
        X[r + (size_t)cc * ld] = make_double2(acc[rt][ct].re0, acc[rt][ct].im0);
        X[r + (size_t)(cc + 1) * ld] = make_double2(acc[rt][ct].re1, acc[rt][ct].im1);
      }
    }
}

// M[mr0:mr0+m, mc0:mc0+n] -= U W^H, U [m x GBW] and W [n x GBW] (ld S); 64 x 64 tiles, DMMA.  The whole
// K = GBW depth of U and W is staged once with cp.async (ld 36 = 4 mod 8: conflict-free fragments) while
// the C tile is read straight into the accumulators; 2 CTAs per SM.
constexpr int RU_T = 64, RU_LD = GBW + 4;
constexpr size_t RU_SMEM = (size_t)2 * RU_T * RU_LD * sizeof(double2);

// TN = 64: 8 warps (4 x 2) per 64 x 64 tile, 2 CTAs/SM; TN = 32: 4 warps per 64 x 32 tile, 4 CTAs/SM.
// M3: the 3M complex product (CTile3) at one CTA per SM (its third accumulator does not fit the 128 registers of
// two CTAs per SM); HX_RU_3M selects it.
template <int TN, bool RE = false, bool M3 = false>
__global__ void __launch_bounds__(2 * TN * 2, M3 ? 1 : (TN == 64 ? 2 : 4)) rank_update_kernel(double2* ws, SlabGeom g,
                                                                                            int mr0, int mc0, int m,
                                                                                            int n, size_t u_off,
                                                                                            size_t w_off) {
  using Tile = std::conditional_t<M3 && !RE, CTile3, CTile>;
  constexpr int NT = 4 * TN;  // threads: 4 row warps x TN/32 column warps
  extern __shared__ __align__(16) double2 ru_sm[];
  double2* Us = ru_sm;                // [RU_T][RU_LD]
  double2* Ws = ru_sm + RU_T * RU_LD;  // [TN][RU_LD]
  double2* base = ws + (size_t)blockIdx.z * g.stride;
  const int ld = g.ld;
  double2* M = base + g.m_off + (size_t)mc0 * ld + mr0;
  const double2* U = base + u_off;
  const double2* W = base + w_off;
  const int I0 = blockIdx.x * RU_T, J0 = blockIdx.y * TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
#pragma unroll
  for (int q = 0; q < RU_T * GBW / NT; ++q) {
    const int p = tid + NT * q, r = p & (RU_T - 1), k = p >> 6;
    const bool oku = I0 + r < m;
    cp_async16_zfill(Us + r * RU_LD + k, U + (oku ? I0 + r + (size_t)k * ld : 0), oku);
  }
#pragma unroll
  for (int q = 0; q < TN * GBW / NT; ++q) {
    const int p = tid + NT * q, r = p % TN, k = p / TN;
    const bool okw = J0 + r < n;
    cp_async16_zfill(Ws + r * RU_LD + k, W + (okw ? J0 + r + (size_t)k * ld : 0), okw);
  }
  cp_async_commit();
  Tile acc[2][4];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = I0 + 16 * wr + 8 * rt + (lane >> 2);
      const int cc = J0 + 32 * wc + 8 * ct + 2 * (lane & 3);
      double2 z0 = make_double2(0.0, 0.0), z1 = make_double2(0.0, 0.0);
      if (r < m && cc < n) z0 = M[r + (size_t)cc * ld];
      if (r < m && cc + 1 < n) z1 = M[r + (size_t)(cc + 1) * ld];
      acc[rt][ct].re0 = z0.x;
      acc[rt][ct].im0 = z0.y;
      acc[rt][ct].re1 = z1.x;
      acc[rt][ct].im1 = z1.y;
      cbegin<RE>(acc[rt][ct]);
    }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int k4 = 0; k4 < GBW / 4; ++k4) {
    const int kc = 4 * k4 + (lane & 3);
    double2 au[2], bw[4];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) au[rt] = Us[(16 * wr + 8 * rt + (lane >> 2)) * RU_LD + kc];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) bw[ct] = gconj(Ws[(32 * wc + 8 * ct + (lane >> 2)) * RU_LD + kc]);
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) cmac<RE>(acc[rt][ct], -au[rt].x, -au[rt].y, bw[ct].x, bw[ct].y);
  }
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = I0 + 16 * wr + 8 * rt + (lane >> 2);
      const int cc = J0 + 32 * wc + 8 * ct + 2 * (lane & 3);
      cend<RE>(acc[rt][ct]);
      if (r < m && cc < n) M[r + (size_t)cc * ld] = make_double2(acc[rt][ct].re0, acc[rt][ct].im0);
      if (r < m && cc + 1 < n) M[r + (size_t)(cc + 1) * ld] = make_double2(acc[rt][ct].re1, acc[rt][ct].im1);
    }
}
template <int TN>
constexpr size_t ru_smem() {
  return (size_t)(RU_T + TN) * RU_LD * sizeof(double2);
}


// A22 -= W V^H + V W^H on the lower 64 x 64 tiles (I >= J) of the m x m block at (r0, r0); the strictly
// upper triangle is written as the conjugate mirror, the diagonal is kept real.
// Both (W, V) pairs are staged with cp.async (K = 32 each, one pair at a time through the same buffers),
// C tile in registers, 2 CTAs per SM (a single K = 64 stage at 1 CTA per SM measured 25 % slower).
constexpr size_t HK_SMEM = RU_SMEM;
static_assert((size_t)RU_T * (RU_T + 1) * sizeof(double2) <= HK_SMEM, "her2k mirror tile does not fit");

// M3: the 3M complex product (CTile3, three DMMAs per fragment product) at 1 CTA per SM (its third
// accumulator does not fit the 128-register budget of 2 CTAs/SM); HX_HERK_3M selects it.
template <bool M3 = false>
static __global__ void __launch_bounds__(256, M3 ? 1 : 2) her2k_kernel(double2* ws, SlabGeom g, int r0, int m,
                                                                       size_t w_off, size_t v_off) {
  using Tile = std::conditional_t<M3, CTile3, CTile>;
  extern __shared__ __align__(16) double2 hk_sm[];
  double2* Ai = hk_sm;                 // [RU_T][RU_LD]  rows I0..: first factor
  double2* Bj = hk_sm + RU_T * RU_LD;  // [RU_T][RU_LD]  rows J0..: second factor (conjugated at use)
  double2* base = ws + (size_t)blockIdx.y * g.stride;
  const int ld = g.ld;
  double2* A22 = base + g.m_off + (size_t)r0 * ld + r0;
  const double2* W = base + w_off;
  const double2* V = base + v_off;
  const int t = blockIdx.x;
  int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  while (I * (I + 1) / 2 > t) --I;
  const int J = t - I * (I + 1) / 2;
  const int I0 = I * RU_T, J0 = J * RU_T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
  auto stage = [&](const double2* P, const double2* Q) {
#pragma unroll
    for (int q = 0; q < RU_T * GBW / 256; ++q) {
      const int p = tid + 256 * q, r = p & (RU_T - 1), k = p >> 6;
      const size_t col = (size_t)k * ld;
      const bool oi = I0 + r < m, oj = J0 + r < m;
      cp_async16_zfill(Ai + r * RU_LD + k, P + (oi ? I0 + r + col : 0), oi);
      cp_async16_zfill(Bj + r * RU_LD + k, Q + (oj ? J0 + r + col : 0), oj);
    }
    cp_async_commit();
  };
  stage(W, V);
  Tile acc[2][4];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = I0 + 16 * wr + 8 * rt + (lane >> 2);
      const int c = J0 + 32 * wc + 8 * ct + 2 * (lane & 3);
      double2 z0 = make_double2(0.0, 0.0), z1 = make_double2(0.0, 0.0);
      if (r < m && c < m) z0 = A22[r + (size_t)c * ld];
      if (r < m && c + 1 < m) z1 = A22[r + (size_t)(c + 1) * ld];
      acc[rt][ct].re0 = z0.x;
      acc[rt][ct].im0 = z0.y;
      acc[rt][ct].re1 = z1.x;
      acc[rt][ct].im1 = z1.y;
      acc[rt][ct].begin();
    }
  auto mac_pass = [&]() {
#pragma unroll
    for (int k4 = 0; k4 < GBW / 4; ++k4) {
      const int kc = 4 * k4 + (lane & 3);
      double2 au[2], bw[4];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) au[rt] = Ai[(16 * wr + 8 * rt + (lane >> 2)) * RU_LD + kc];
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) bw[ct] = gconj(Bj[(32 * wc + 8 * ct + (lane >> 2)) * RU_LD + kc]);
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) acc[rt][ct].mac(-au[rt].x, -au[rt].y, bw[ct].x, bw[ct].y);
    }
  };
  cp_async_wait<0>();
  __syncthreads();
  mac_pass();  // -= W V^H
  __syncthreads();
  stage(V, W);
  cp_async_wait<0>();
  __syncthreads();
  mac_pass();  // -= V W^H
  // lower part straight from the fragments; the conjugate mirror (upper triangle) through shared memory
  // so that its stores are coalesced along the columns of the mirrored tile
  __syncthreads();
  constexpr int TL = RU_T + 1;
  double2* Tt = hk_sm;  // [RU_T][TL]: tile element (r, c) at Tt[r * TL + c]
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int rl = 16 * wr + 8 * rt + (lane >> 2);
      const int cl = 32 * wc + 8 * ct + 2 * (lane & 3);
      const int r = I0 + rl, c = J0 + cl;
      acc[rt][ct].end();
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = c + e;
        double2 z = e ? make_double2(acc[rt][ct].re1, acc[rt][ct].im1) : make_double2(acc[rt][ct].re0, acc[rt][ct].im0);
        if (cc == r) z.y = 0.0;
        Tt[rl * TL + cl + e] = z;
        if (r < m && cc < m && cc <= r) A22[r + (size_t)cc * ld] = z;
      }
    }
  __syncthreads();
  // mirror: A22[J0 + c][I0 + r] = conj(tile(r, c)) for every lower element with c < r in global indices
  for (int p = tid; p < RU_T * RU_T; p += 256) {
    const int rl = p >> 6, cl = p & (RU_T - 1);  // consecutive threads: consecutive rows cl of column rl
    const int r = I0 + rl, cc = J0 + cl;
    if (r < m && cc < r) A22[cc + (size_t)r * ld] = gconj(Tt[rl * TL + cl]);
  }
}

}  // namespace hx
