// Bipartite (graphene) banded tier: singular values of the nA x nB block C of T = [[0, C], [C^H, 0]].
//
// eig(T) = +-sigma(C) plus |nA - nB| zeros (exact), and for the commuting pencil eps = (eps0 + t l)/(1 + s l).
// C is assembled into an S x S slab (S = max sublattice size, zero padded: the padding stays exactly
// zero under every reflector) and reduced in two stages:
//   stage 1 (dense -> upper band, width BW), per step k0:
//     column panel QR  C[k0:, k0:k0+BW] = Q1 R          (cluster/DSMEM panel kernel, mode 0)
//     X1 = (C_tr^H V1) T1 ; C_tr -= V1 X1^H              (left update Q1^H C_tr, DMMA; T in the epilogue)
//     row panel LQ     C[k0:k0+BW, k0+BW:] = R^H Q2^H  (QR of the conj-transposed block, mode 1)
//     Z = (C_tr2 V2) T2 ; C_tr2 -= Z V2^H                 (right update C_tr2 Q2, DMMA)
//   stage 2 (upper band -> bidiagonal) by bulge chasing (bd_chase_kernel below, one warp per sweep).
// The Golub-Kahan tridiagonal (zero diagonal, off-diagonals alpha_0, gamma_0, alpha_1, ...) truncated to
// d = nA + nB entries has exactly the eigenvalues of T; it goes through the shared bisection + IDOS kernel.
// Flops: ~4/3 S'^3 ... i.e. 4x fewer than tridiagonalising T, on a 4x smaller slab.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "hx_band.cuh"
#include "hx_bidiag.cuh"
#include "hx_dense.cuh"
#include "hx_dmma.cuh"
#include "hx_gemm.cuh"
#include "hx_kernels.cuh"
#include "hx_panel.cuh"
#include "hx_bdchase.cuh"
#include "hx_real.cuh"
#include "hx_gram.cuh"

namespace hx {

// warp-pair bulge chase (HX_CHASE_PAIR=0: one warp per task)
static bool bd_chase_pair() { return opt("HX_CHASE_PAIR", 1) != 0; }
// real bulge chase for real (periodic-gauge) batches (HX_CHASE_REAL=0: complex)
static bool bd_chase_real() { return opt("HX_CHASE_REAL", 1) != 0; }
// real storage + arithmetic in stage 1 of real batches, S % 4 == 0 (HX_REAL_STAGE1=0)
static bool bd_real_stage1() { return opt("HX_REAL_STAGE1", 1) != 0; }


constexpr int BB = 32;  // band width

static std::string g_bd_err;
const char* bd_last_error() { return g_bd_err.c_str(); }

#define BD_CUDA(call)                                                 \
  do {                                                                \
    cudaError_t e_ = (call);                                          \
    if (e_ != cudaSuccess) {                                          \
      g_bd_err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      return -1;                                                      \
    }                                                                 \
  } while (0)

struct BdWs {
  size_t c_off, v1_off, v2_off, x_off, z_off, t1_off, t2_off, band_off, tgk_off;  // double2 units
  size_t stride;
  int S;
  static BdWs make(int S) {
    BdWs w;
    w.S = S;
    w.c_off = 0;
    w.v1_off = (size_t)S * S;
    w.v2_off = w.v1_off + (size_t)S * BB;
    w.x_off = w.v2_off + (size_t)S * BB;
    w.z_off = w.x_off + (size_t)S * BB;
    w.t1_off = w.z_off + (size_t)S * BB;
    w.t2_off = w.t1_off + (size_t)BB * BB;
    w.band_off = w.t2_off + (size_t)BB * BB;  // real chase: compact band, S x RB_LD doubles
    w.tgk_off = w.band_off + (size_t)S * RB_LD / 2 + 1;  // diag[2S] + e2[2S] doubles = 2S double2
    w.stride = (w.tgk_off + (size_t)2 * S + 16 + 15) & ~(size_t)15;
    return w;
  }
};


// ------------------------------------------------------------------------------------------------
// C = A-B block of the phase matrix per (mask, k), zero padded to S x S; dims = nA + nB.
// real: the batch's k-points make the periodic-gauge matrix real (hx_capi batch_is_real): C is assembled as
// C[ia][jb] = Re(h exp(i k.(pos_a - pos_b))) (the unitary diagonal gauge change keeps the singular values;
// the dropped imaginary part is rounding), so every later stage sees exactly real data.
__global__ void __launch_bounds__(256) bd_assemble_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                          const uint64_t* __restrict__ masks, int64_t mat0,
                                                          double2* ws, BdWs L, int* dims, int* status, int real) {
  extern __shared__ int bsm[];
  int* idx_a = bsm;
  int* idx_b = idx_a + c.N;
  int* cnt = idx_b + c.N;
  const int64_t mat = mat0 + blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  double2* C = ws + (size_t)blockIdx.x * L.stride + L.c_off;
  const int2 nn = block_compact_bipartite(c, masks + mk * c.words, idx_a, idx_b, cnt);
  const int d = nn.x + nn.y;
  if (threadIdx.x == 0) {
    dims[blockIdx.x] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  // real == 2: real storage (doubles, ld S) for the real stage 1 (hx_real.cuh)
  assemble_bipartite(c, idx_a, idx_b, kpts[kk], C, L.S, L.S, L.S, false, real != 0,
                     real == 2 ? reinterpret_cast<double*>(C) : nullptr);
}

// ------------------------------------------------------------------------------------------------
// Gram-path assembly: G = C^T C of the real (periodic-gauge) block C straight from the hop tables - the sparse
// rows of C (A dof -> its kept B partners) and columns (B dof -> its kept A partners) go to scratch lists, and one
// thread per column j accumulates G[:, j] = sum_{i in col(j)} C_ij C[i, :]^T in list order (fixed: deterministic).
// Replaces bd_assemble_kernel + gram_build_kernel (dense C, then an O(S^2) scan per matrix for its nonzeros).
template <class F>
static __device__ __forceinline__ void for_each_partner(const CellDev& c, int r, F&& f) {
  for (int e = c.h_ptr[r]; e < c.h_ptr[r + 1]; ++e) {
    const int cb = c.h_col[e];
    bool dup = false;
    for (int e2 = c.h_ptr[r]; e2 < e; ++e2) dup |= (c.h_col[e2] == cb);
    if (!dup) f(cb);
  }
  for (int t = c.ht_ptr[r]; t < c.ht_ptr[r + 1]; ++t) {
    const int cb = c.h_src[c.ht_inst[t]];
    bool dup = false;
    for (int e2 = c.h_ptr[r]; e2 < c.h_ptr[r + 1]; ++e2) dup |= (c.h_col[e2] == cb);
    for (int t2 = c.ht_ptr[r]; t2 < t; ++t2) dup |= (c.h_src[c.ht_inst[t2]] == cb);
    if (!dup) f(cb);
  }
}

// Real periodic-gauge element C[a][b] (the arithmetic of assemble_bipartite's real branch).
static __device__ __forceinline__ double gram_celem(const CellDev& c, int ra, int cb, double2 k) {
  const double2 h = herm_element(c.h_ptr, c.h_col, c.h_amp, c.h_disp, ra, cb, k);
  const double2 pa = c.pos[ra], pb = c.pos[cb];
  double sn, cs;
  sincos(k.x * (pa.x - pb.x) + k.y * (pa.y - pb.y), &sn, &cs);
  return h.x * cs - h.y * sn;
}

__global__ void __launch_bounds__(256) gram_assemble_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                            const uint64_t* __restrict__ masks, int64_t mat0,
                                                            double2* ws, BdWs L, int* dims, int* status) {
  extern __shared__ int bsm[];
  int* idx_a = bsm;
  int* idx_b = idx_a + c.N;
  int* cnt = idx_b + c.N;
  __shared__ int over;
  const int64_t mat = mat0 + blockIdx.x;
  const int64_t mk = mat / nk;
  const double2 k = kpts[(int)(mat - mk * nk)];
  const int S = L.S, tid = threadIdx.x;
  double* base = reinterpret_cast<double*>(ws + (size_t)blockIdx.x * L.stride);
  double* G = base + 2 * L.c_off;
  double* colVal = base + 2 * L.v1_off;                                // [S][GRAM_K]
  double* rowVal = colVal + (size_t)S * GRAM_K;                        // [S][GRAM_K]
  int* colIdx = reinterpret_cast<int*>(rowVal + (size_t)S * GRAM_K);   // [S][GRAM_K]
  int* rowIdx = colIdx + (size_t)S * GRAM_K;                           // [S][GRAM_K]
  int* colCnt = rowIdx + (size_t)S * GRAM_K;                           // [S]
  int* rowCnt = colCnt + S;                                            // [S]
  if (tid == 0) over = 0;
  const int2 nn = block_compact_bipartite(c, masks + mk * c.words, idx_a, idx_b, cnt);
  const int d = nn.x + nn.y;
  if (tid == 0) {
    dims[blockIdx.x] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  {
    double2* G2 = reinterpret_cast<double2*>(G);
    const size_t n2 = (size_t)S * S / 2;  // S % 4 == 0
    for (size_t p = tid; p < n2; p += blockDim.x) G2[p] = make_double2(0.0, 0.0);
  }
  for (int i = tid; i < S; i += blockDim.x) {
    colCnt[i] = 0;
    rowCnt[i] = 0;
  }
  __syncthreads();
  for (int r = tid; r < c.N; r += blockDim.x) {
    const int ia = idx_a[r], jb = idx_b[r];
    if (ia >= 0) {
      int n = 0;
      for_each_partner(c, r, [&](int cb) {
        const int j = idx_b[cb];
        if (j < 0) return;
        if (n < GRAM_K) {
          rowIdx[(size_t)ia * GRAM_K + n] = j;
          rowVal[(size_t)ia * GRAM_K + n] = gram_celem(c, r, cb, k);
        } else {
          over = 1;
        }
        ++n;
      });
      rowCnt[ia] = min(n, GRAM_K);
    } else if (jb >= 0) {
      int n = 0;
      for_each_partner(c, r, [&](int ca) {
        const int i = idx_a[ca];
        if (i < 0) return;
        if (n < GRAM_K) {
          colIdx[(size_t)jb * GRAM_K + n] = i;
          colVal[(size_t)jb * GRAM_K + n] = gram_celem(c, ca, r, k);
        } else {
          over = 1;
        }
        ++n;
      });
      colCnt[jb] = min(n, GRAM_K);
    }
  }
  __syncthreads();
  for (int j = tid; j < S; j += blockDim.x) {
    double* Gj = G + (size_t)j * S;
    const int nc = colCnt[j];
    for (int a = 0; a < nc; ++a) {
      const int i = colIdx[(size_t)j * GRAM_K + a];
      const double cij = colVal[(size_t)j * GRAM_K + a];
      const int nr = rowCnt[i];
      for (int b = 0; b < nr; ++b) {
        const int kk = rowIdx[(size_t)i * GRAM_K + b];
        Gj[kk] = fma(cij, rowVal[(size_t)i * GRAM_K + b], Gj[kk]);
      }
    }
  }
  if (tid == 0 && over) status[mat] = 2;  // HX_ST_NONFINITE: surfaces as an error, never silently
}

// Complex Gram assembly (non-time-reversal-invariant k): G = C^H C (Hermitian, S x S double2, both triangles) in
// the Hermitian tier's slab, from the sparse rows and columns of the complex block C.  dims_t = nA + nB (the
// dimension of T for the counts), dims_g = nB (the leading nonzero block of G); the tridiagonal output region is
// zeroed (the chase writes its first dims_g entries only).
__global__ void __launch_bounds__(256) gram_assemble_c_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                              const uint64_t* __restrict__ masks, int64_t mat0,
                                                              double2* ws, HermSlab H, int S, int* dims_t, int* dims_g,
                                                              int* status) {
  extern __shared__ int bsm[];
  int* idx_a = bsm;
  int* idx_b = idx_a + c.N;
  int* cnt = idx_b + c.N;
  __shared__ int over;
  const int64_t mat = mat0 + blockIdx.x;
  const int64_t mk = mat / nk;
  const double2 k = kpts[(int)(mat - mk * nk)];
  const int tid = threadIdx.x;
  double2* base = ws + (size_t)blockIdx.x * H.stride;
  double2* G = base + H.a_off;
  double2* colVal = base + H.scratch_off;                             // [S][GRAM_K]
  double2* rowVal = colVal + (size_t)S * GRAM_K;                      // [S][GRAM_K]
  int* colIdx = reinterpret_cast<int*>(rowVal + (size_t)S * GRAM_K);  // [S][GRAM_K]
  int* rowIdx = colIdx + (size_t)S * GRAM_K;                          // [S][GRAM_K]
  int* colCnt = rowIdx + (size_t)S * GRAM_K;                          // [S]
  int* rowCnt = colCnt + S;                                           // [S]
  if (tid == 0) over = 0;
  const int2 nn = block_compact_bipartite(c, masks + mk * c.words, idx_a, idx_b, cnt);
  const int d = nn.x + nn.y;
  if (tid == 0) {
    dims_t[blockIdx.x] = d;
    dims_g[blockIdx.x] = nn.y;
    status[mat] = d == 0 ? 3 : 0;
  }
  const double2 zero = make_double2(0.0, 0.0);
  for (size_t p = tid; p < (size_t)S * S; p += blockDim.x) G[p] = zero;
  {
    double* dg = reinterpret_cast<double*>(base + H.dg_off);
    for (int i = tid; i < 2 * S; i += blockDim.x) dg[i] = 0.0;
  }
  for (int i = tid; i < S; i += blockDim.x) {
    colCnt[i] = 0;
    rowCnt[i] = 0;
  }
  __syncthreads();
  for (int r = tid; r < c.N; r += blockDim.x) {
    const int ia = idx_a[r], jb = idx_b[r];
    if (ia >= 0) {
      int n = 0;
      for_each_partner(c, r, [&](int cb) {
        const int j = idx_b[cb];
        if (j < 0) return;
        if (n < GRAM_K) {
          rowIdx[(size_t)ia * GRAM_K + n] = j;
          rowVal[(size_t)ia * GRAM_K + n] = herm_element(c.h_ptr, c.h_col, c.h_amp, c.h_disp, r, cb, k);
        } else {
          over = 1;
        }
        ++n;
      });
      rowCnt[ia] = min(n, GRAM_K);
    } else if (jb >= 0) {
      int n = 0;
      for_each_partner(c, r, [&](int ca) {
        const int i = idx_a[ca];
        if (i < 0) return;
        if (n < GRAM_K) {
          colIdx[(size_t)jb * GRAM_K + n] = i;
          colVal[(size_t)jb * GRAM_K + n] = herm_element(c.h_ptr, c.h_col, c.h_amp, c.h_disp, ca, r, k);
        } else {
          over = 1;
        }
        ++n;
      });
      colCnt[jb] = min(n, GRAM_K);
    }
  }
  __syncthreads();
  // G[kk][j] = sum_i conj(C_i,kk) C_ij, one thread per column j (fixed order: deterministic)
  for (int j = tid; j < S; j += blockDim.x) {
    double2* Gj = G + (size_t)j * S;
    const int nc = colCnt[j];
    for (int a = 0; a < nc; ++a) {
      const int i = colIdx[(size_t)j * GRAM_K + a];
      const double2 cij = colVal[(size_t)j * GRAM_K + a];
      const int nr = rowCnt[i];
      for (int b = 0; b < nr; ++b) {
        const int kk = rowIdx[(size_t)i * GRAM_K + b];
        const double2 cik = rowVal[(size_t)i * GRAM_K + b];
        double2 acc = Gj[kk];
        acc.x = fma(cik.x, cij.x, fma(cik.y, cij.y, acc.x));
        acc.y = fma(cik.x, cij.y, fma(-cik.y, cij.x, acc.y));
        if (kk == j) acc.y = 0.0;
        Gj[kk] = acc;
      }
    }
  }
  if (tid == 0 && over) status[mat] = 2;  // HX_ST_NONFINITE: surfaces as an error, never silently
}

// ------------------------------------------------------------------------------------------------
bool launch_cluster_panel(double2* ws, const PanelArgs& a, int64_t cnt, cudaStream_t st);

// M[mr0.., mc0..] -= U W^H (m x n, K = 32): 64 x 64 tiles at 2 CTAs/SM (HX_RU_TN=32: 64 x 32 at 4/SM, same speed)
template <bool RE = false>
static void launch_rank_update(double2* ws, const SlabGeom& G, int mr0, int mc0, int m, int n, size_t u_off,
                               size_t w_off, int64_t cnt, cudaStream_t st) {
  const int tn = opt("HX_RU_TN", 64) == 32 ? 32 : 64;
  const unsigned gx = (unsigned)((m + RU_T - 1) / RU_T);
  if (tn == 64) {
    if (!RE && opt("HX_RU_3M", 0) != 0)
      rank_update_kernel<64, false, true><<<dim3(gx, (unsigned)((n + 63) / 64), (unsigned)cnt), 256, ru_smem<64>(), st>>>(
          ws, G, mr0, mc0, m, n, u_off, w_off);
    else
      rank_update_kernel<64, RE><<<dim3(gx, (unsigned)((n + 63) / 64), (unsigned)cnt), 256, ru_smem<64>(), st>>>(
          ws, G, mr0, mc0, m, n, u_off, w_off);
  } else
    rank_update_kernel<32, RE><<<dim3(gx, (unsigned)((n + 31) / 32), (unsigned)cnt), 128, ru_smem<32>(), st>>>(
        ws, G, mr0, mc0, m, n, u_off, w_off);
}

// Stage 1.  Default: per step  L-panel -> X1 = (C_tr^H V1) T1 -> C_tr -= V1 X1^H -> R-panel ->
// Z = (C_tr2 V2) T2 -> C_tr2 -= Z V2^H.  Optional (HX_FUSED_UPDATE=1) the trailing updates are fused into the
// next product (one pass over the trailing matrix per side instead of two):
//   L-panel(k0) -> V1, T1
//   X1 = (C[k0:, k0+32:]^H V1) T1        (xv<1>; from step 2 on it first applies the pending right
//                                         update of the previous step to the chunks it streams)
//   C[k0:k0+32, k0+32:] -= V1[:32] X1^H   (the 32 rows the row panel needs)
//   R-panel(k0) -> V2, T2
//   Z = (C[k0+32:, k0+32:] V2) T2         (xv<0>, applying the pending left update V1[32:] X1^H on the fly)
//   C[k0+32:, k0+32:k0+64] -= Z V2[:32]^H (the 32 columns the next column panel needs)
// and C[k0+32:, k0+64:] -= Z V2[32:]^H stays pending for the next step's xv<1>.
// RE: the batch is real (periodic gauge, bd_assemble_kernel): the stage-1 products issue only the real DMMAs
// (the panel and chase kernels keep their complex arithmetic; on real data their results stay real).
template <bool RE>
static int bd_reduce(double2* ws, const BdWs& L, int64_t cnt, const int* dims, cudaStream_t st) {
  const int S = L.S;
  NvtxRange nvtx_red("bipartite SVD reduce S=%d cnt=%lld", S, (long long)cnt);
  const SlabGeom G{L.stride, S, L.c_off};
  // HX_FUSED_UPDATE=1: fold the trailing rank updates into the next product (one pass over the trailing
  // matrix per side).  Correct, but measured ~10% slower than separate rank updates on sm_100a (the fused
  // kernel needs ~210 registers: 2 CTAs/SM instead of 3, and the DMMA pipe idles during the update), so
  // it is off by default.
  const bool fused = opt("HX_FUSED_UPDATE", 0) == 1;
  bool pend = false;  // right update of the previous step pending on columns >= k0 + 32
  for (int k0 = 0; k0 < S; k0 += BB) {
    const int m1 = S - k0, n2 = S - k0 - BB;
    // ---- left: column panel QR, C_tr = C[k0:, k0+BB:] <- Q1^H C_tr
    PanelArgs p1{L.stride, L.c_off, S, k0, k0, m1, 0, L.v1_off, S, L.t1_off};
    if (!launch_cluster_panel(ws, p1, cnt, st)) {
      g_bd_err = "panel does not fit the cluster shared memory";
      return -1;
    }
    count_launch();
    if (n2 <= 0) break;
    const dim3 gx1((unsigned)((n2 + XV_TM - 1) / XV_TM), (unsigned)cnt);
    if (!pend)
      xv_kernel<1, false, RE><<<gx1, 128, XV_SMEM, st>>>(ws, G, k0, k0 + BB, n2, m1, L.v1_off, L.x_off, L.t1_off);
    else  // pending: C[r][c] -= Z[r - k0] conj(V2[32 + c - (k0 + 32)])
      xv_kernel<1, true><<<gx1, 128, XV_SMEM_UPD, st>>>(ws, G, k0, k0 + BB, n2, m1, L.v1_off, L.x_off, L.t1_off,
                                                         L.v2_off + BB, L.z_off);
    launch_rank_update<RE>(ws, G, k0, k0 + BB, fused ? std::min(BB, m1) : m1, n2, L.v1_off, L.x_off, cnt, st);
    count_launch(2);
    // ---- right: row panel LQ of the (updated) rows k0..k0+BB, C_tr2 = C[k0+BB:, k0+BB:] <- C_tr2 Q2
    PanelArgs p2{L.stride, L.c_off, S, k0, k0 + BB, n2, 1, L.v2_off, S, L.t2_off};
    if (!launch_cluster_panel(ws, p2, cnt, st)) {
      g_bd_err = "panel does not fit the cluster shared memory";
      return -1;
    }
    count_launch();
    const int m3 = S - k0 - BB;
    pend = false;
    if (m3 > 0 && !fused) {
      xv_kernel<0, false, RE><<<dim3((unsigned)((m3 + XV_TM - 1) / XV_TM), (unsigned)cnt), 128, XV_SMEM, st>>>(
          ws, G, k0 + BB, k0 + BB, m3, n2, L.v2_off, L.z_off, L.t2_off);
      launch_rank_update<RE>(ws, G, k0 + BB, k0 + BB, m3, n2, L.z_off, L.v2_off, cnt, st);
      count_launch(2);
    } else if (m3 > 0) {
      // Z = (C_tr2 V2) T2 with the pending left update C[r][c] -= V1[32 + r - (k0+32)] conj(X1[c - (k0+32)])
      xv_kernel<0, true><<<dim3((unsigned)((m3 + XV_TM - 1) / XV_TM), (unsigned)cnt), 128, XV_SMEM_UPD, st>>>(
          ws, G, k0 + BB, k0 + BB, m3, n2, L.v2_off, L.z_off, L.t2_off, L.v1_off + BB, L.x_off);
      launch_rank_update(ws, G, k0 + BB, k0 + BB, m3, std::min(BB, n2), L.z_off, L.v2_off, cnt, st);
      count_launch(2);
      pend = n2 > BB;
    }
    BD_CUDA(cudaGetLastError());
  }
  // ---- stage 2: enough sweeps in flight to fill the SMs (single-tile variant: 19 KB per warp).
  const int chase_mode = (int)opt("HX_CHASE_MODE", 0);
  const int64_t want = (148 * 11 + cnt - 1) / cnt;
  const size_t a1 = L.stride, a2 = L.c_off, a3 = L.tgk_off;
#define BD_CHASE(NW, DUAL, CL)                                                                          \
  {                                                                                                     \
    cudaLaunchConfig_t cfg = {};                                                                        \
    cudaLaunchAttribute attr[1];                                                                        \
    cfg.gridDim = dim3((unsigned)(cnt * CL));                                                           \
    cfg.blockDim = dim3(NW * 32);                                                                       \
    cfg.dynamicSmemBytes = bd_chase_smem<NW, BB, DUAL>();                                               \
    cfg.stream = st;                                                                                    \
    attr[0].id = cudaLaunchAttributeClusterDimension;                                                   \
    attr[0].val.clusterDim.x = CL;                                                                      \
    attr[0].val.clusterDim.y = 1;                                                                       \
    attr[0].val.clusterDim.z = 1;                                                                       \
    cfg.attrs = attr;                                                                                   \
    cfg.numAttrs = 1;                                                                                   \
    BD_CUDA(cudaLaunchKernelEx(&cfg, bd_chase_kernel<NW, BB, DUAL, CL>, ws, a1, a2, a3, S, dims)); \
  }
#define BD_CHASE_PAIR(NT)                                                                                \
  {                                                                                                     \
    bd_chase_pair_kernel<NT, BB><<<(unsigned)cnt, NT * 64, bd_chase_pair_smem<NT, BB>(), st>>>(ws, a1, a2, a3, S, \
                                                                                                 dims);  \
    BD_CUDA(cudaGetLastError());                                                                        \
  }
#define BD_CHASE_REAL(NW)                                                                                \
  {                                                                                                     \
    bd_chase_real_kernel<NW, BB><<<(unsigned)cnt, NW * 32, bd_chase_real_smem<NW, BB>(), st>>>(ws, a1, L.band_off, \
                                                                                                a3, S, dims); \
    BD_CUDA(cudaGetLastError());                                                                        \
  }
  if (RE && bd_chase_real()) {
    bd_band_extract_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, L.stride, L.c_off, L.band_off, S);
    count_launch();
    // real band: a quarter of the arithmetic and half the shared memory per sweep
    if (want >= 6) BD_CHASE_REAL(16)
    else if (want >= 2) BD_CHASE_REAL(2)
    else BD_CHASE_REAL(1)
    count_launch();
    return 0;
  }
#undef BD_CHASE_REAL
  const bool pair = chase_mode >= 4 || (chase_mode == 0 && bd_chase_pair());
  // warp-pair tasks for every launch size: the pair kernel's task arithmetic (two half sums per reduction)
  // differs in rounding from the one-warp kernel's, so one family for all batch sizes keeps a mask's curve
  // bitwise independent of the batch it is solved in (the one-warp kernel was 3 % faster on the latency-bound
  // one-CTA-per-matrix launch: 24.3 vs 25.1 ms; HX_CHASE_PAIR=0 selects it everywhere)
  if (pair) {
    if (want >= 6) BD_CHASE_PAIR(10)
    else if (want >= 2) BD_CHASE_PAIR(2)
    else BD_CHASE_PAIR(1)
  } else if (want >= 6) {
    // one CTA (11 sweeps in flight) per matrix: in the concurrent tier schedule the 2-CTA cluster variant
    // (16 sweeps, 3-6 % lower latency alone) costs more than it gains by occupying twice the SMs
    if (chase_mode == 2) BD_CHASE(8, false, 2)
    else if (chase_mode == 3) BD_CHASE(6, true, 1)
    else BD_CHASE(11, false, 1)
  } else if (want >= 2) {
    BD_CHASE(2, false, 1)
  } else {
    BD_CHASE(1, false, 1)
  }
#undef BD_CHASE_PAIR
#undef BD_CHASE
  count_launch();
  BD_CUDA(cudaGetLastError());
  return 0;
}

// ------------------------------------------------------------------------------------------------
// Real stage 1 (hx_real.cuh): the slab holds C as an S x S double matrix (ld S) at 2 * c_off, V1/V2/X/Z as
// S x 32 doubles and T1/T2 as 32 x 32 doubles at twice their double2 offsets.
static __global__ void __launch_bounds__(256) bd_band_extract_real_kernel(double* ws, size_t stride, size_t c_off,
                                                                           size_t band_off, int S) {
  double* base = ws + (size_t)blockIdx.x * stride;
  const double* C = base + c_off;
  double* B = base + band_off;
  const size_t n = (size_t)S * RB_LD;
  for (size_t p = threadIdx.x; p < n; p += blockDim.x) {
    const int c = (int)(p / RB_LD), r = c + (int)(p % RB_LD) - RB_OFF;
    B[p] = (r >= 0 && r < S) ? C[r + (size_t)c * S] : 0.0;
  }
}

template <int CL, int GR, int RPT>
static void launch_real_panel(double* ws, const RPanelArgs& a, int64_t cnt, cudaStream_t st) {
  const int r = (a.m + CL - 1) / CL;
  panel_qr_real_kernel<CL, GR, RPT><<<dim3((unsigned)CL, (unsigned)cnt), 32 * GR, 0, st>>>(ws, a, r);
}

// Smallest configuration whose CTA (or cluster of CTAs of up to 512 rows) holds the m panel rows: real
// rows take half the registers of complex ones, so a CTA holds twice as many (half the cluster barriers).
static bool launch_real_cluster_panel(double* ws, const RPanelArgs& a, int64_t cnt, cudaStream_t st) {
  const int m = a.m;
  if (m <= 32) launch_real_panel<1, 8, 4>(ws, a, cnt, st);
  else if (m <= 64) launch_real_panel<1, 8, 8>(ws, a, cnt, st);
  else if (m <= 128) launch_real_panel<1, 16, 8>(ws, a, cnt, st);
  else if (m <= 256) launch_real_panel<1, 16, 16>(ws, a, cnt, st);
  else if (m <= 512) launch_real_panel<1, 16, 32>(ws, a, cnt, st);
  else if (m <= 1024) launch_real_panel<2, 16, 32>(ws, a, cnt, st);
  else if (m <= 2048) launch_real_panel<4, 16, 32>(ws, a, cnt, st);
  else if (m <= 4096) launch_real_panel<8, 16, 32>(ws, a, cnt, st);
  else return false;
  return true;
}

// 3-D tensor map (rows, columns, matrix) of the batch's S x S real matrices for the TMA rank update: boxes of
// 16 rows x 64 columns, 128-byte swizzle.  cuTensorMapEncodeTiled comes from the driver through the runtime's
// entry-point query (no libcuda link dependency).
static bool make_matrix_tmap(CUtensorMap* map, double* base, int S, size_t ld, size_t slab_stride, int64_t cnt) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)S, (cuuint64_t)S, (cuuint64_t)cnt};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)slab_stride * 8};
  const cuuint32_t box[3] = {16, 64, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static void launch_rank_update_real_tma(const CUtensorMap& map, double* ws, const RSlab& G, int mr0, int mc0, int m,
                                        int n, size_t u_off, size_t w_off, int64_t cnt, cudaStream_t st) {
  const int ti = (m + 63) / 64, tj = (n + 63) / 64;
  const int64_t ntiles = cnt * ti * tj;
  if (ntiles <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, 148);
  rank_update_real_tma_kernel<<<grid, 256, rru_tma_smem(), st>>>(map, ws, G, mr0, mc0, m, n, u_off, w_off, ti, tj,
                                                                  ntiles);
}

// bulk-copy persistent rank update (HX_RU_BULK=0: the load-compute-store kernel); one CTA per SM
static void launch_rank_update_real_bulk(double* ws, const RSlab& G, int mr0, int mc0, int m, int n, size_t u_off,
                                         size_t w_off, int64_t cnt, cudaStream_t st) {
  const int ti = (m + RBU_T - 1) / RBU_T, tj = (n + RBU_T - 1) / RBU_T;
  const int64_t ntiles = cnt * ti * tj;
  if (ntiles <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, 148);
  rank_update_real_bulk_kernel<<<grid, 256, rru_bulk_smem(), st>>>(ws, G, mr0, mc0, m, n, u_off, w_off, ti, tj, ntiles);
}

template <int RT>
static void launch_rank_update_real(double* ws, const RSlab& G, int mr0, int mc0, int m, int n, size_t u_off,
                                    size_t w_off, int64_t cnt, cudaStream_t st) {
  rank_update_real_kernel<RT><<<dim3((unsigned)((m + RT - 1) / RT), (unsigned)((n + RRU_TN - 1) / RRU_TN), (unsigned)cnt),
                                256, rru_smem<RT>(), st>>>(ws, G, mr0, mc0, m, n, u_off, w_off);
}

static int bd_reduce_real(double2* ws2, const BdWs& L, int64_t cnt, const int* dims, cudaStream_t st) {
  const int S = L.S;
  NvtxRange nvtx_red("bipartite SVD reduce (real) S=%d cnt=%lld", S, (long long)cnt);
  double* ws = reinterpret_cast<double*>(ws2);
  const size_t sd = 2 * L.stride, c0 = 2 * L.c_off, v1 = 2 * L.v1_off, v2 = 2 * L.v2_off, x = 2 * L.x_off,
               z = 2 * L.z_off, t1 = 2 * L.t1_off, t2 = 2 * L.t2_off;
  const RSlab G{sd, S, c0};
  const int ru_rt = opt("HX_RRU_RT", 64) == 128 ? 128 : 64;
  // HX_RU_BULK=1: the persistent bulk-copy rank update (hx_real.cuh) - correct, but measured 3.2x slower
  // (0.292 vs 0.090 ms per launch on the N = 2048 tier): one cp.async.bulk per 512-byte tile column is bound by
  // the copy engine's per-request cost, not by HBM; kept as an option, off by default
  const bool ru_bulk = opt("HX_RU_BULK", 0) != 0;
  // HX_RU_TMA=1: the TMA rank update (tensor-map boxes, 128-byte swizzle, 3 stages in flight) for the trailing
  // updates that run to row and column S.  Correct, but measured slower than the cp.async kernel on the N = 2048
  // tier (0.125 vs 0.091 ms per launch, 2.6 vs 3.7 TB/s: the C tile's extra round trip through shared memory and
  // one CTA per SM), so it is off by default
  CUtensorMap cmap;
  const bool ru_tma = opt("HX_RU_TMA", 0) != 0 && make_matrix_tmap(&cmap, ws + c0, S, (size_t)S, sd, cnt);
  auto rank_update = [&](int mr0, int mc0, int m, int n, size_t u, size_t w) {
    if (ru_tma && mr0 + m == S && mc0 + n == S) launch_rank_update_real_tma(cmap, ws, G, mr0, mc0, m, n, u, w, cnt, st);
    else if (ru_bulk) launch_rank_update_real_bulk(ws, G, mr0, mc0, m, n, u, w, cnt, st);
    else if (ru_rt == 128) launch_rank_update_real<128>(ws, G, mr0, mc0, m, n, u, w, cnt, st);
    else launch_rank_update_real<64>(ws, G, mr0, mc0, m, n, u, w, cnt, st);
  };
  // Fused schedule (HX_REAL_FUSED=1 forces it on, =0 off; default on for S >= 2048): the trailing rank update
  // of each side is applied by the next product while it streams the matrix (xv_real_kernel<MODE, true>),
  // two passes over the trailing matrix fewer per step.  The DRAM-bound updates dominate a lone large tier
  // (c4, S = 4096); in the concurrent c2 schedule it measured even (64.4 vs 63.9 ms), so smaller S keep the
  // separate updates.
  const int fused_env = (int)opt("HX_REAL_FUSED", -1);
  const bool fused = fused_env >= 0 ? fused_env != 0 : S >= 2048;
  bool pend = false;  // right update of the previous step pending on columns >= k0 + 32
  for (int k0 = 0; k0 < S; k0 += BB) {
    const int m1 = S - k0, n2 = S - k0 - BB;
    // ---- left: column panel QR, C_tr = C[k0:, k0+BB:] <- Q1^T C_tr
    const RPanelArgs p1{sd, c0, S, k0, k0, m1, 0, v1, S, t1};
    if (!launch_real_cluster_panel(ws, p1, cnt, st)) {
      g_bd_err = "panel does not fit the cluster shared memory";
      return -1;
    }
    count_launch();
    if (n2 <= 0) break;
    const dim3 gx1((unsigned)((n2 + RXV_TM - 1) / RXV_TM), (unsigned)cnt);
    if (!pend)
      xv_real_kernel<1><<<gx1, 128, RXV_SMEM, st>>>(ws, G, k0, k0 + BB, n2, m1, v1, x, t1);
    else  // pending: C[r][c] -= Z[r - k0] . V2[32 + c - (k0 + 32)]
      xv_real_kernel<1, true><<<gx1, 128, RXV_SMEM_UPD, st>>>(ws, G, k0, k0 + BB, n2, m1, v1, x, t1, v2 + BB, z);
    rank_update(k0, k0 + BB, fused ? std::min(BB, m1) : m1, n2, v1, x);
    count_launch(2);
    // ---- right: row panel LQ of rows k0..k0+BB, C_tr2 = C[k0+BB:, k0+BB:] <- C_tr2 Q2
    const RPanelArgs p2{sd, c0, S, k0, k0 + BB, n2, 1, v2, S, t2};
    if (!launch_real_cluster_panel(ws, p2, cnt, st)) {
      g_bd_err = "panel does not fit the cluster shared memory";
      return -1;
    }
    count_launch();
    const int m3 = S - k0 - BB;
    pend = false;
    const dim3 gx3((unsigned)((m3 + RXV_TM - 1) / RXV_TM), (unsigned)cnt);
    if (m3 > 0 && !fused) {
      xv_real_kernel<0><<<gx3, 128, RXV_SMEM, st>>>(ws, G, k0 + BB, k0 + BB, m3, n2, v2, z, t2);
      rank_update(k0 + BB, k0 + BB, m3, n2, z, v2);
      count_launch(2);
    } else if (m3 > 0) {
      // Z = (C_tr2 V2) T2 with the pending left update C[r][c] -= V1[32 + r - (k0+32)] . X1[c - (k0+32)]
      xv_real_kernel<0, true><<<gx3, 128, RXV_SMEM_UPD, st>>>(ws, G, k0 + BB, k0 + BB, m3, n2, v2, z, t2,
                                                              v1 + BB, x);
      rank_update(k0 + BB, k0 + BB, m3, std::min(BB, n2), z, v2);
      count_launch(2);
      pend = n2 > BB;
    }
    BD_CUDA(cudaGetLastError());
  }
  bd_band_extract_real_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, sd, c0, 2 * L.band_off, S);
  count_launch();
  const int64_t want = (148 * 11 + cnt - 1) / cnt;
  const size_t a1 = L.stride, a3 = L.tgk_off;
  // Many-matrix launches (2 <= want < 6, e.g. the 1024 N = 512 matrices of a c2 level): 4 sweeps per matrix
  // and at most 5 CTAs per SM (padded dynamic shared memory), which bounds the bands in flight (~740 x
  // 196 KB) - measured 3-4 % faster per pass than 2 sweeps at full occupancy (the launch is L2-capacity
  // bound: 17.7 GB DRAM traffic for 200 MB of bands).  HX_CHASE_RNW / HX_CHASE_CAP override (0 = off).
  const int rnw = (int)opt("HX_CHASE_RNW", -1);
  const int cap = (int)opt("HX_CHASE_CAP", 5);
  // cluster size of the few-matrix launches: HX_CHASE_RCL overrides; default 1 (one CTA per matrix)
  const int rcl_env = (int)opt("HX_CHASE_RCL", -1);
  int rcl = rcl_env >= 0 ? rcl_env : (S >= 2048 ? 8 : 1);  // c4 (S = 4096, 32 matrices): 14.5 -> 17.1 samples/s
  rcl = rcl >= 8 ? 8 : rcl >= 4 ? 4 : rcl >= 2 ? 2 : 1;
  while (rcl > 1 && (cnt * rcl > 148 || rcl * 16 > S / BB)) rcl /= 2;  // co-resident; <= one slot per task
  auto smem_of = [&](size_t need) {
    return cap > 0 && want < 6 && want >= 2 ? std::max(need, (size_t)(220 * 1024) / cap) : need;
  };
  // register-row chase for the many-matrix launches (HX_CHASE_REG=1 forces it everywhere, =0 off): measured
  // 7.19 -> 6.69 ms on the 1024-matrix N = 512 launch; the one-CTA-per-matrix launches (16 warps) keep the
  // shared-memory-tile kernel, whose 93 registers leave room on their SMs for the concurrent tiers' blocks
  // (the 128-register variant fills the register file: c2 step 63.7 -> 64.7 ms)
  const int reg_opt = (int)opt("HX_CHASE_REG", -1);
  const bool regrow = reg_opt >= 0 ? reg_opt != 0 : (want < 6 || (rcl <= 1 && opt("HX_CHASE_BIGNW", 8) <= 8));
#define BD_CHASE_REAL(NW)                                                                                  \
  do {                                                                                                     \
    if (regrow)                                                                                            \
      bd_chase_realr_kernel<NW><<<(unsigned)cnt, NW * 32, smem_of(bd_chase_realr_smem<NW>()), st>>>(       \
          ws2, a1, L.band_off, a3, S, dims);                                                               \
    else                                                                                                   \
      bd_chase_real_kernel<NW, BB><<<(unsigned)cnt, NW * 32, smem_of(bd_chase_real_smem<NW, BB>()), st>>>( \
          ws2, a1, L.band_off, a3, S, dims);                                                               \
  } while (0)
  // HX_CHASE_RNW forces the warps per matrix for every batch size (tests run each variant on a few matrices)
  if (rnw == 1) BD_CHASE_REAL(1);
  else if (rnw == 2) BD_CHASE_REAL(2);
  else if (rnw == 4) BD_CHASE_REAL(4);
  else if (rnw == 8) BD_CHASE_REAL(8);
  else if (rnw == 16) BD_CHASE_REAL(16);
  else if (want >= 6 && rcl > 1) {
    // few matrices with long sweeps: CL CTAs (SMs) per matrix, CL x 16 sweeps in flight
#define BD_CHASE_REAL_CL(CLN)                                                                                 \
  do {                                                                                                        \
    if (regrow)                                                                                               \
      bd_chase_realr_kernel<16, CLN><<<(unsigned)(cnt * CLN), 16 * 32, bd_chase_realr_smem<16>(), st>>>(      \
          ws2, a1, L.band_off, a3, S, dims);                                                                  \
    else                                                                                                      \
      bd_chase_real_kernel<16, BB, CLN><<<(unsigned)(cnt * CLN), 16 * 32, bd_chase_real_smem<16, BB>(), st>>>( \
          ws2, a1, L.band_off, a3, S, dims);                                                                  \
  } while (0)
    // HX_CHASE_CLNW=8: 8 warps per CTA in the pairs of CTAs (the same 16 sweeps in flight per matrix as one
    // 16-warp CTA, spread over two SMs: half the warps competing for each SM's issue slots)
    if (rcl == 2 && opt("HX_CHASE_CLNW", 16) == 8) {
      if (regrow)
        bd_chase_realr_kernel<8, 2><<<(unsigned)(cnt * 2), 8 * 32, bd_chase_realr_smem<8>(), st>>>(
            ws2, a1, L.band_off, a3, S, dims);
      else
        bd_chase_real_kernel<8, BB, 2><<<(unsigned)(cnt * 2), 8 * 32, bd_chase_real_smem<8, BB>(), st>>>(
            ws2, a1, L.band_off, a3, S, dims);
    } else if (rcl == 2) BD_CHASE_REAL_CL(2);
    else if (rcl == 4) BD_CHASE_REAL_CL(4);
    else BD_CHASE_REAL_CL(8);
#undef BD_CHASE_REAL_CL
  } else if (want >= 6) {
    // few matrices, one CTA each: 8 warps of the register-row chase (N = 2048 tier of c2: 10.0 ms against
    // 12.9 ms for 16 warps of the shared-memory-tile chase - fewer warps competing for the SM's issue slots and
    // L1 pipe shorten every task; c2 step 63.1 -> 62.0 ms).  HX_CHASE_BIGNW = 6 / 12 / 16 and HX_CHASE_REG
    // select the others.
    const int bnw = (int)opt("HX_CHASE_BIGNW", 8);
    if (bnw == 6) BD_CHASE_REAL(6);
    else if (bnw == 12) BD_CHASE_REAL(12);
    else if (bnw == 16) BD_CHASE_REAL(16);
    else BD_CHASE_REAL(8);
  }
  else if (want >= 2) BD_CHASE_REAL(4);
  else BD_CHASE_REAL(1);
#undef BD_CHASE_REAL
  count_launch();
  BD_CUDA(cudaGetLastError());
  return 0;
}

// Gram path (hx_gram.cuh): G = C^T C of the real batch formed in the slab, symmetric two-stage reduction to its
// tridiagonal (diag[S], e2[S] doubles at the TGK offset).
static int bd_reduce_gram(double2* ws2, const BdWs& L, int64_t cnt, const int* dims, int* status, bool direct,
                          cudaStream_t st) {
  const int S = L.S;
  NvtxRange nvtx_red("gram reduce S=%d cnt=%lld: stage 1 (panel, xv, W, rank-2k) + symmetric chase", S, (long long)cnt);
  double* ws = reinterpret_cast<double*>(ws2);
  const size_t sd = 2 * L.stride, c0 = 2 * L.c_off, v1 = 2 * L.v1_off, x = 2 * L.x_off, t1 = 2 * L.t1_off;
  const RSlab G{sd, S, c0};
  if (!direct) {
    gram_build_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, sd, c0, v1, S, status);
    count_launch();
  }
  const bool wsplit = opt("HX_GRAM_WSPLIT", 1) != 0, sym2 = opt("HX_GRAM_SYM2", 1) != 0;
  const int tri = opt("HX_GRAM_TRI", 1) != 0;  // lower tiles only + mirror (hx_real.cuh)
  const size_t pz = 2 * L.z_off;  // partial V^T Y blocks (z is unused by the Gram path)
  for (int k0 = 0; S - k0 - BB > 0; k0 += BB) {
    const int m = S - k0 - BB;
    const RPanelArgs p{sd, c0, S, k0 + BB, k0, m, 0, v1, S, t1};
    if (!launch_real_cluster_panel(ws, p, cnt, st)) {
      g_bd_err = "panel does not fit the cluster shared memory";
      return -1;
    }
    xv_real_kernel<0><<<dim3((unsigned)((m + RXV_TM - 1) / RXV_TM), (unsigned)cnt), 128, RXV_SMEM, st>>>(
        ws, G, k0 + BB, k0 + BB, m, m, v1, x, t1);
    if (wsplit) {
      const int nch = (m + GRAM_WR - 1) / GRAM_WR;
      gram_vty_kernel<<<dim3((unsigned)nch, (unsigned)cnt), 256, 0, st>>>(ws, G, m, v1, x, pz);
      gram_wfix_kernel<<<dim3((unsigned)nch, (unsigned)cnt), 256, 0, st>>>(ws, G, m, nch, v1, x, t1, pz);
      count_launch();
    } else {
      w_fix_real_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, G, m, v1, x, t1);
    }
    if (sym2) {  // G22 -= W V^T + V W^T in one pass
      rank_update_real_kernel<64, true>
          <<<dim3((unsigned)((m + 63) / 64), (unsigned)((m + RRU_TN - 1) / RRU_TN), (unsigned)cnt), 256,
             rru_smem<64, true>(), st>>>(ws, G, k0 + BB, k0 + BB, m, m, x, v1, tri);
      count_launch(4);
    } else {
      launch_rank_update_real<64>(ws, G, k0 + BB, k0 + BB, m, m, x, v1, cnt, st);  // G22 -= W V^T
      launch_rank_update_real<64>(ws, G, k0 + BB, k0 + BB, m, m, v1, x, cnt, st);  // G22 -= V W^T
      count_launch(5);
    }
    BD_CUDA(cudaGetLastError());
  }
  const int64_t want = (148 * 11 + cnt - 1) / cnt;
  if (opt("HX_GRAM_CHASE", 1) == 0) {
    // dense-slab symmetric chase (shared-memory tiles): the first version, kept for comparison
#define SYM_CHASE(NW)                                                                                      \
  sym_chase_real_kernel<NW><<<(unsigned)cnt, NW * 32, sym_chase_real_smem<NW>(), st>>>(ws, sd, c0,          \
                                                                                      2 * L.tgk_off, S)
    if (want >= 6) SYM_CHASE(16);
    else if (want >= 2) SYM_CHASE(4);
    else SYM_CHASE(1);
#undef SYM_CHASE
    count_launch();
    BD_CUDA(cudaGetLastError());
    return 0;
  }
  // compact lower band (64 doubles per column) + register-row chase; launch shapes as the bidiagonal chase
  NvtxRange nvtx_chase("gram symmetric chase S=%d cnt=%lld", S, (long long)cnt);
  const size_t bo = 2 * L.band_off, to = 2 * L.tgk_off;
  sym_band_extract_kernel<<<(unsigned)cnt, 256, 0, st>>>(ws, sd, c0, bo, S);
  // no shared-memory padding (occupancy cap) here: 4 CTAs / SM by registers, and the smaller carve-out leaves more
  // L1 (c2 step 40.4 -> 39.8 ms); HX_SYM_CAP = n pads to n CTAs / SM
  const int cap = (int)opt("HX_SYM_CAP", 0);
  const int rnw = (int)opt("HX_CHASE_RNW", -1);
  const int rcl_env = (int)opt("HX_CHASE_RCL", -1);
  int rcl = rcl_env >= 0 ? rcl_env : (S >= 2048 ? 8 : 1);
  rcl = rcl >= 8 ? 8 : rcl >= 4 ? 4 : rcl >= 2 ? 2 : 1;
  while (rcl > 1 && (cnt * rcl > 148 || rcl * 16 > S / BB)) rcl /= 2;
  auto smem_of = [&](size_t need) {
    return cap > 0 && want < 6 && want >= 2 ? std::max(need, (size_t)(220 * 1024) / cap) : need;
  };
#define SYM_CHASE_R(NW)                                                                                          \
  sym_chase_realr_kernel<NW><<<(unsigned)cnt, NW * 32, smem_of(sym_chase_realr_smem<NW>()), st>>>(ws, sd, bo, to, \
                                                                                                  S, dims)
#define SYM_CHASE_CL(CLN)                                                                                       \
  sym_chase_realr_kernel<16, CLN><<<(unsigned)(cnt * CLN), 16 * 32, sym_chase_realr_smem<16>(), st>>>(ws, sd, bo, \
                                                                                                      to, S, dims)
  if (rnw == 1) SYM_CHASE_R(1);
  else if (rnw == 2) SYM_CHASE_R(2);
  else if (rnw == 4) SYM_CHASE_R(4);
  else if (rnw == 8) SYM_CHASE_R(8);
  else if (rnw == 16) SYM_CHASE_R(16);
  else if (want >= 6 && rcl == 2) SYM_CHASE_CL(2);
  else if (want >= 6 && rcl == 4) SYM_CHASE_CL(4);
  else if (want >= 6 && rcl == 8) SYM_CHASE_CL(8);
  else if (want >= 6 && opt("HX_SYM_BIGNW", 8) == 16) SYM_CHASE_R(16);
  else if (want >= 6) SYM_CHASE_R(8);
  else if (want >= 2 && opt("HX_SYM_SMALLNW", 4) == 2) SYM_CHASE_R(2);
  else if (want >= 2 && opt("HX_SYM_SMALLNW", 4) == 8) SYM_CHASE_R(8);
  else if (want >= 2) SYM_CHASE_R(4);
  else SYM_CHASE_R(1);
#undef SYM_CHASE_R
#undef SYM_CHASE_CL
  count_launch(2);
  BD_CUDA(cudaGetLastError());
  return 0;
}

void bd_init_attributes() {
  set_smem_attr(sym_chase_real_kernel<16>, (int)sym_chase_real_smem<16>());
  set_smem_attr(sym_chase_real_kernel<4>, (int)sym_chase_real_smem<4>());
  set_smem_attr(sym_chase_real_kernel<1>, (int)sym_chase_real_smem<1>());
  set_smem_attr(sym_chase_realr_kernel<1>, 220 * 1024);
  set_smem_attr(sym_chase_realr_kernel<2>, 220 * 1024);
  set_smem_attr(sym_chase_realr_kernel<4>, 220 * 1024);
  set_smem_attr(sym_chase_realr_kernel<8>, 220 * 1024);
  set_smem_attr(sym_chase_realr_kernel<16>, 220 * 1024);
  set_smem_attr(sym_chase_realr_kernel<16, 2>, (int)sym_chase_realr_smem<16>());
  set_smem_attr(sym_chase_realr_kernel<16, 4>, (int)sym_chase_realr_smem<16>());
  set_smem_attr(sym_chase_realr_kernel<16, 8>, (int)sym_chase_realr_smem<16>());
  set_smem_attr(xv_real_kernel<0>, (int)RXV_SMEM);
  set_smem_attr(xv_real_kernel<1>, (int)RXV_SMEM);
  set_smem_attr(xv_real_kernel<0, true>, (int)RXV_SMEM_UPD);
  set_smem_attr(xv_real_kernel<1, true>, (int)RXV_SMEM_UPD);
  set_smem_attr(rank_update_real_kernel<64>, (int)rru_smem<64>());
  set_smem_attr(rank_update_real_kernel<128>, (int)rru_smem<128>());
  set_smem_attr(rank_update_real_bulk_kernel, (int)rru_bulk_smem());
  set_smem_attr(rank_update_real_tma_kernel, (int)rru_tma_smem());
  set_smem_attr(xv_kernel<0>, (int)XV_SMEM);
  set_smem_attr(xv_kernel<1>, (int)XV_SMEM);
  set_smem_attr(xv_kernel<0, true>, XV_SMEM_UPD);
  set_smem_attr(xv_kernel<1, true>, XV_SMEM_UPD);
  set_smem_attr(rank_update_kernel<64>, (int)ru_smem<64>());
  set_smem_attr(rank_update_kernel<32>, (int)ru_smem<32>());
  set_smem_attr(rank_update_kernel<64, true>, (int)ru_smem<64>());
  set_smem_attr(rank_update_kernel<64, false, true>, (int)ru_smem<64>());
  set_smem_attr(rank_update_kernel<32, true>, (int)ru_smem<32>());
  set_smem_attr(xv_kernel<0, false, true>, (int)XV_SMEM);
  set_smem_attr(xv_kernel<1, false, true>, (int)XV_SMEM);
  set_smem_attr(bd_assemble_kernel, 140 * 1024);
  set_smem_attr(gram_assemble_kernel, 140 * 1024);
  set_smem_attr(gram_assemble_c_kernel, 140 * 1024);
  set_smem_attr(rank_update_real_kernel<64, true>, (int)rru_smem<64, true>());
#define BD_CHASE_ATTR(NW, DUAL, CL)                                                                        \
  set_smem_attr(bd_chase_kernel<NW, BB, DUAL, CL>, bd_chase_smem<NW, BB, DUAL>())
  BD_CHASE_ATTR(1, false, 1);
  BD_CHASE_ATTR(2, false, 1);
  BD_CHASE_ATTR(6, true, 1);
  BD_CHASE_ATTR(11, false, 1);
  BD_CHASE_ATTR(8, false, 2);
#undef BD_CHASE_ATTR
  set_smem_attr(bd_chase_pair_kernel<1, BB>, bd_chase_pair_smem<1, BB>());
  set_smem_attr(bd_chase_pair_kernel<2, BB>, bd_chase_pair_smem<2, BB>());
  set_smem_attr(bd_chase_pair_kernel<10, BB>, bd_chase_pair_smem<10, BB>());
  set_smem_attr(bd_chase_real_kernel<1, BB>, 220 * 1024);
  set_smem_attr(bd_chase_real_kernel<2, BB>, 220 * 1024);
  set_smem_attr(bd_chase_real_kernel<16, BB>, 220 * 1024);
  set_smem_attr(bd_chase_real_kernel<16, BB, 2>, bd_chase_real_smem<16, BB>());
  set_smem_attr(bd_chase_real_kernel<16, BB, 4>, bd_chase_real_smem<16, BB>());
  set_smem_attr(bd_chase_real_kernel<16, BB, 8>, bd_chase_real_smem<16, BB>());
  set_smem_attr(bd_chase_real_kernel<4, BB>, 220 * 1024);
  set_smem_attr(bd_chase_real_kernel<8, BB>, 220 * 1024);
  set_smem_attr(bd_chase_real_kernel<12, BB>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<12>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<6>, 220 * 1024);
  set_smem_attr(bd_chase_real_kernel<6, BB>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<1>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<2>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<4>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<8>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<16>, 220 * 1024);
  set_smem_attr(bd_chase_realr_kernel<16, 2>, bd_chase_realr_smem<16>());
  set_smem_attr(bd_chase_realr_kernel<8, 2>, bd_chase_realr_smem<8>());
  set_smem_attr(bd_chase_real_kernel<8, BB, 2>, bd_chase_real_smem<8, BB>());
  set_smem_attr(bd_chase_realr_kernel<16, 4>, bd_chase_realr_smem<16>());
  set_smem_attr(bd_chase_realr_kernel<16, 8>, bd_chase_realr_smem<16>());
  const char* sp = getenv("HX_CHASE_SPIN_NS");
  if (sp && sp[0]) {
    const unsigned v = (unsigned)atoi(sp);
    cudaMemcpyToSymbol(g_spin_ns, &v, sizeof(v));
  }
}

int bd_eval(const CellDev& c, const double2* kp, int nk, const uint64_t* masks, int64_t nmasks, const GridDev& g,
            int* diff, unsigned long long* trans, double* eigs, int* status, int sharp, bool real,
            size_t ws_budget, const Alloc& alloc, cudaStream_t st, RefineItem* refine,
            unsigned long long* refine_count) {
  const int S = c.nsub;
  const int64_t nmat = nmasks * nk;
  // Complex Gram path (HX_GRAM_C, default on): IDOS-only batches at k-points that are not time-reversal invariant,
  // zones clear of lambda = 0: G = C^H C (Hermitian) through the Hermitian banded tier (panel QR, 3M xv, her2k,
  // register-row chase) - half the flops of bidiagonalising C - and the mu = sigma^2 eigenvalue stage
  {
    CellDev cgc = c;
    cgc.N = S;
    if (!real && !eigs && refine && refine_count && opt("HX_GRAM_C", 1) != 0 && S > 80 &&
        gram_zones_ok(cgc, g, sharp, 1e-3)) {
      const HermSlab H = herm_slab(S);
      const size_t perg = H.stride * sizeof(double2) + 2 * sizeof(int);
      int64_t chunk = std::max<int64_t>(1, (int64_t)(ws_budget / perg));
      chunk = std::min<int64_t>(std::min<int64_t>(chunk, nmat), 65535);
      unsigned char* buf = static_cast<unsigned char*>(alloc(perg * (size_t)chunk + 256));
      if (!buf) {
        g_bd_err = "workspace allocation failed";
        return -1;
      }
      double2* ws = reinterpret_cast<double2*>(buf);
      int* dims_t = reinterpret_cast<int*>(buf + H.stride * sizeof(double2) * chunk);
      int* dims_g = dims_t + chunk;
      const size_t smem = (size_t)c.N * 8 + 2 * ((c.N + 31) / 32) * 4 + 64;
      for (int64_t m0 = 0; m0 < nmat; m0 += chunk) {
        const int64_t cnt = std::min(chunk, nmat - m0);
        gram_assemble_c_kernel<<<(unsigned)cnt, 256, smem, st>>>(c, kp, nk, masks, m0, ws, H, S, dims_t, dims_g,
                                                                 status);
        count_launch();
        BD_CUDA(cudaGetLastError());
        if (herm_reduce(ws, S, cnt, dims_g, st)) {
          g_bd_err = std::string("Hermitian reduction of the Gram matrix: ") + band_last_error();
          return -1;
        }
        launch_gram_idos(cgc, nk, g, m0, cnt, reinterpret_cast<const double*>(ws + H.dg_off), H.stride * 2, dims_t,
                         diff, trans, status, sharp, st, refine, refine_count);
        BD_CUDA(cudaGetLastError());
      }
      return 0;
    }
  }
  const BdWs L = BdWs::make(S);
  const size_t per = L.stride * sizeof(double2) + sizeof(int);
  const bool real_s1 = real && bd_real_stage1() && bd_chase_real() && S % 4 == 0;
  int64_t chunk = std::max<int64_t>(1, (int64_t)(ws_budget / per));
  chunk = std::min<int64_t>(std::min<int64_t>(chunk, nmat), 65535);
  unsigned char* buf = static_cast<unsigned char*>(alloc(per * (size_t)chunk + 256));
  if (!buf) {
    g_bd_err = "workspace allocation failed";
    return -1;
  }
  double2* ws = reinterpret_cast<double2*>(buf);
  int* dims = reinterpret_cast<int*>(buf + L.stride * sizeof(double2) * chunk);
  const size_t smem = (size_t)c.N * 8 + 2 * ((c.N + 31) / 32) * 4 + 64;
  // TGK tridiagonal of dimension up to 2S: eigenvalue kernel over cells of width 2S
  CellDev ce = c;
  ce.N = 2 * S;
  // Gram path (HX_GRAM=1): real IDOS-only batches whose transition zones stay clear of lambda = 0.  Correct
  // (tests/test_variants_gpu.py::test_gram_path_*), but measured slower on c2 (86.8 vs 63.0 ms per step): the
  // symmetric chase on the dense slab runs at half the speed of the tuned compact-band bidiagonal chase and the
  // panel / product savings (panels 11 -> 5 ms, xv 7.9 -> 3.7 ms per pass) do not cover it; off by default
  CellDev cg = c;
  cg.N = S;
  const bool gram = real_s1 && !eigs && refine && refine_count && opt("HX_GRAM", 1) != 0 &&
                    gram_zones_ok(cg, g, sharp, 1e-3);
  const bool gram_direct = gram && opt("HX_GRAM_ASSEMBLE", 1) != 0;
  for (int64_t m0 = 0; m0 < nmat; m0 += chunk) {
    const int64_t cnt = std::min(chunk, nmat - m0);
    if (gram_direct)
      gram_assemble_kernel<<<(unsigned)cnt, 256, smem, st>>>(c, kp, nk, masks, m0, ws, L, dims, status);
    else
      bd_assemble_kernel<<<(unsigned)cnt, 256, smem, st>>>(c, kp, nk, masks, m0, ws, L, dims, status,
                                                           real ? (real_s1 ? 2 : 1) : 0);
    count_launch();
    BD_CUDA(cudaGetLastError());
    if (gram) {
      if (bd_reduce_gram(ws, L, cnt, dims, status + m0, gram_direct, st)) return -1;
      launch_gram_idos(cg, nk, g, m0, cnt, reinterpret_cast<const double*>(ws + L.tgk_off), L.stride * 2, dims, diff,
                       trans, status, sharp, st, refine, refine_count);
      BD_CUDA(cudaGetLastError());
      continue;
    }
    const int rc = real_s1 ? bd_reduce_real(ws, L, cnt, dims, st)
                           : (real ? bd_reduce<true>(ws, L, cnt, dims, st) : bd_reduce<false>(ws, L, cnt, dims, st));
    if (rc) return -1;
    launch_eig_idos(ce, nk, g, m0, cnt, reinterpret_cast<const double*>(ws + L.tgk_off), L.stride * 2, dims, diff,
                    trans, eigs, status, sharp, st, refine, refine_count, true);
    BD_CUDA(cudaGetLastError());
  }
  return 0;
}

#ifdef HX_CHASE_PROFILE
extern "C" int hx_debug_chase_prof(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, hx_chase_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(hx_chase_prof, z, sizeof(z));
  }
  return 0;
}
#endif

bool bd_path_supported(const CellDev& c) {
  return c.bipartite && c.nsub >= 48 && 2 * c.nsub == c.N && c.N <= HX_MAX_N;
}

}  // namespace hx
