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
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "hx_band.cuh"
#include "hx_bidiag.cuh"
#include "hx_dense.cuh"
#include "hx_dmma.cuh"
#include "hx_kernels.cuh"
#include "hx_panel.cuh"
#include "hx_bdchase.cuh"

namespace hx {

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
  size_t c_off, v1_off, v2_off, x_off, t1_off, t2_off, tgk_off;  // double2 units
  size_t stride;
  int S;
  static BdWs make(int S) {
    BdWs w;
    w.S = S;
    w.c_off = 0;
    w.v1_off = (size_t)S * S;
    w.v2_off = w.v1_off + (size_t)S * BB;
    w.x_off = w.v2_off + (size_t)S * BB;
    w.t1_off = w.x_off + (size_t)S * BB;
    w.t2_off = w.t1_off + (size_t)BB * BB;
    w.tgk_off = w.t2_off + (size_t)BB * BB;  // diag[2S] + e2[2S] doubles = 2S double2
    w.stride = (w.tgk_off + (size_t)2 * S + 16 + 15) & ~(size_t)15;
    return w;
  }
};

__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

// ------------------------------------------------------------------------------------------------
// C = A-B block of the phase matrix per (mask, k), zero padded to S x S; dims = nA + nB.
__global__ void __launch_bounds__(256) bd_assemble_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                          const uint64_t* __restrict__ masks, int64_t mat0,
                                                          double2* ws, BdWs L, int* dims, int* status) {
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
  assemble_bipartite(c, idx_a, idx_b, kpts[kk], C, L.S, L.S, L.S, false);
}

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

// X[rows x BB] = op(A) V, op(A)[i][k] = M[ar0+i][ac0+k] (MODE 0) or conj(M[ar0+k][ac0+i]) (MODE 1),
// V [K x BB] (ld S).  64-row tiles, 4 warps x (16 x 32), DMMA m8n8k4 f64, K in chunks of 16 through a
// 3-stage cp.async pipeline.  Shared layouts keep the fragment loads conflict-free:
//   MODE 0: As[k][i] (i contiguous, the matrix's column direction), ld 66 (= 2 mod 8 in 16 B units)
//   MODE 1: As[i][k] (k contiguous), ld 20 (= 4 mod 8); the conjugate is applied at fragment load.
constexpr int XV_TM = 64, XV_TK = 16, XV_ST = 3;
constexpr int XV_LD0 = XV_TM + 2, XV_LD1 = XV_TK + 4, XV_LDV = XV_TK + 4;
constexpr int XV_A_ELEMS = XV_TK * XV_LD0 > XV_TM * XV_LD1 ? XV_TK * XV_LD0 : XV_TM * XV_LD1;
constexpr size_t XV_SMEM = (size_t)XV_ST * (XV_A_ELEMS + BB * XV_LDV) * sizeof(double2);
static_assert((size_t)(XV_TM + BB) * (BB + 4) * sizeof(double2) <= XV_SMEM, "xv epilogue tile does not fit");

template <int MODE>
__global__ void __launch_bounds__(128) xv_kernel(double2* ws, BdWs L, int ar0, int ac0, int rows, int K,
                                                 size_t v_off, size_t x_off, size_t t_off) {
  extern __shared__ __align__(16) double2 xv_sm[];
  double2* As = xv_sm;                         // [XV_ST][XV_A_ELEMS]
  double2* Vs = xv_sm + XV_ST * XV_A_ELEMS;    // [XV_ST][BB][XV_LDV]
  double2* base = ws + (size_t)blockIdx.y * L.stride;
  const int ld = L.S;
  const double2* M = base + L.c_off;
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
    double2* Vt = Vs + stg * BB * XV_LDV;
#pragma unroll
    for (int q = 0; q < BB * XV_TK / 128; ++q) {
      const int p = tid + 128 * q, kc = p & (XV_TK - 1), n = p >> 4;
      const int gk = kk + kc;
      const bool ok = gk < K;
      cp_async16_zfill(Vt + n * XV_LDV + kc, V + (ok ? gk + (size_t)n * ld : 0), ok);
    }
  };
  CTile acc[2][4];
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
    const double2* A = As + stg * XV_A_ELEMS;
    const double2* Vt = Vs + stg * BB * XV_LDV;
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
        for (int ct = 0; ct < 4; ++ct) acc[rt][ct].mac(a[rt].x, a[rt].y, b[ct].x, b[ct].y);
    }
  }
  // ---- epilogue: X <- (op(A) V) T with T (BB x BB, column-major) - the block reflector's T factor,
  //      applied on the tile in shared memory (DMMA), saving a pass over X
  cp_async_wait<0>();
  __syncthreads();
  constexpr int XL = BB + 4;  // 4 (mod 8): conflict-free fragments
  double2* Xs = xv_sm;        // [XV_TM][XL]   (reuses the pipeline stages)
  double2* Ts = xv_sm + XV_TM * XL;  // [BB (n)][XL (k)] = T[k][n]
  const double2* T = base + t_off;
  for (int p = tid; p < BB * BB; p += 128) Ts[(p / BB) * XL + (p % BB)] = T[p];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = 16 * warp + 8 * rt + (lane >> 2);
      const int cc = 8 * ct + 2 * (lane & 3);
      Xs[r * XL + cc] = make_double2(acc[rt][ct].re0, acc[rt][ct].im0);
      Xs[r * XL + cc + 1] = make_double2(acc[rt][ct].re1, acc[rt][ct].im1);
      acc[rt][ct].zero();
    }
  __syncthreads();
#pragma unroll
  for (int k4 = 0; k4 < BB / 4; ++k4) {
    const int kc = 4 * k4 + (lane & 3);
    double2 a[2], b[4];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) a[rt] = Xs[(16 * warp + 8 * rt + (lane >> 2)) * XL + kc];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) b[ct] = Ts[(8 * ct + (lane >> 2)) * XL + kc];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) acc[rt][ct].mac(a[rt].x, a[rt].y, b[ct].x, b[ct].y);
  }
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = i0 + 16 * warp + 8 * rt + (lane >> 2);
      const int cc = 8 * ct + 2 * (lane & 3);
      if (r < rows) {
        X[r + (size_t)cc * ld] = make_double2(acc[rt][ct].re0, acc[rt][ct].im0);
        X[r + (size_t)(cc + 1) * ld] = make_double2(acc[rt][ct].re1, acc[rt][ct].im1);
      }
    }
}

// M[mr0:mr0+m, mc0:mc0+n] -= U W^H, U [m x BB] and W [n x BB] (ld S); 64 x 64 tiles, DMMA.  The whole
// K = BB depth of U and W is staged once with cp.async (ld 36 = 4 mod 8: conflict-free fragments) while
// the C tile is read straight into the accumulators; 2 CTAs per SM.
constexpr int RU_T = 64, RU_LD = BB + 4;
constexpr size_t RU_SMEM = (size_t)2 * RU_T * RU_LD * sizeof(double2);

__global__ void __launch_bounds__(256, 2) rank_update_kernel(double2* ws, BdWs L, int mr0, int mc0, int m, int n,
                                                             size_t u_off, size_t w_off) {
  extern __shared__ __align__(16) double2 ru_sm[];
  double2* Us = ru_sm;                // [RU_T][RU_LD]
  double2* Ws = ru_sm + RU_T * RU_LD;  // [RU_T][RU_LD]
  double2* base = ws + (size_t)blockIdx.z * L.stride;
  const int ld = L.S;
  double2* M = base + L.c_off + (size_t)mc0 * ld + mr0;
  const double2* U = base + u_off;
  const double2* W = base + w_off;
  const int I0 = blockIdx.x * RU_T, J0 = blockIdx.y * RU_T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
#pragma unroll
  for (int q = 0; q < RU_T * BB / 256; ++q) {
    const int p = tid + 256 * q, r = p & (RU_T - 1), k = p >> 6;
    const size_t col = (size_t)k * ld;
    const bool oku = I0 + r < m, okw = J0 + r < n;
    cp_async16_zfill(Us + r * RU_LD + k, U + (oku ? I0 + r + col : 0), oku);
    cp_async16_zfill(Ws + r * RU_LD + k, W + (okw ? J0 + r + col : 0), okw);
  }
  cp_async_commit();
  CTile acc[2][4];
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
    }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int k4 = 0; k4 < BB / 4; ++k4) {
    const int kc = 4 * k4 + (lane & 3);
    double2 au[2], bw[4];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) au[rt] = Us[(16 * wr + 8 * rt + (lane >> 2)) * RU_LD + kc];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) bw[ct] = conj2(Ws[(32 * wc + 8 * ct + (lane >> 2)) * RU_LD + kc]);
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) acc[rt][ct].mac(-au[rt].x, -au[rt].y, bw[ct].x, bw[ct].y);
  }
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int r = I0 + 16 * wr + 8 * rt + (lane >> 2);
      const int cc = J0 + 32 * wc + 8 * ct + 2 * (lane & 3);
      if (r < m && cc < n) M[r + (size_t)cc * ld] = make_double2(acc[rt][ct].re0, acc[rt][ct].im0);
      if (r < m && cc + 1 < n) M[r + (size_t)(cc + 1) * ld] = make_double2(acc[rt][ct].re1, acc[rt][ct].im1);
    }
}


// ------------------------------------------------------------------------------------------------
bool launch_cluster_panel(double2* ws, const PanelArgs& a, int64_t cnt, cudaStream_t st);

static int bd_reduce(double2* ws, const BdWs& L, int64_t cnt, const int* dims, cudaStream_t st) {
  const int S = L.S;
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
    xv_kernel<1><<<dim3((unsigned)((n2 + XV_TM - 1) / XV_TM), (unsigned)cnt), 128, XV_SMEM, st>>>(
        ws, L, k0, k0 + BB, n2, m1, L.v1_off, L.x_off, L.t1_off);
    rank_update_kernel<<<dim3((unsigned)((m1 + RU_T - 1) / RU_T), (unsigned)((n2 + RU_T - 1) / RU_T), (unsigned)cnt),
                         256, RU_SMEM, st>>>(ws, L, k0, k0 + BB, m1, n2, L.v1_off, L.x_off);
    count_launch(2);
    // ---- right: row panel LQ, C_tr2 = C[k0+BB:, k0+BB:] <- C_tr2 Q2
    PanelArgs p2{L.stride, L.c_off, S, k0, k0 + BB, n2, 1, L.v2_off, S, L.t2_off};
    if (!launch_cluster_panel(ws, p2, cnt, st)) {
      g_bd_err = "panel does not fit the cluster shared memory";
      return -1;
    }
    count_launch();
    const int m3 = S - k0 - BB;
    if (m3 > 0) {
      xv_kernel<0><<<dim3((unsigned)((m3 + XV_TM - 1) / XV_TM), (unsigned)cnt), 128, XV_SMEM, st>>>(
          ws, L, k0 + BB, k0 + BB, m3, n2, L.v2_off, L.x_off, L.t2_off);
      rank_update_kernel<<<dim3((unsigned)((m3 + RU_T - 1) / RU_T), (unsigned)((n2 + RU_T - 1) / RU_T),
                                (unsigned)cnt),
                           256, RU_SMEM, st>>>(ws, L, k0 + BB, k0 + BB, m3, n2, L.x_off, L.v2_off);
      count_launch(2);
    }
    BD_CUDA(cudaGetLastError());
  }
  // ---- stage 2: enough sweeps in flight to fill the SMs.  Large batches (throughput-bound) use the
  // single-tile variant (12 warps per SM); small ones the dual-tile one (lower latency per task).
  static const int chase_mode = [] {
    const char* e = getenv("HX_CHASE_MODE");
    return e ? atoi(e) : 0;
  }();
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
  if (want >= 6) {
    if (chase_mode == 1) BD_CHASE(11, false, 1)
    else if (chase_mode == 2) BD_CHASE(6, true, 1)
    else BD_CHASE(8, false, 2)
  } else if (want >= 2) {
    BD_CHASE(2, false, 1)
  } else {
    BD_CHASE(1, false, 1)
  }
#undef BD_CHASE
  count_launch();
  BD_CUDA(cudaGetLastError());
  return 0;
}

void bd_init_attributes() {
  cudaFuncSetAttribute(xv_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XV_SMEM);
  cudaFuncSetAttribute(xv_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XV_SMEM);
  cudaFuncSetAttribute(rank_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RU_SMEM);
  cudaFuncSetAttribute(bd_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
#define BD_CHASE_ATTR(NW, DUAL, CL)                                                                        \
  cudaFuncSetAttribute(bd_chase_kernel<NW, BB, DUAL, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       (int)bd_chase_smem<NW, BB, DUAL>())
  BD_CHASE_ATTR(1, false, 1);
  BD_CHASE_ATTR(2, false, 1);
  BD_CHASE_ATTR(6, true, 1);
  BD_CHASE_ATTR(11, false, 1);
  BD_CHASE_ATTR(8, false, 2);
#undef BD_CHASE_ATTR
}

int bd_eval(const CellDev& c, const double2* kp, int nk, const uint64_t* masks, int64_t nmasks, const GridDev& g,
            int* diff, unsigned long long* trans, double* eigs, int* status, int sharp, size_t ws_budget,
            const Alloc& alloc, cudaStream_t st, RefineItem* refine, unsigned long long* refine_count) {
  const int S = c.nsub;
  const BdWs L = BdWs::make(S);
  const size_t per = L.stride * sizeof(double2) + sizeof(int);
  const int64_t nmat = nmasks * nk;
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
  for (int64_t m0 = 0; m0 < nmat; m0 += chunk) {
    const int64_t cnt = std::min(chunk, nmat - m0);
    bd_assemble_kernel<<<(unsigned)cnt, 256, smem, st>>>(c, kp, nk, masks, m0, ws, L, dims, status);
    count_launch();
    BD_CUDA(cudaGetLastError());
    if (bd_reduce(ws, L, cnt, dims, st)) return -1;
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
