// Gram path of the bipartite (graphene) banded tier for real (time-reversal-invariant) IDOS batches.
//
// The eigenvalues of T = [[0, C], [C^T, 0]] are +-sigma(C) (plus zeros), and sigma^2 are the eigenvalues of
// G = C^T C.  G is symmetric with ~7 nonzeros per column (B sites sharing an A neighbour), formed in O(S) from
// the sparsity of C; its tridiagonalisation is a one-sided-per-step symmetric two-stage reduction - ONE panel
// QR and ONE product per step instead of the two of the bidiagonal reduction of C - followed by a symmetric
// band chase, and its tridiagonal has dimension S instead of the 2S of the TGK form.  The eigenvalue stage
// counts and refines in mu = sigma^2 (zone_count_gram_kernel); sigma^2 keeps full relative accuracy away from
// sigma = 0, and the host uses the path only when no transition zone comes near lambda = 0 (gram_zones_ok).
//
//   gram_build_kernel       dense C (slab, ld S) -> sparse column / row lists -> dense G in place
//   stage 1 (per k0)        panel_qr_real (column panel below the band) -> Y = G22 V T (xv_real) ->
//                           w_fix_real_kernel: W = Y - 1/2 V (T^T (V^T Y)) -> G22 -= W V^T, G22 -= V W^T (DMMA)
//   sym_chase_real_kernel   symmetric band (lower, width 32) -> tridiagonal (diag, e2)
#pragma once
#include "hx_dense.cuh"
#include "hx_real.cuh"

namespace hx {

constexpr int GRAM_K = 8;  // nonzeros kept per row / column of C (graphene: 3)

// One CTA per matrix.  C: S x S doubles (ld S) at base + c_off; scratch (>= S * GRAM_K * 6 + 2 S doubles) at
// base + l_off; G overwrites C.  Every column of G is accumulated by one thread in a fixed order (the lists are
// in row / column order), so the result is deterministic.  A row or column of C with more than GRAM_K nonzeros
// (not graphene) marks the matrix failed (status, this chunk's rows).
__global__ void __launch_bounds__(256) gram_build_kernel(double* ws, size_t stride, size_t c_off, size_t l_off, int S,
                                                         int* status) {
  double* base = ws + (size_t)blockIdx.x * stride;
  double* C = base + c_off;
  double* colVal = base + l_off;                                   // [S][GRAM_K]
  double* rowVal = colVal + (size_t)S * GRAM_K;                    // [S][GRAM_K]
  int* colIdx = reinterpret_cast<int*>(rowVal + (size_t)S * GRAM_K);  // [S][GRAM_K]
  int* rowIdx = colIdx + (size_t)S * GRAM_K;                       // [S][GRAM_K]
  int* colCnt = rowIdx + (size_t)S * GRAM_K;                       // [S]
  int* rowCnt = colCnt + S;                                        // [S]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ int over;
  if (tid == 0) over = 0;
  __syncthreads();
  // columns: one warp per column, lanes over rows (coalesced), ballot-compacted in row order
  for (int j = warp; j < S; j += nw) {
    int cnt = 0;
    for (int r0 = 0; r0 < S; r0 += 32) {
      const int r = r0 + lane;
      const double v = r < S ? C[r + (size_t)j * S] : 0.0;
      const unsigned nzb = __ballot_sync(0xffffffffu, v != 0.0);
      const int pos = cnt + __popc(nzb & ((1u << lane) - 1u));
      if (v != 0.0) {
        if (pos < GRAM_K) {
          colIdx[(size_t)j * GRAM_K + pos] = r;
          colVal[(size_t)j * GRAM_K + pos] = v;
        } else {
          over = 1;
        }
      }
      cnt += __popc(nzb);
    }
    if (lane == 0) colCnt[j] = min(cnt, GRAM_K);
  }
  // rows: one thread per row, columns in order (consecutive threads read consecutive rows: coalesced)
  for (int i = tid; i < S; i += blockDim.x) {
    int cnt = 0;
    for (int c = 0; c < S; ++c) {
      const double v = C[i + (size_t)c * S];
      if (v != 0.0) {
        if (cnt < GRAM_K) {
          rowIdx[(size_t)i * GRAM_K + cnt] = c;
          rowVal[(size_t)i * GRAM_K + cnt] = v;
        } else {
          over = 1;
        }
        ++cnt;
      }
    }
    rowCnt[i] = min(cnt, GRAM_K);
  }
  __syncthreads();
  for (size_t p = tid; p < (size_t)S * S; p += blockDim.x) C[p] = 0.0;
  __syncthreads();
  // G[:, j] = sum_{i in col(j)} C_ij C[i, :]^T
  for (int j = tid; j < S; j += blockDim.x) {
    double* Gj = C + (size_t)j * S;
    const int nc = colCnt[j];
    for (int a = 0; a < nc; ++a) {
      const int i = colIdx[(size_t)j * GRAM_K + a];
      const double cij = colVal[(size_t)j * GRAM_K + a];
      const int nr = rowCnt[i];
      for (int b = 0; b < nr; ++b) {
        const int k = rowIdx[(size_t)i * GRAM_K + b];
        Gj[k] = fma(cij, rowVal[(size_t)i * GRAM_K + b], Gj[k]);
      }
    }
  }
  if (tid == 0 && over) status[blockIdx.x] = 2;  // HX_ST_NONFINITE: surfaces as an error, never silently
}

// W = Y - 1/2 V (T^T (V^T Y)) for the m rows of the step (Y = X at x_off, overwritten), V at v_off, T at t_off
// (doubles, ld = ld), one CTA per matrix.
__global__ void __launch_bounds__(256) w_fix_real_kernel(double* ws, RSlab g, int m, size_t v_off, size_t x_off,
                                                         size_t t_off) {
  __shared__ double Vs[32][33], Ys[32][33], Zs[32][33], Ms[32][33];
  double* base = ws + (size_t)blockIdx.x * g.stride;
  const double* V = base + v_off;
  double* Y = base + x_off;
  const double* T = base + t_off;
  const int ld = g.ld, tid = threadIdx.x;
  const int a0 = tid >> 5, b = tid & 31;  // this thread: Z[a0 + 8 q][b], q < 4
  double z[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r0 = 0; r0 < m; r0 += 32) {
    for (int p = tid; p < 1024; p += 256) {
      const int rr = p & 31, c = p >> 5;
      const bool ok = r0 + rr < m;
      Vs[rr][c] = ok ? V[r0 + rr + (size_t)c * ld] : 0.0;
      Ys[rr][c] = ok ? Y[r0 + rr + (size_t)c * ld] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      const double y = Ys[rr][b];
#pragma unroll
      for (int q = 0; q < 4; ++q) z[q] = fma(Vs[rr][a0 + 8 * q], y, z[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) Zs[a0 + 8 * q][b] = z[q];
  for (int p = tid; p < 1024; p += 256) Vs[p & 31][p >> 5] = T[p];  // Vs[l][a] = T[l][a] (column-major T)
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // Ms = 1/2 T^T Z: Ms[a][b] = 1/2 sum_l T[l][a] Z[l][b]
    const int a = a0 + 8 * q;
    double t = 0.0;
    for (int l = 0; l < 32; ++l) t = fma(Vs[l][a], Zs[l][b], t);
    Ms[a][b] = 0.5 * t;
  }
  __syncthreads();
  for (int r0 = 0; r0 < m; r0 += 32) {
    for (int p = tid; p < 1024; p += 256) {
      const int rr = p & 31, c = p >> 5;
      Vs[rr][c] = r0 + rr < m ? V[r0 + rr + (size_t)c * ld] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rr = a0 + 8 * q;
      if (r0 + rr < m) {
        double w = Y[r0 + rr + (size_t)b * ld];
        for (int a = 0; a < 32; ++a) w = fma(-Vs[rr][a], Ms[a][b], w);
        Y[r0 + rr + (size_t)b * ld] = w;
      }
    }
    __syncthreads();
  }
}

// W = Y - 1/2 V (T^T (V^T Y)) in two launches with row-chunk parallelism (w_fix_real_kernel runs one CTA per
// matrix: 0.53 ms per step on the 64-matrix N = 2048 tier).  gram_vty_kernel: partial Z = V^T Y of each chunk of
// GRAM_WR rows (grid: chunks x matrices) to P[chunk][32 x 32]; gram_wfix_kernel: every CTA sums the partials in
// chunk order (fixed order: deterministic), forms M = 1/2 T^T Z and updates its own rows, W = Y - V M.
constexpr int GRAM_WR = 128;

__global__ void __launch_bounds__(256) gram_vty_kernel(double* ws, RSlab g, int m, size_t v_off, size_t x_off,
                                                       size_t p_off) {
  __shared__ double Vs[32][33], Ys[32][33];
  double* base = ws + (size_t)blockIdx.y * g.stride;
  const double* V = base + v_off;
  const double* Y = base + x_off;
  double* P = base + p_off + (size_t)blockIdx.x * 1024;
  const int ld = g.ld, tid = threadIdx.x;
  const int rb = blockIdx.x * GRAM_WR, re = min(m, rb + GRAM_WR);
  const int a0 = tid >> 5, b = tid & 31;  // this thread: Z[a0 + 8 q][b], q < 4
  double z[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r0 = rb; r0 < re; r0 += 32) {
    for (int p = tid; p < 1024; p += 256) {
      const int rr = p & 31, c = p >> 5;
      const bool ok = r0 + rr < re;
      Vs[rr][c] = ok ? V[r0 + rr + (size_t)c * ld] : 0.0;
      Ys[rr][c] = ok ? Y[r0 + rr + (size_t)c * ld] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      const double y = Ys[rr][b];
#pragma unroll
      for (int q = 0; q < 4; ++q) z[q] = fma(Vs[rr][a0 + 8 * q], y, z[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) P[(a0 + 8 * q) * 32 + b] = z[q];
}

__global__ void __launch_bounds__(256) gram_wfix_kernel(double* ws, RSlab g, int m, int nchunks, size_t v_off,
                                                        size_t x_off, size_t t_off, size_t p_off) {
  __shared__ double Vs[32][33], Zs[32][33], Ms[32][33];
  double* base = ws + (size_t)blockIdx.y * g.stride;
  const double* V = base + v_off;
  double* Y = base + x_off;
  const double* T = base + t_off;
  const double* P = base + p_off;
  const int ld = g.ld, tid = threadIdx.x;
  const int rb = blockIdx.x * GRAM_WR, re = min(m, rb + GRAM_WR);
  const int a0 = tid >> 5, b = tid & 31;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = a0 + 8 * q;
    double z = 0.0;
    for (int ch = 0; ch < nchunks; ++ch) z += P[(size_t)ch * 1024 + a * 32 + b];
    Zs[a][b] = z;
  }
  for (int p = tid; p < 1024; p += 256) Vs[p & 31][p >> 5] = T[p];  // Vs[l][a] = T[l][a] (column-major T)
  __syncthreads();
  {  // Ms[a][b] = 1/2 sum_l T[l][a] Z[l][b], a = a0 + 8 q: one Z load per four products
    double t[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
    for (int l = 0; l < 32; ++l) {
      const double zl = Zs[l][b];
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = fma(Vs[l][a0 + 8 * q], zl, t[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) Ms[a0 + 8 * q][b] = 0.5 * t[q];
  }
  __syncthreads();
  // rows: lane = row (coalesced Y loads and stores), warp + 8 q = column; one V load per four products (the
  // kernel was bound by its shared-memory loads: two per FMA, 144 us on the 1024-matrix launches)
  for (int r0 = rb; r0 < re; r0 += 32) {
    for (int p = tid; p < 1024; p += 256) {
      const int rr = p & 31, c = p >> 5;
      Vs[rr][c] = r0 + rr < re ? V[r0 + rr + (size_t)c * ld] : 0.0;
    }
    __syncthreads();
    if (r0 + b < re) {
      double w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = Y[r0 + b + (size_t)(a0 + 8 * q) * ld];
#pragma unroll 8
      for (int a = 0; a < 32; ++a) {
        const double va = Vs[b][a];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = fma(-va, Ms[a][a0 + 8 * q], w[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Y[r0 + b + (size_t)(a0 + 8 * q) * ld] = w[q];
    }
    __syncthreads();
  }
}

// Real symmetric band (lower, width BWc, dense slab A with ld S) -> tridiagonal (diag[S], e2[S] doubles at
// out), pipelined over sweeps exactly as bulge_chase_pipe_kernel (hx_chase.cuh) on real data: task t of sweep
// i updates the diagonal block D = A[s:s+len, s:s+len] two-sidedly (p = D v, w = tau p - tau^2/2 (v.p) v,
// D -= v w^T + w v^T) and the block below it, B'' = B - q v^T - v' z^T (q = tau B v; H' from column 0 of B H).
struct SymChaseSmem {
  double D[32][33];
  double v[32], w[32], vp[32], z[32];
};

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) sym_chase_real_kernel(double* ws, size_t stride, size_t a_off,
                                                                     size_t out_off, int S) {
  constexpr int BWc = 32;
  extern __shared__ __align__(16) unsigned char scs_raw[];
  SymChaseSmem* all = reinterpret_cast<SymChaseSmem*>(scs_raw);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SymChaseSmem& W = all[warp];
  double* base = ws + (size_t)blockIdx.x * stride;
  double* A = base + a_off;
  double* diag = base + out_off;
  double* e2 = diag + S;
  const int lda = S, d = S;
  if (lane == 0) prog[warp] = -1;
  for (int q = threadIdx.x; q < 2 * S; q += blockDim.x) diag[q] = 0.0;
  __syncthreads();
  const int nsweeps = d - 1;
  for (int i = warp; i < nsweeps; i += NW) {
    const int tasks = (d - 1 - i + BWc - 1) / BWc;
    const int prev_tasks = i > 0 ? (d - i + BWc - 1) / BWc : 0;
    const int pw = (i - 1 + NW) % NW;
    double tau = 0.0;
    for (int t = 0; t < tasks; ++t) {
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 2, prev_tasks);
        if (lane == 0)
          while (prog[pw] < need) __nanosleep(20);
        __syncwarp();
        __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, d - s);
      const int lb = max(0, min(BWc, d - s - len));
      double* const colp = A + ((size_t)s * lda + s + lane);  // (s + lane, s + c) at colp[c * lda]
      // D: lower triangle, mirrored
#pragma unroll 4
      for (int c = 0; c < BWc; ++c) W.D[lane][c] = (c < len && lane >= c && lane < len) ? colp[(size_t)c * lda] : 0.0;
      if (t == 0) {
        const double x = lane < len ? A[s + lane + (size_t)i * lda] : 0.0;  // column i, rows s ..
        const double sig2 = warp_sum(x * x);
        const QuickReflectorR h = quick_reflector_r(__shfl_sync(0xffffffffu, x, 0), sig2);
        tau = h.tau;
        W.v[lane] = lane == 0 ? 1.0 : (lane < len ? x * h.scale : 0.0);
        if (lane < len && tau != 0.0) A[s + lane + (size_t)i * lda] = lane == 0 ? h.beta : 0.0;
        if (lane == 0) {
          diag[i] = A[i + (size_t)i * lda];
          e2[i] = sig2;
        }
      }
      __syncwarp();
#pragma unroll 4
      for (int c = 0; c < BWc; ++c)
        if (c > lane) W.D[lane][c] = W.D[c][lane];
      __syncwarp();
      // p = D v (lane = row), w = tau p - tau^2/2 (v.p) v
      double p;
      {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int c = 0; c < BWc; c += 2) {
          a0 = fma(W.D[lane][c], W.v[c], a0);
          a1 = fma(W.D[lane][c + 1], W.v[c + 1], a1);
        }
        p = a0 + a1;
      }
      const double vr = W.v[lane];
      const double cval = warp_sum(vr * p);
      const double wr = tau * p - 0.5 * tau * tau * cval * vr;
      W.w[lane] = wr;
      __syncwarp();
      if (lane < len) {
#pragma unroll 4
        for (int c = 0; c < BWc; ++c) {
          const double z = W.D[lane][c] - (vr * W.w[c] + wr * W.v[c]);
          if (c <= lane && c < len) colp[(size_t)c * lda] = z;
        }
      }
      if (lb > 0) {
        __syncwarp();
#pragma unroll 4
        for (int c = 0; c < BWc; ++c) W.D[lane][c] = (c < len && lane < lb) ? colp[len + (size_t)c * lda] : 0.0;
        __syncwarp();
        // q = tau B v (lane = row); column 0 of B - q v^T -> H'
        double q;
        {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
          for (int c = 0; c < BWc; c += 2) {
            a0 = fma(W.D[lane][c], W.v[c], a0);
            a1 = fma(W.D[lane][c + 1], W.v[c + 1], a1);
          }
          q = tau * (a0 + a1);
        }
        const double x0 = W.D[lane][0] - q;
        const double sg2 = warp_sum(x0 * x0);
        const QuickReflectorR hp = quick_reflector_r(__shfl_sync(0xffffffffu, x0, 0), sg2);
        const double vpr = lane == 0 ? 1.0 : x0 * hp.scale;  // zero on padded rows
        W.vp[lane] = vpr;
        const double wq = warp_sum(vpr * q);
        __syncwarp();
        // column pass (lane = column): z_c = tau' (v'.B[:, c] - wq v_c)
        {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
          for (int r = 0; r < BWc; r += 2) {
            a0 = fma(W.vp[r], W.D[r][lane], a0);
            a1 = fma(W.vp[r + 1], W.D[r + 1][lane], a1);
          }
          W.z[lane] = hp.tau * (a0 + a1 - wq * W.v[lane]);
        }
        __syncwarp();
        if (lane < lb) {
#pragma unroll 4
          for (int c = 0; c < BWc; ++c) {
            double y = W.D[lane][c] - (q * W.v[c] + vpr * W.z[c]);
            if (c == 0 && hp.tau != 0.0) y = lane == 0 ? hp.beta : 0.0;
            if (c < len) colp[len + (size_t)c * lda] = y;
          }
        }
        __syncwarp();
        W.v[lane] = vpr;
        tau = hp.tau;
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[warp] = i * 65536 + t + 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) diag[d - 1] = A[d - 1 + (size_t)(d - 1) * lda];
}

template <int NW>
constexpr size_t sym_chase_real_smem() {
  return NW * sizeof(SymChaseSmem) + 64;
}

// ---------------------------------------------------------------------------------------------------
// Register-row symmetric chase on a compact lower band (the layout and task pipeline of bd_chase_realr_kernel,
// hx_bdchase.cuh, for the symmetric band of the Gram path).  Element (r, c), c <= r <= c + 63 (the band of width
// 32 plus the bulge of the tile below the diagonal tile) at Bs[c * SB_LD + r - c]: 64 doubles per column instead
// of the 96 of the bidiagonal chase's band (and of the S of the dense slab), so the bands of a many-matrix launch
// stay in L2.  The lane's row of the diagonal tile D (lower triangle from the band, coalesced; the mirrored part
// through the transposed shared-memory copy) and then of the tile B below it live in 32 registers: p = D v, the
// rank-2 updates D -= v w^T + w v^T and B -= q v^T + v' z^T run on registers, shared memory carries only the
// broadcast vectors and the transposed tile of the column pass.  One reflector and two reduction rounds per task
// (the bidiagonal task has two reflectors and two paired rounds).
constexpr int SB_LD = 64;

// Progress counters of the cluster launches: release / acquire at cluster scope on the (distributed) shared-memory
// word instead of device-scope fences around a volatile access.  The tile stores of the 32 lanes are ordered
// before lane 0's release by the __syncwarp() in front of it (cumulativity); the consumer's tile loads
// (ld.global.cg) follow lane 0's acquire through the __syncwarp() behind the poll.
__device__ __forceinline__ void st_release_cluster(volatile int* p, int v) {
  asm volatile("st.release.cluster.s32 [%0], %1;" ::"l"(const_cast<int*>(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cluster(const volatile int* p) {
  int v;
  asm volatile("ld.acquire.cluster.s32 %0, [%1];" : "=r"(v) : "l"(const_cast<int*>(p)) : "memory");
  return v;
}

struct __align__(16) SymChaseSmemRR {
  double v[32], w[32], vp[32], z[32];
  double Xt[32][33];  // Xt[c][r] = tile (r, c)
};

// Lower band (width 32) of the dense S x S slab A into the compact band; the bulge window starts as zero.
static __global__ void __launch_bounds__(256) sym_band_extract_kernel(double* ws, size_t stride, size_t a_off,
                                                                       size_t band_off, int S) {
  double* base = ws + (size_t)blockIdx.x * stride;
  const double* A = base + a_off;
  double* B = base + band_off;
  const size_t n = (size_t)S * SB_LD;
  for (size_t p = threadIdx.x; p < n; p += blockDim.x) {
    const int c = (int)(p / SB_LD), j = (int)(p % SB_LD), r = c + j;
    B[p] = (j <= 32 && r < S) ? A[r + (size_t)c * S] : 0.0;
  }
}

template <int NW, int CL = 1>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NW * 32, NW == 4 ? 4 : (NW <= 2 ? 8 : 1))
    sym_chase_realr_kernel(double* ws, size_t stride, size_t band_off, size_t out_off, int S, const int* dims) {
  constexpr int BWc = 32, RS = SB_LD - 1;  // RS: one column to the right along a row
  // Progress counters count HALF tasks (D part, B part).  HALF (few matrices, critical-path-bound launches): the D
  // part of task t waits only for the D part of task t + 1 of the previous sweep (its last overlap is the element
  // (s + 31, s + 31)), the B part for that task's B part - sweep i + 1 trails sweep i by 1.5 tasks instead of 2.
  // Many-matrix launches keep one wait and one publish per task.
  constexpr bool HALF = CL > 1 || NW >= 8;
  extern __shared__ __align__(16) unsigned char scr_raw[];
  SymChaseSmemRR* all = reinterpret_cast<SymChaseSmemRR*>(scr_raw);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SymChaseSmemRR& W = all[warp];
  const int rank = CL > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int gw = rank * NW + warp;
  constexpr int TW = CL * NW;
  const int64_t mat = blockIdx.x / CL;
  double* base = ws + (size_t)mat * stride;
  double* B = base + band_off;
  double* diag = base + out_off;
  double* e2 = diag + S;
  for (int q = threadIdx.x + rank * blockDim.x; q < 2 * S; q += blockDim.x * CL) diag[q] = 0.0;
  if (lane == 0) prog[warp] = -1;
  if constexpr (CL > 1) {
    __threadfence();
    cooperative_groups::this_cluster().sync();
  } else {
    __syncthreads();
  }
  const bool skip = dims && dims[mat] == 0;
  const int nsweeps = skip ? 0 : S - 1;
  for (int i = gw; i < nsweeps; i += TW) {
    const int tasks = (S - 1 - i + BWc - 1) / BWc;
    const int prev_tasks = i > 0 ? (S - i + BWc - 1) / BWc : 0;
    volatile int* pflag;  // progress counter of the warp that owns sweep i - 1
    {
      const int gp = (i - 1 + TW) % TW;
      if constexpr (CL > 1)
        pflag = cooperative_groups::this_cluster().map_shared_rank(const_cast<int*>(prog), gp / NW) + gp % NW;
      else pflag = prog + gp;
    }
    double tau = 0.0, vr = 0.0;
    for (int t = 0; t < tasks; ++t) {
      if (i > 0) {
        const int need = (i - 1) * 65536 + (HALF ? min(2 * t + 3, 2 * prev_tasks) : 2 * min(t + 2, prev_tasks));
        if constexpr (CL > 1) {
          if (lane == 0)
            while (ld_acquire_cluster(pflag) < need) __nanosleep(g_spin_ns);
          __syncwarp();
        } else {
          if (lane == 0)
            while (*pflag < need) __nanosleep(g_spin_ns);
          __syncwarp();
          __threadfence_block();
        }
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, S - s);
      const int lb = max(0, min(BWc, S - s - len));
      double* const blk = B + ((size_t)s * SB_LD + lane);  // (s + lane, s + c), c <= lane, at blk[c * RS]
      double xr[BWc];
      {
        const int nc = lane < len ? lane + 1 : 0;  // lower triangle of the diagonal tile
#pragma unroll
        for (int cc = 0; cc < BWc; ++cc) xr[cc] = cc < nc ? ld_band<CL>(blk + cc * RS) : 0.0;
      }
      if (t == 0) {
        // reflector from column i, rows [s, s + len): column i -> (beta, 0, ...)
        double* const coli = B + ((size_t)i * SB_LD + 1 + lane);  // (s + lane, i)
        const double x = lane < len ? ld_band<CL>(coli) : 0.0;
        const double sig2 = warp_sum(x * x);
        const QuickReflectorR h = quick_reflector_r(__shfl_sync(0xffffffffu, x, 0), sig2);
        tau = h.tau;
        vr = lane == 0 ? 1.0 : (lane < len ? x * h.scale : 0.0);
        W.v[lane] = vr;
        if (lane < len && tau != 0.0) *coli = lane == 0 ? h.beta : 0.0;
        if (lane == 0) {
          diag[i] = ld_band<CL>(B + (size_t)i * SB_LD);
          e2[i] = sig2;
        }
      }
#pragma unroll
      for (int cc = 0; cc < BWc; ++cc) W.Xt[cc][lane] = xr[cc];
      __syncwarp();
      // mirrored part of the lane's row: D[lane][c] = D[c][lane] for c > lane
#pragma unroll
      for (int cc = 1; cc < BWc; ++cc)
        if (cc > lane) xr[cc] = W.Xt[lane][cc];
      // ---- p = D v (registers), w = tau p - tau^2/2 (v.p) v
      double p;
      {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int c = 0; c < BWc; c += 2) {
          const double2 u = lds2(&W.v[c]);
          a0 = fma(xr[c], u.x, a0);
          a1 = fma(xr[c + 1], u.y, a1);
        }
        p = a0 + a1;
      }
      const double cval = warp_sum(vr * p);
      const double wr = tau * p - 0.5 * tau * tau * cval * vr;
      W.w[lane] = wr;
      __syncwarp();
      // ---- D' = D - v w^T - w v^T on the lower triangle, straight to the band
      if (lane < len) {
#pragma unroll
        for (int c = 0; c < BWc; c += 2) {
          const double2 u = lds2(&W.v[c]), b = lds2(&W.w[c]);
          const double z0 = fma(-wr, u.x, fma(-vr, b.x, xr[c]));
          const double z1 = fma(-wr, u.y, fma(-vr, b.y, xr[c + 1]));
          if (c <= lane) blk[c * RS] = z0;
          if (c + 1 <= lane) blk[(c + 1) * RS] = z1;
          if ((c & 7) == 6) asm volatile("" ::: "memory");  // bound the broadcast loads in flight (registers)
        }
      }
      if constexpr (HALF) {
        // D part done: publish, then wait for the B part of task t + 1 of the previous sweep
        if constexpr (CL > 1) {
          __syncwarp();
          if (lane == 0) st_release_cluster(&prog[warp], i * 65536 + 2 * t + 1);
        } else {
          __threadfence_block();
          __syncwarp();
          if (lane == 0) prog[warp] = i * 65536 + 2 * t + 1;
        }
        if (i > 0 && lb > 0) {
          const int need = (i - 1) * 65536 + min(2 * t + 4, 2 * prev_tasks);
          if constexpr (CL > 1) {
            if (lane == 0)
              while (ld_acquire_cluster(pflag) < need) __nanosleep(g_spin_ns);
            __syncwarp();
          } else {
            if (lane == 0)
              while (*pflag < need) __nanosleep(g_spin_ns);
            __syncwarp();
            __threadfence_block();
          }
        }
      }
      if (lb > 0) {
        // tile below: (s + 32 + lane, s + c) at blk[32 + c * RS] (len == 32 here)
        double* const blk2 = blk + BWc;
        {
          const bool rowok = lane < lb;
#pragma unroll
          for (int cc = 0; cc < BWc; ++cc) xr[cc] = rowok ? ld_band<CL>(blk2 + cc * RS) : 0.0;
        }
#pragma unroll
        for (int cc = 0; cc < BWc; ++cc) W.Xt[cc][lane] = xr[cc];
        // ---- q = tau B v (registers); column 0 of B - q v^T -> H'
        double q;
        {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int c = 0; c < BWc; c += 2) {
            const double2 u = lds2(&W.v[c]);
            a0 = fma(xr[c], u.x, a0);
            a1 = fma(xr[c + 1], u.y, a1);
          }
          q = tau * (a0 + a1);
        }
        const double x0 = xr[0] - q;
        // one reduction round for |x0|^2 and sum_{r>=1} x0_r q_r: v'.q = q_0 + scale * that
        double sg2 = x0 * x0, qx = lane == 0 ? 0.0 : x0 * q;
        warp_sum2(sg2, qx);
        const QuickReflectorR hp = quick_reflector_r(__shfl_sync(0xffffffffu, x0, 0), sg2);
        const double vpr = lane == 0 ? 1.0 : x0 * hp.scale;  // zero on padded rows
        const double wq = fma(hp.scale, qx, __shfl_sync(0xffffffffu, q, 0));
        W.vp[lane] = vpr;
        __syncwarp();
        // ---- column pass (lane = column): z_c = tau' (v'.B[:, c] - (v'.q) v_c)
        {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int r = 0; r < BWc; r += 2) {
            const double2 vv = lds2(&W.vp[r]);
            a0 = fma(vv.x, W.Xt[lane][r], a0);
            a1 = fma(vv.y, W.Xt[lane][r + 1], a1);
          }
          W.z[lane] = hp.tau * (a0 + a1 - wq * W.v[lane]);
        }
        __syncwarp();
        // ---- B'' = B - q v^T - v' z^T, to the band
        if (lane < lb) {
          const bool row0 = hp.tau != 0.0;
#pragma unroll
          for (int c = 0; c < BWc; c += 2) {
            const double2 u = lds2(&W.v[c]), zz = lds2(&W.z[c]);
            double y0 = fma(-vpr, zz.x, fma(-q, u.x, xr[c]));
            const double y1 = fma(-vpr, zz.y, fma(-q, u.y, xr[c + 1]));
            if (c == 0 && row0) y0 = lane == 0 ? hp.beta : 0.0;
            blk2[c * RS] = y0;
            blk2[(c + 1) * RS] = y1;
            if ((c & 7) == 6) asm volatile("" ::: "memory");
          }
        }
        __syncwarp();  // every lane is done with v
        W.v[lane] = vpr;
        vr = vpr;
        tau = hp.tau;
      }
      if constexpr (CL > 1) {
        __syncwarp();
        if (lane == 0) st_release_cluster(&prog[warp], i * 65536 + 2 * t + 2);
      } else {
        __threadfence_block();
        __syncwarp();
        if (lane == 0) prog[warp] = i * 65536 + 2 * t + 2;
      }
    }
  }
  if constexpr (CL > 1) {
    __threadfence();
    cooperative_groups::this_cluster().sync();
  } else {
    __syncthreads();
  }
  if (rank == 0 && threadIdx.x == 0 && !skip) diag[S - 1] = ld_band<CL>(B + (size_t)(S - 1) * SB_LD);
}

template <int NW>
constexpr size_t sym_chase_realr_smem() {
  return NW * sizeof(SymChaseSmemRR) + 64;
}

}  // namespace hx
