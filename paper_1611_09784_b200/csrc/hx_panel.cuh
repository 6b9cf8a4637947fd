// Panel QR of stage 1 (m x 32 column panel, or conj-transposed row panel, of a matrix slab in HBM):
// Householder vectors V (explicit, unit diagonal), R and the block-reflector factor T (zlarft).
//
// The panel is addressed through PanelArgs so the same kernel serves
//   mode 0  P[i][j] = M[r0 + i][c0 + j]           (column panel; R written back, zeros below)
//   mode 1  P[i][j] = conj(M[r0 + j][c0 + i])     (row panel of the bidiagonal reduction: LQ of the row
//                                                  block; R^H written back, zeros right of it)
// with M column-major (leading dimension ld) inside each matrix slab of the batch.
#pragma once
#include <cooperative_groups.h>

#include "hx_dense.cuh"

namespace hx {

namespace cgx = cooperative_groups;

struct PanelArgs {
  size_t stride;  // per-matrix slab (double2 units)
  size_t m_off;   // matrix offset inside the slab
  int ld;         // leading dimension of the matrix
  int r0, c0;     // panel origin (see mode)
  int m;          // panel rows
  int mode;       // 0: column panel, 1: conj-transposed row panel
  size_t v_off;   // explicit V (m x BW, leading dimension ldv)
  int ldv;
  size_t t_off;   // T (BW x BW, column-major)
};

__device__ __forceinline__ double2* panel_elem(double2* M, const PanelArgs& a, int i, int j) {
  return a.mode == 0 ? M + (size_t)(a.c0 + j) * a.ld + a.r0 + i : M + (size_t)(a.c0 + i) * a.ld + a.r0 + j;
}

// Register-resident panel QR.  NT = 32*GR threads = 32 columns x GR row groups: thread (c, g) owns
// column c and the local rows g, g+GR, ..., g+(RPT-1)GR of it IN REGISTERS (GR*RPT rows per CTA; the
// columns of a warp are 32/GR consecutive ones, lane = (c % (32/GR)) * GR + g).  Per column j only the
// Householder vector goes through shared memory (scaled, zero above row j, 1 at row j, so every dot
// product and update is a uniform loop without row predicates); the 32 dot products v^H x_c are reduced
// over the GR lanes of each column group with xor-shuffles, so a column costs ONE CTA barrier.  Taller
// panels split their rows over a thread-block cluster of CL CTAs: the column norm (+ alpha) and the 32
// dot products are combined across the cluster through DSMEM in fixed rank order (deterministic) - two
// cluster barriers per column.  T (zlarft, forward/columnwise) is built one column behind the
// factorisation by all threads (GR-way split inner products).

struct PanelSlots {
  double sig2;
  double2 alpha;
  double2 dots[32];
};

// Shared-memory load the compiler may not merge with an earlier load of the same address (keeps the
// update loop from pinning the v values of the dot-product loop in registers).
__device__ __forceinline__ double2 lds_fresh(const double2* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

template <int RPT>
__device__ __forceinline__ double2 pick_row(const double2 (&x)[RPT], int r) {
  double2 out = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < RPT; ++k)
    if (k == r) out = x[k];
  return out;
}

template <int GR>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = 1; o < GR; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// T[l][jt] = -tau_jt sum_{l'=l}^{jt-1} T[l][l'] w[l'] (zlarft forward/columnwise), T[jt][jt] = tau_jt.
template <int GR>
__device__ __forceinline__ void build_t_column(double2 (*Ts)[33], const double2* w, const double* tauS, int jt) {
  const int tid = threadIdx.x, l = tid / GR, part = tid % GR;
  double2 t = make_double2(0.0, 0.0);
  if (l < jt)
#pragma unroll 1
    for (int lp = l + part; lp < jt; lp += GR) {
      const double2 tv = Ts[l][lp], wv = w[lp];
      t.x += tv.x * wv.x - tv.y * wv.y;
      t.y += tv.x * wv.y + tv.y * wv.x;
    }
  t.x = group_sum<GR>(t.x);
  t.y = group_sum<GR>(t.y);
  if (jt >= 0) {
    const double tj = tauS[jt];
    if (part == 0 && l < jt) Ts[l][jt] = make_double2(-tj * t.x, -tj * t.y);
    if (tid == 0) Ts[jt][jt] = make_double2(tj, 0.0);
  }
}

// grid = (CL, batch), cluster = (CL, 1, 1), 32*GR threads, R = rows per CTA (<= GR * RPT).
template <int CL, int GR, int RPT>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(32 * GR, GR == 8 && RPT <= 8 ? 2 : 1)
    panel_qr_reg_kernel(double2* ws, PanelArgs a, int R) {
  constexpr int BWc = 32, NT = 32 * GR, CPW = 32 / GR;  // columns per warp
  __shared__ __align__(16) double2 vbuf[2][GR * RPT];
  __shared__ double2 wbuf[2][BWc];
  __shared__ double2 Ts[BWc][BWc + 1];
  __shared__ double tauS[BWc];
  __shared__ PanelSlots slot;

  const int tid = threadIdx.x, lane = tid & 31;
  const int c = (tid >> 5) * CPW + lane / GR, g = lane % GR;
  int rank = 0;
  if constexpr (CL > 1) rank = (int)cgx::this_cluster().block_rank();
  double2* base = ws + (size_t)blockIdx.y * a.stride;
  double2* M = base + a.m_off;
  double2* V = base + a.v_off;
  const int m = a.m;
  const int r0 = rank * R;
  const int rows = max(0, min(R, m - r0));
  const bool conj_in = a.mode == 1;

  for (int p = tid; p < BWc * (BWc + 1); p += NT) (&Ts[0][0])[p] = make_double2(0.0, 0.0);
  double2 x[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int li = g + GR * r;
    x[r] = make_double2(0.0, 0.0);
    if (li < rows) {
      const double2 z = *panel_elem(M, a, r0 + li, c);
      x[r] = conj_in ? make_double2(z.x, -z.y) : z;
    }
  }

  const int jmax = min(BWc, m);
#pragma unroll 1
  for (int j = 0; j < jmax; ++j) {
    const int buf = j & 1;
    const int jl = j - r0;                      // local index of row j (may be outside [0, rows))
    const bool own_row = jl >= 0 && jl < rows;  // uniform
    // ---- norm (rows >= j) and alpha of column j: computed by its warp, combined with warp-wide
    //      shuffles outside the (warp-uniform) branch
    double sig2 = 0.0;
    double2 alpha = make_double2(0.0, 0.0);
    if ((tid >> 5) == j / CPW) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (g + GR * r >= jl) sig2 = fma(x[r].x, x[r].x, fma(x[r].y, x[r].y, sig2));
      alpha = pick_row(x, jl / GR);
    }
    sig2 = group_sum<GR>(sig2);
    {
      const int src = (lane & ~(GR - 1)) | (jl & (GR - 1));
      alpha.x = __shfl_sync(0xffffffffu, alpha.x, src);
      alpha.y = __shfl_sync(0xffffffffu, alpha.y, src);
    }
    if (!own_row) alpha = make_double2(0.0, 0.0);
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
    // ---- owners of column j: reflector, publish v, keep (beta, V) in registers
    if (c == j) {
      const QuickReflector h = quick_reflector(alpha, sig2);
      const double2 beta = h.beta;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int li = g + GR * r;
        double2 v;
        if (li < jl) {
          v = make_double2(0.0, 0.0);
        } else if (li == jl) {
          v = make_double2(1.0, 0.0);
          x[r] = h.tau == 0.0 ? x[r] : beta;
        } else {
          v = cmul(x[r], h.scale);
          x[r] = v;
        }
        vbuf[buf][li] = v;
      }
      if (g == 0) tauS[j] = h.tau;
    }
    __syncthreads();
    const double tau = tauS[j];
    // ---- all: s_c = v^H x_c (c < j: conj -> w for T; c > j: update).  No branches around the
    //      shuffles (tau == 0 just skips the update).
    double2 s;
    {
      double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < RPT; r += 2) {
        const double2 v = vbuf[buf][g + GR * r];
        s0.x = fma(v.x, x[r].x, fma(v.y, x[r].y, s0.x));
        s0.y = fma(v.x, x[r].y, fma(-v.y, x[r].x, s0.y));
        if (r + 1 < RPT) {
          const double2 u = vbuf[buf][g + GR * (r + 1)];
          s1.x = fma(u.x, x[r + 1].x, fma(u.y, x[r + 1].y, s1.x));
          s1.y = fma(u.x, x[r + 1].y, fma(-u.y, x[r + 1].x, s1.y));
        }
      }
      s = make_double2(group_sum<GR>(s0.x + s1.x), group_sum<GR>(s0.y + s1.y));
    }
    if constexpr (CL > 1) {
      cgx::cluster_group cluster = cgx::this_cluster();
      if (g == 0) slot.dots[c] = s;
      cluster.sync();
      s = make_double2(0.0, 0.0);
      for (int q = 0; q < CL; ++q) {
        const double2 u = cluster.map_shared_rank(&slot, q)->dots[c];
        s.x += u.x;
        s.y += u.y;
      }
    }
    if (c > j && tau != 0.0) {
      const double2 q = make_double2(tau * s.x, tau * s.y);
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const double2 v = lds_fresh(&vbuf[buf][g + GR * r]);
        x[r].x = fma(-q.x, v.x, fma(q.y, v.y, x[r].x));
        x[r].y = fma(-q.x, v.y, fma(-q.y, v.x, x[r].y));
      }
    }
    if (g == 0 && c < j) wbuf[buf][c] = make_double2(s.x, -s.y);  // V_c^H v_j
    // ---- T column j-1 (one column behind; nothing at j = 0)
    build_t_column<GR>(Ts, wbuf[(j - 1) & 1], tauS, j - 1);
  }
  __syncthreads();
  build_t_column<GR>(Ts, wbuf[(jmax - 1) & 1], tauS, jmax - 1);
  // ---- write back: R (upper part) into the matrix, zeros below; explicit V (unit diagonal)
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int li = g + GR * r;
    if (li < rows) {
      const int gi = r0 + li;
      const double2 rv = gi <= c ? x[r] : make_double2(0.0, 0.0);
      *panel_elem(M, a, gi, c) = conj_in ? make_double2(rv.x, -rv.y) : rv;
      double2 vv;
      if (c >= jmax || gi < c) vv = make_double2(0.0, 0.0);
      else if (gi == c) vv = make_double2(1.0, 0.0);
      else vv = x[r];
      V[gi + (size_t)c * a.ldv] = vv;
    }
  }
  __syncthreads();
  if (rank == 0) {
    double2* T = base + a.t_off;
    for (int p = tid; p < BWc * BWc; p += NT) T[(p % BWc) + (p / BWc) * BWc] = Ts[p % BWc][p / BWc];
  }
  if constexpr (CL > 1) cgx::this_cluster().sync();  // keep shared memory alive for remote readers
}

}  // namespace hx
