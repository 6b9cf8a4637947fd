// Panel QR of stage 1 on a thread-block CLUSTER: an m x BW panel is split by rows over the CL CTAs of
// a cluster and held in their shared memory for the whole factorisation; the two reductions per column
// (column norm, dot products with the remaining columns) are combined across the cluster through
// distributed shared memory (fixed rank order -> deterministic).  Replaces up to 3 passes over an
// L2-resident panel per column with shared-memory sweeps + 2 cluster barriers.
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

template <int BWc>
struct PanelSlot {
  double2 norm_alpha[2];  // (sigma^2 partial, 0), alpha (owner of row j only)
  double2 dots[BWc];
};

// Recursive-halving reduce-scatter of 32 complex per-lane values: afterwards lane l holds the warp sum
// of index l (in a[0]).
__device__ __forceinline__ void warp_reduce_scatter32(double2 (&a)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const double2 send = up ? a[k] : a[k + s];
      const double2 keep = up ? a[k + s] : a[k];
      const double rx = __shfl_xor_sync(0xffffffffu, send.x, s);
      const double ry = __shfl_xor_sync(0xffffffffu, send.y, s);
      a[k] = make_double2(keep.x + rx, keep.y + ry);
    }
  }
}

// grid = (CL, batch), cluster = (CL, 1, 1), 256 threads; dynamic smem = panel_cluster_smem(R).
template <int CL, int BWc>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(256, 2)
    panel_qr_cluster_kernel(double2* ws, PanelArgs a, int R) {
  extern __shared__ __align__(16) unsigned char psm[];
  cgx::cluster_group cluster = cgx::this_cluster();
  const int rank = (int)cluster.block_rank();
  double2* Ps = reinterpret_cast<double2*>(psm);  // Ps[c * (R+1) + i]  (column-major slice)
  const int ldp = R + 1;
  PanelSlot<BWc>* slot = reinterpret_cast<PanelSlot<BWc>*>(Ps + (size_t)BWc * ldp);
  __shared__ double wred[8];
  __shared__ double2 wdots[8][BWc];
  __shared__ double2 s[BWc];
  __shared__ double2 Ts[BWc][BWc + 1];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* base = ws + (size_t)blockIdx.y * a.stride;
  double2* M = base + a.m_off;
  double2* V = base + a.v_off;
  const int m = a.m;
  const int r0 = rank * R;
  const int rows = max(0, min(R, m - r0));
  const bool conj_in = a.mode == 1;

  for (int p = tid; p < BWc * (BWc + 1); p += 256) (&Ts[0][0])[p] = make_double2(0.0, 0.0);
  if (!conj_in) {
    for (int c = 0; c < BWc; ++c)
      for (int i = tid; i < rows; i += 256) Ps[c * ldp + i] = *panel_elem(M, a, r0 + i, c);
  } else {
    // row panel: consecutive threads walk j (contiguous in memory for a fixed panel row i)
    for (int p = tid; p < rows * BWc; p += 256) {
      const int i = p / BWc, c = p % BWc;
      const double2 z = *panel_elem(M, a, r0 + i, c);
      Ps[c * ldp + i] = make_double2(z.x, -z.y);
    }
  }
  __syncthreads();

  for (int j = 0; j < BWc; ++j) {
    if (j >= m) break;  // uniform over the cluster
    // ---- (1) column norm partial over my rows >= j; alpha from the owner of row j
    double part = 0.0;
    for (int i = tid; i < rows; i += 256) {
      if (r0 + i < j) continue;
      const double2 x = Ps[j * ldp + i];
      part += x.x * x.x + x.y * x.y;
    }
    part = warp_sum(part);
    if (lane == 0) wred[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += wred[w];
      slot->norm_alpha[0] = make_double2(t, 0.0);
      if (j >= r0 && j < r0 + rows) slot->norm_alpha[1] = Ps[j * ldp + (j - r0)];
    }
    cluster.sync();
    double sig2 = 0.0;
    for (int q = 0; q < CL; ++q) sig2 += cluster.map_shared_rank(slot, q)->norm_alpha[0].x;
    const int owner = j / R;
    const double2 alpha = cluster.map_shared_rank(slot, owner)->norm_alpha[1];
    const Reflector h = make_reflector(alpha, sig2);
    const double tau = h.tau;
    // ---- (2) v in place (rows > j), dot products of v with every other column (V for c < j)
    double2 acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = make_double2(0.0, 0.0);
    for (int i = tid; i < rows; i += 256) {
      const int gi = r0 + i;
      if (gi < j) continue;
      double2 vi;
      if (gi == j) {
        vi = make_double2(1.0, 0.0);
      } else {
        vi = tau == 0.0 ? make_double2(0.0, 0.0) : cmul(Ps[j * ldp + i], h.scale);
        Ps[j * ldp + i] = vi;
      }
      if (tau == 0.0) continue;
#pragma unroll
      for (int c = 0; c < BWc; ++c) {
        if (c == j) continue;
        double2 x;
        if (c > j) x = Ps[c * ldp + i];
        else x = gi > c ? Ps[c * ldp + i] : (gi == c ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0));
        acc[c].x += vi.x * x.x + vi.y * x.y;
        acc[c].y += vi.x * x.y - vi.y * x.x;
      }
    }
    warp_reduce_scatter32(acc);
    if (lane < BWc) wdots[warp][lane] = acc[0];
    __syncthreads();
    if (tid < BWc) {
      double2 t = make_double2(0.0, 0.0);
      for (int w = 0; w < 8; ++w) t = make_double2(t.x + wdots[w][tid].x, t.y + wdots[w][tid].y);
      slot->dots[tid] = t;
    }
    cluster.sync();
    if (tid < BWc) {
      double2 t = make_double2(0.0, 0.0);
      for (int q = 0; q < CL; ++q) {
        const double2 u = cluster.map_shared_rank(slot, q)->dots[tid];
        t = make_double2(t.x + u.x, t.y + u.y);
      }
      s[tid] = t;
    }
    __syncthreads();
    // ---- (3) update my rows of the remaining columns; R diagonal beta; T column j
    if (tau != 0.0) {
      for (int i = tid; i < rows; i += 256) {
        const int gi = r0 + i;
        if (gi < j) continue;
        const double2 vi = gi == j ? make_double2(1.0, 0.0) : Ps[j * ldp + i];
        const double2 tv = make_double2(tau * vi.x, tau * vi.y);
        for (int c = j + 1; c < BWc; ++c) {
          const double2 sc = s[c];
          double2 x = Ps[c * ldp + i];
          x.x -= tv.x * sc.x - tv.y * sc.y;
          x.y -= tv.x * sc.y + tv.y * sc.x;
          Ps[c * ldp + i] = x;
        }
      }
      if (tid == 0 && j >= r0 && j < r0 + rows) {
        const double sg = sqrt(sig2), aa = hypot(alpha.x, alpha.y);
        const double2 ph = aa > 0.0 ? make_double2(alpha.x / aa, alpha.y / aa) : make_double2(1.0, 0.0);
        Ps[j * ldp + (j - r0)] = make_double2(-ph.x * sg, -ph.y * sg);
      }
    }
    if (tid < j) {
      double2 t = make_double2(0.0, 0.0);
      for (int l = tid; l < j; ++l)
        t = make_double2(t.x + (Ts[tid][l].x * s[l].x + Ts[tid][l].y * s[l].y),
                         t.y + (Ts[tid][l].y * s[l].x - Ts[tid][l].x * s[l].y));
      Ts[tid][j] = make_double2(-tau * t.x, -tau * t.y);
    }
    if (tid == 0) Ts[j][j] = make_double2(tau, 0.0);
    __syncthreads();
  }
  // ---- write back: R (upper part) into the matrix, zeros below; explicit V; T from rank 0
  for (int p = tid; p < rows * BWc; p += 256) {
    int i, c;
    if (!conj_in) {
      c = p / rows;
      i = p - c * rows;
    } else {
      i = p / BWc;
      c = p % BWc;
    }
    const int gi = r0 + i;
    const double2 x = Ps[c * ldp + i];
    const double2 rv = gi <= c ? x : make_double2(0.0, 0.0);
    *panel_elem(M, a, gi, c) = conj_in ? make_double2(rv.x, -rv.y) : rv;
    double2 vv;
    if (c >= m) vv = make_double2(0.0, 0.0);
    else if (gi < c) vv = make_double2(0.0, 0.0);
    else if (gi == c) vv = make_double2(1.0, 0.0);
    else vv = x;
    V[gi + (size_t)c * a.ldv] = vv;
  }
  if (rank == 0) {
    double2* T = base + a.t_off;
    for (int p = tid; p < BWc * BWc; p += 256) T[(p % BWc) + (p / BWc) * BWc] = Ts[p % BWc][p / BWc];
  }
  cluster.sync();  // keep every CTA's shared memory alive until remote reads are done
}

template <int BWc>
constexpr size_t panel_cluster_smem(int R) {
  return (size_t)BWc * (R + 1) * sizeof(double2) + sizeof(PanelSlot<BWc>) + 64;
}

}  // namespace hx
