// Stage 2 of the banded path: band (lower, width BW) -> real symmetric tridiagonal by Householder
// bulge chasing, pipelined over sweeps.
//
// Sweep i annihilates column i below the subdiagonal and chases the bulge down the band in tasks
// t = 0, 1, ...; task t works on D_t = A[s:s+len, s:s+len] (s = i+1+t*BW) and the block below it
// B_t = A[s+len : s+len+lb, s:s+len]:
//     D <- H D H,  B <- B H,  H' = reflector(B[:,0]),  B <- H' B,  pass H' to task t+1.
// Task t of sweep i touches columns [s-1, s+BW); task t of sweep i+1 only columns left of task t+2
// of sweep i, so sweep i+1 may run task t as soon as sweep i has completed task t+1.  One warp owns
// the sweeps i = w (mod NW) of its CTA's matrix and waits on a per-warp progress counter in shared
// memory (no CTA-wide barriers).  Inside a warp lane r owns row r of D in registers (full Hermitian
// row), B lives in the warp's shared-memory tile (copied in with cp.async), vectors are broadcast
// from shared memory.
#pragma once
#include "hx_dense.cuh"

namespace hx {

// 16-byte global -> shared asynchronous copy (LDGSTS): all of a tile's loads are in flight at once.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int BWc>
struct ChaseWarpSmem {
  double2 B[BWc][BWc + 1];
  double2 v[BWc], w[BWc], vp[BWc], z[BWc];
};

__device__ __forceinline__ double2 cfma_acc(double2 acc, double2 a, double2 b) {  // acc + a*b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cfma_conj_acc(double2 acc, double2 a, double2 b) {  // acc + conj(a)*b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}

template <int NW, int BWc>
__global__ void __launch_bounds__(NW * 32) bulge_chase_pipe_kernel(double2* ws, size_t stride, size_t a_off,
                                                                    size_t dg_off, int N, const int* dims) {
  extern __shared__ __align__(16) unsigned char chase_smem[];
  ChaseWarpSmem<BWc>* all = reinterpret_cast<ChaseWarpSmem<BWc>*>(chase_smem);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);  // per warp: sweep*65536 + tasks done
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ChaseWarpSmem<BWc>& S = all[warp];
  double2* base = ws + (size_t)blockIdx.x * stride;
  double2* A = base + a_off;
  double* diag = reinterpret_cast<double*>(base + dg_off);
  double* e2 = diag + N;
  const int lda = N;
  const int d = dims ? dims[blockIdx.x] : N;
  if (lane == 0) prog[warp] = -1;
  __syncthreads();
  if (d <= 0) return;
  const int nsweeps = d - 1;  // sweeps i = 0 .. d-2
  for (int i = warp; i < nsweeps; i += NW) {
    const int tasks = (d - 1 - i + BWc - 1) / BWc;
    const int prev_tasks = i > 0 ? (d - i + BWc - 1) / BWc : 0;
    const int pw = (i - 1 + NW) % NW;
    double tau = 0.0;
    for (int t = 0; t < tasks; ++t) {
      // ---- wait until sweep i-1 has completed task t+1 (or all of its tasks)
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 2, prev_tasks);
        if (lane == 0)
          while (prog[pw] < need) {
          }
        __syncwarp();
        __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, d - s);
      const int lb = max(0, min(BWc, d - s - len));
      if (t == 0) {
        // reflector from column i, rows s .. s+len-1
        double2 x = make_double2(0.0, 0.0);
        if (lane < len) x = A[s + lane + (size_t)i * lda];
        const double sig2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 alpha = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const Reflector h = make_reflector(alpha, sig2);
        tau = h.tau;
        if (lane < len) {
          S.v[lane] = lane == 0 ? make_double2(1.0, 0.0) : cmul(x, h.scale);
          if (tau != 0.0) {
            double2 outv = make_double2(0.0, 0.0);
            if (lane == 0) {
              const double sg = sqrt(sig2), aa = hypot(alpha.x, alpha.y);
              const double2 ph = aa > 0.0 ? make_double2(alpha.x / aa, alpha.y / aa) : make_double2(1.0, 0.0);
              outv = make_double2(-ph.x * sg, -ph.y * sg);
            }
            A[s + lane + (size_t)i * lda] = outv;
          }
        }
        if (lane == 0) {
          diag[i] = A[i + (size_t)i * lda].x;
          e2[i] = sig2;
        }
        __syncwarp();
      }
      // ---- stage D (lower triangle) through the B tile, build full rows in registers
#pragma unroll
      for (int c = 0; c < BWc; ++c)
        if (c < len && lane >= c && lane < len) cp_async16(&S.B[lane][c], A + s + lane + (size_t)(s + c) * lda);
      cp_async_wait_all();
      __syncwarp();
      double2 dr[BWc];
#pragma unroll
      for (int c = 0; c < BWc; ++c) {
        double2 z = make_double2(0.0, 0.0);
        if (lane < len && c < len) {
          if (c <= lane) {
            z = S.B[lane][c];
          } else {
            const double2 u = S.B[c][lane];
            z = make_double2(u.x, -u.y);
          }
        }
        dr[c] = z;
      }
      __syncwarp();
      // ---- B tile (completes while p = D v is computed from registers)
#pragma unroll
      for (int c = 0; c < BWc; ++c)
        if (c < len && lane < lb) cp_async16(&S.B[lane][c], A + s + len + lane + (size_t)(s + c) * lda);
      // ---- p = D v (4 independent partial sums); cval = v^H p ; w = tau p - 1/2 tau^2 cval v
      double2 pp[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                       make_double2(0.0, 0.0)};
#pragma unroll
      for (int c = 0; c < BWc; ++c)
        if (c < len) pp[c & 3] = cfma_acc(pp[c & 3], dr[c], S.v[c]);
      const double2 p = make_double2((pp[0].x + pp[1].x) + (pp[2].x + pp[3].x), (pp[0].y + pp[1].y) + (pp[2].y + pp[3].y));
      const double2 vr = lane < len ? S.v[lane] : make_double2(0.0, 0.0);
      const double cval = warp_sum(lane < len ? vr.x * p.x + vr.y * p.y : 0.0);
      const double hc = 0.5 * tau * tau * cval;
      const double2 wr = make_double2(tau * p.x - hc * vr.x, tau * p.y - hc * vr.y);
      if (lane < len) S.w[lane] = wr;
      __syncwarp();
      // ---- D -= v w^H + w v^H ; write the lower triangle back
#pragma unroll
      for (int c = 0; c < BWc; ++c) {
        if (c < len) {
          const double2 vc = S.v[c], wc = S.w[c];
          dr[c].x -= vr.x * wc.x + vr.y * wc.y + wr.x * vc.x + wr.y * vc.y;
          dr[c].y -= (vr.y * wc.x - vr.x * wc.y) + (wr.y * vc.x - wr.x * vc.y);
          if (lane < len && c <= lane) {
            double2 z = dr[c];
            if (c == lane) z.y = 0.0;
            A[s + lane + (size_t)(s + c) * lda] = z;
          }
        }
      }
      cp_async_wait_all();
      __syncwarp();
      if (lb > 0) {
        // ---- B <- B H : q = B v ; B -= tau q v^H  (lane = row)
        double2 qq[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                         make_double2(0.0, 0.0)};
        double2 brow[BWc];
#pragma unroll
        for (int c = 0; c < BWc; ++c) {
          brow[c] = (c < len && lane < lb) ? S.B[lane][c] : make_double2(0.0, 0.0);
          if (c < len) qq[c & 3] = cfma_acc(qq[c & 3], brow[c], S.v[c]);
        }
        const double2 q = make_double2(tau * ((qq[0].x + qq[1].x) + (qq[2].x + qq[3].x)),
                                       tau * ((qq[0].y + qq[1].y) + (qq[2].y + qq[3].y)));
#pragma unroll
        for (int c = 0; c < BWc; ++c) {
          if (c < len) {
            const double2 vc = S.v[c];
            brow[c].x -= q.x * vc.x + q.y * vc.y;
            brow[c].y -= q.y * vc.x - q.x * vc.y;
          }
        }
        // ---- H' from B[:, 0] (lane r holds B[r][0] in brow[0])
        const double2 x = lane < lb ? brow[0] : make_double2(0.0, 0.0);
        const double sg2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const Reflector hp = make_reflector(al, sg2);
        const double2 vpr = lane == 0 ? make_double2(1.0, 0.0) : cmul(x, hp.scale);
        if (lane < lb) {
          S.vp[lane] = vpr;
#pragma unroll
          for (int c = 0; c < BWc; ++c)
            if (c < len) S.B[lane][c] = brow[c];
        }
        __syncwarp();
        // ---- z_c = v'^H B[:, c] (lane = column)
        if (lane < len && lane > 0) {
          double2 zz[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                           make_double2(0.0, 0.0)};
#pragma unroll
          for (int r = 0; r < BWc; ++r)
            if (r < lb) zz[r & 3] = cfma_conj_acc(zz[r & 3], S.vp[r], S.B[r][lane]);
          S.z[lane] = make_double2(hp.tau * ((zz[0].x + zz[1].x) + (zz[2].x + zz[3].x)),
                                   hp.tau * ((zz[0].y + zz[1].y) + (zz[2].y + zz[3].y)));
        }
        __syncwarp();
        // ---- B <- H' B (lane = row), column 0 -> beta' e1 ; write B back (coalesced per column)
        if (lane < lb) {
#pragma unroll
          for (int c = 1; c < BWc; ++c) {
            if (c < len && hp.tau != 0.0) {
              const double2 zc = S.z[c];
              brow[c].x -= vpr.x * zc.x - vpr.y * zc.y;
              brow[c].y -= vpr.x * zc.y + vpr.y * zc.x;
            }
          }
          if (hp.tau != 0.0) {
            double2 b0 = make_double2(0.0, 0.0);
            if (lane == 0) {
              const double sg = sqrt(sg2), aa = hypot(al.x, al.y);
              const double2 ph = aa > 0.0 ? make_double2(al.x / aa, al.y / aa) : make_double2(1.0, 0.0);
              b0 = make_double2(-ph.x * sg, -ph.y * sg);
            }
            brow[0] = b0;
          }
#pragma unroll
          for (int c = 0; c < BWc; ++c)
            if (c < len) A[s + len + lane + (size_t)(s + c) * lda] = brow[c];
        }
        __syncwarp();
        // carry H' to the next task of this sweep
        if (lane < lb) S.v[lane] = vpr;
        tau = hp.tau;
      }
      // ---- publish progress (release the global writes of this task to the other warps)
      __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[warp] = i * 65536 + t + 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) diag[d - 1] = A[d - 1 + (size_t)(d - 1) * lda].x;
}

template <int NW, int BWc>
constexpr size_t chase_smem_bytes() {
  return NW * sizeof(ChaseWarpSmem<BWc>) + 64;
}

}  // namespace hx
