// Stage 2 of the bipartite banded tier: upper band (width BWc) -> upper bidiagonal by bulge chasing,
// emitting the Golub-Kahan tridiagonal (zero diagonal, e2 = |alpha_0|^2, |gamma_0|^2, |alpha_1|^2, ...).
//
// Sweep i annihilates row i right of the superdiagonal and chases the bulge; task t (block start
// s = i + 1 + t*BWc, width len, next width lb):
//   right reflector G (from row s-BWc, built by task t-1; for t = 0 from row i) on columns [s, s+len):
//       applied to the rows above the block that intersect those columns ("top rows") and to the block
//       X = C[s:s+len, s:s+len];
//   left reflector H from X[:, 0] (gives alpha_s), applied to rows [s, s+len) over X and the block to its
//       right Y = C[s:s+len, s+len:s+len+lb];
//   next right reflector from Y[0, :] (row s, gives gamma_s), carried to task t+1.
// Sweep i may run task t once sweep i-1 has completed task t+2 (regions are disjoint beyond that), so
// one warp owns the sweeps i = w (mod NW) and waits on a per-warp progress counter (no CTA barriers).
#pragma once
#include "hx_dense.cuh"

namespace hx {

template <int BWc>
struct BdChaseSmem {
  double2 X[BWc][BWc + 1];
  double2 Y[BWc][BWc + 1];
  double2 ug[BWc];  // current right reflector vector (ug[0] = 1)
  double2 vh[BWc];  // current left reflector vector (vh[0] = 1)
};

__device__ __forceinline__ void bd_cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void bd_cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int NW, int BWc>
__global__ void __launch_bounds__(NW * 32) bd_chase_kernel(double2* ws, size_t stride, size_t c_off, size_t tgk_off,
                                                            int S, const int* dims) {
  extern __shared__ __align__(16) unsigned char bd_smem[];
  BdChaseSmem<BWc>* all = reinterpret_cast<BdChaseSmem<BWc>*>(bd_smem);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  BdChaseSmem<BWc>& W = all[warp];
  double2* base = ws + (size_t)blockIdx.x * stride;
  double2* C = base + c_off;
  double* diag = reinterpret_cast<double*>(base + tgk_off);
  double* e2 = diag + 2 * S;
  const int ld = S;
  for (int q = threadIdx.x; q < 2 * S; q += blockDim.x) {
    diag[q] = 0.0;
    e2[q] = 0.0;
  }
  if (lane == 0) prog[warp] = -1;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double2 a0 = C[0];
    e2[0] = a0.x * a0.x + a0.y * a0.y;  // alpha_0: final after stage 1
  }
  if (dims && dims[blockIdx.x] == 0) return;
  const int nsweeps = S - 1;
  for (int i = warp; i < nsweeps; i += NW) {
    const int tasks = (S - 1 - i + BWc - 1) / BWc;
    const int prev_tasks = i > 0 ? (S - i + BWc - 1) / BWc : 0;
    const int pw = (i - 1 + NW) % NW;
    double taug = 0.0;
    for (int t = 0; t < tasks; ++t) {
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 3, prev_tasks);
        if (lane == 0)
          while (prog[pw] < need) {
          }
        __syncwarp();
        __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, S - s);
      const int lb = max(0, min(BWc, S - s - len));
      // ---- X and Y tiles (asynchronous; Y is not needed until the left reflector)
      for (int cc = 0; cc < len; ++cc)
        if (lane < len) bd_cp_async16(&W.X[lane][cc], C + (size_t)(s + cc) * ld + s + lane);
      for (int cc = 0; cc < lb; ++cc)
        if (lane < len) bd_cp_async16(&W.Y[lane][cc], C + (size_t)(s + len + cc) * ld + s + lane);
      if (t == 0) {
        // right reflector from row i, columns [s, s+len): row i -> (gamma_i, 0, ...)
        double2 x = make_double2(0.0, 0.0);
        if (lane < len) {
          const double2 z = C[(size_t)(s + lane) * ld + i];
          x = make_double2(z.x, -z.y);
        }
        const double sig2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const Reflector h = make_reflector(al, sig2);
        taug = h.tau;
        if (lane < len) {
          W.ug[lane] = lane == 0 ? make_double2(1.0, 0.0) : cmul(x, h.scale);
          if (taug != 0.0) {
            double2 o = make_double2(0.0, 0.0);
            if (lane == 0) {
              const double sg = sqrt(sig2), aa = hypot(al.x, al.y);
              const double2 ph = aa > 0.0 ? make_double2(al.x / aa, al.y / aa) : make_double2(1.0, 0.0);
              o = make_double2(-ph.x * sg, ph.y * sg);  // conj(beta)
            }
            C[(size_t)(s + lane) * ld + i] = o;
          }
        }
        if (lane == 0) e2[2 * i + 1] = sig2;
        __syncwarp();
      } else if (taug != 0.0) {
        // top rows [s-BWc+1, s): apply G from the right (lane = row), straight from/to global memory
        const int ntop = BWc - 1;
        if (lane < ntop) {
          const int r = s - BWc + 1 + lane;
          double2 row[BWc];
          double2 w = make_double2(0.0, 0.0);
#pragma unroll
          for (int cc = 0; cc < BWc; ++cc) {
            row[cc] = cc < len ? C[(size_t)(s + cc) * ld + r] : make_double2(0.0, 0.0);
            if (cc < len) {
              const double2 u = W.ug[cc];
              w.x += row[cc].x * u.x - row[cc].y * u.y;
              w.y += row[cc].x * u.y + row[cc].y * u.x;
            }
          }
          w = make_double2(taug * w.x, taug * w.y);
#pragma unroll
          for (int cc = 0; cc < BWc; ++cc) {
            if (cc < len) {
              const double2 u = W.ug[cc];
              double2 z = row[cc];
              z.x -= w.x * u.x + w.y * u.y;
              z.y -= w.y * u.x - w.x * u.y;
              C[(size_t)(s + cc) * ld + r] = z;
            }
          }
        }
      }
      bd_cp_async_wait_all();
      __syncwarp();
      // ---- G on X (lane = row)
      if (taug != 0.0 && lane < len) {
        double2 w = make_double2(0.0, 0.0);
        for (int cc = 0; cc < len; ++cc) {
          const double2 a = W.X[lane][cc], u = W.ug[cc];
          w.x += a.x * u.x - a.y * u.y;
          w.y += a.x * u.y + a.y * u.x;
        }
        w = make_double2(taug * w.x, taug * w.y);
        for (int cc = 0; cc < len; ++cc) {
          const double2 u = W.ug[cc];
          double2 z = W.X[lane][cc];
          z.x -= w.x * u.x + w.y * u.y;
          z.y -= w.y * u.x - w.x * u.y;
          W.X[lane][cc] = z;
        }
      }
      __syncwarp();
      // ---- H from X[:, 0] (alpha_s)
      const double2 xh = lane < len ? W.X[lane][0] : make_double2(0.0, 0.0);
      const double sh2 = warp_sum(xh.x * xh.x + xh.y * xh.y);
      const double2 ah = make_double2(__shfl_sync(0xffffffffu, xh.x, 0), __shfl_sync(0xffffffffu, xh.y, 0));
      const Reflector hh = make_reflector(ah, sh2);
      if (t == 0 && lane == 0) e2[2 * s] = sh2;
      if (lane < len) W.vh[lane] = lane == 0 ? make_double2(1.0, 0.0) : cmul(xh, hh.scale);
      __syncwarp();
      if (hh.tau != 0.0) {
        if (lane < len) {
          double2 b0 = make_double2(0.0, 0.0);
          if (lane == 0) {
            const double sg = sqrt(sh2), aa = hypot(ah.x, ah.y);
            const double2 ph = aa > 0.0 ? make_double2(ah.x / aa, ah.y / aa) : make_double2(1.0, 0.0);
            b0 = make_double2(-ph.x * sg, -ph.y * sg);
          }
          W.X[lane][0] = b0;
        }
        // left application (lane = column): X columns 1..len-1, then Y columns 0..lb-1
        if (lane >= 1 && lane < len) {
          double2 z = make_double2(0.0, 0.0);
          for (int r = 0; r < len; ++r) {
            const double2 v = W.vh[r], a = W.X[r][lane];
            z.x += v.x * a.x + v.y * a.y;
            z.y += v.x * a.y - v.y * a.x;
          }
          z = make_double2(hh.tau * z.x, hh.tau * z.y);
          for (int r = 0; r < len; ++r) {
            const double2 v = W.vh[r];
            double2 a = W.X[r][lane];
            a.x -= v.x * z.x - v.y * z.y;
            a.y -= v.x * z.y + v.y * z.x;
            W.X[r][lane] = a;
          }
        }
        if (lane < lb) {
          double2 z = make_double2(0.0, 0.0);
          for (int r = 0; r < len; ++r) {
            const double2 v = W.vh[r], a = W.Y[r][lane];
            z.x += v.x * a.x + v.y * a.y;
            z.y += v.x * a.y - v.y * a.x;
          }
          z = make_double2(hh.tau * z.x, hh.tau * z.y);
          for (int r = 0; r < len; ++r) {
            const double2 v = W.vh[r];
            double2 a = W.Y[r][lane];
            a.x -= v.x * z.x - v.y * z.y;
            a.y -= v.x * z.y + v.y * z.x;
            W.Y[r][lane] = a;
          }
        }
      }
      __syncwarp();
      // ---- next right reflector from Y[0, :] (row s)
      double next_tau = 0.0;
      if (lb > 0) {
        double2 x = make_double2(0.0, 0.0);
        if (lane < lb) x = make_double2(W.Y[0][lane].x, -W.Y[0][lane].y);
        const double sg2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const Reflector hg = make_reflector(al, sg2);
        next_tau = hg.tau;
        __syncwarp();
        if (lane < lb) {
          W.ug[lane] = lane == 0 ? make_double2(1.0, 0.0) : cmul(x, hg.scale);
          if (next_tau != 0.0) {
            double2 o = make_double2(0.0, 0.0);
            if (lane == 0) {
              const double sg = sqrt(sg2), aa = hypot(al.x, al.y);
              const double2 ph = aa > 0.0 ? make_double2(al.x / aa, al.y / aa) : make_double2(1.0, 0.0);
              o = make_double2(-ph.x * sg, ph.y * sg);
            }
            W.Y[0][lane] = o;
          }
        }
      }
      __syncwarp();
      // ---- write X and Y back (lane = row, coalesced per column)
      if (lane < len) {
        for (int cc = 0; cc < len; ++cc) C[(size_t)(s + cc) * ld + s + lane] = W.X[lane][cc];
        for (int cc = 0; cc < lb; ++cc) C[(size_t)(s + len + cc) * ld + s + lane] = W.Y[lane][cc];
      }
      taug = next_tau;
      __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[warp] = i * 65536 + t + 1;
    }
  }
}

template <int NW, int BWc>
constexpr size_t bd_chase_smem() {
  return NW * sizeof(BdChaseSmem<BWc>) + 64;
}

}  // namespace hx
