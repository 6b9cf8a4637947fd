// Stage 2 of the bipartite banded tier: upper band (width BWc) -> upper bidiagonal by bulge chasing,
// emitting the Golub-Kahan tridiagonal (zero diagonal, e2 = |alpha_0|^2, |gamma_0|^2, |alpha_1|^2, ...).
//
// Sweep i annihilates row i right of the superdiagonal and chases the bulge; task t works on the block
// rows [s, s+len), s = i + 1 + t*BWc, over X = C[s:s+len, s:s+len] and Y = C[s:s+len, s+len:s+len+lb]:
//   X' = H X G       G = I - tau_g u u^H  (right reflector carried in from the previous task; for t = 0
//                                          built here from row i, which becomes (conj beta, 0, ...))
//                    H = I - tau_h v v^H  (left reflector from column 0 of X G, gives alpha_s)
//   Y' = H Y G'      G' from row 0 of H Y (gives gamma_s), carried to task t+1
// Both are applied as one fused rank-2 row update per tile: with y = X u, p = v^H X, w = v^H (tau_g y),
//   X'[r][c] = X[r][c] - tau_g y_r conj(u_c) - v_r * tau_h (p_c - w conj(u_c)),
// and with q = v^H Y, f = Y u' - tau_h v (q . u'),
//   Y'[r][c] = Y[r][c] - v_r * tau_h q_c - tau_g' f_r conj(u'_c),
// so each tile is read twice from shared memory (one row pass, one column pass), updated in registers
// (lane = row) and stored straight to HBM.  Applying G' to Y here (instead of to the "top rows" at the
// start of task t+1) removes every dependent global load from the chase except row i at t = 0.
// Task t of sweep i touches rows [s, s+32) x columns [s, s+64) only, so it may run once sweep i-1 has
// completed its tasks 0..t+1; one warp owns the sweeps i = w (mod NW) and waits on a per-warp progress
// counter in shared memory (no CTA barriers).
#pragma once
#include <cooperative_groups.h>

#include "hx_dense.cuh"

namespace hx {

// DUAL: X and Y tiles staged together (lowest latency per task); otherwise one tile buffer, Y loaded
// after the X update (half the shared memory per warp -> twice the warps per SM).
template <int BWc, bool DUAL>
struct BdChaseSmem {
  double2 X[BWc][BWc + 1];  // tiles, zero-padded to BWc x BWc
  double2 Y[DUAL ? BWc : 1][BWc + 1];
  double2 ug[BWc];  // current right reflector vector (ug[0] = 1, zero-padded)
  double2 vh[BWc];  // left reflector vector (vh[0] = 1, zero-padded)
  double2 cb[BWc];  // per-column update coefficients
};

// L1-cached copies when every sweep of a matrix runs on one SM; L2 (.cg) when the sweeps of a matrix are
// spread over a cluster (another SM's stores are not visible through this SM's L1).
template <bool L2ONLY>
__device__ __forceinline__ void bd_cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (L2ONLY) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void bd_cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ double2 cmul_cj(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 warp_csum(double2 v) { return make_double2(warp_sum(v.x), warp_sum(v.y)); }

#ifdef HX_CHASE_PROFILE
// Debug builds only: per-phase clock64() totals of the warps of block 0 (phase k in slot k).
__device__ unsigned long long hx_chase_prof[16];
#define HX_PROF_MARK(k)                                                      \
  do {                                                                       \
    if (blockIdx.x == 0 && lane == 0) {                                      \
      const long long now_ = clock64();                                      \
      atomicAdd(&hx_chase_prof[k], (unsigned long long)(now_ - prof_t0_));   \
      prof_t0_ = now_;                                                       \
    }                                                                        \
  } while (0)
#else
#define HX_PROF_MARK(k) \
  do {                  \
  } while (0)
#endif

// CL > 1: the sweeps of one matrix are dealt round-robin to the warps of a CL-CTA cluster (CL x NW sweeps
// in flight, CL SMs per matrix); progress counters are read across the cluster through DSMEM and the
// tiles go through L2.
template <int NW, int BWc, bool DUAL, int CL>
__global__ void __launch_bounds__(NW * 32, 1) bd_chase_kernel(double2* ws, size_t stride, size_t c_off,
                                                               size_t tgk_off, int S, const int* dims) {
  extern __shared__ __align__(16) unsigned char bd_smem[];
  BdChaseSmem<BWc, DUAL>* all = reinterpret_cast<BdChaseSmem<BWc, DUAL>*>(bd_smem);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  BdChaseSmem<BWc, DUAL>& W = all[warp];
  auto Yt = [&]() -> double2(*)[BWc + 1] { return DUAL ? W.Y : W.X; };
  constexpr bool L2ONLY = CL > 1;
  const int rank = CL > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int64_t mat = blockIdx.x / CL;
  constexpr int TW = CL * NW;  // sweeps in flight per matrix
  const int gw = rank * NW + warp;
  double2* base = ws + (size_t)mat * stride;
  double2* C = base + c_off;
  double* diag = reinterpret_cast<double*>(base + tgk_off);
  double* e2 = diag + 2 * S;
  const int ld = S;
  const double2 zero = make_double2(0.0, 0.0);
  if (rank == 0) {
    for (int q = threadIdx.x; q < 2 * S; q += blockDim.x) {
      diag[q] = 0.0;
      e2[q] = 0.0;
    }
  }
  if (lane == 0) prog[warp] = -1;
  if (CL > 1) cooperative_groups::this_cluster().sync();
  else __syncthreads();
  if (rank == 0 && threadIdx.x == 0) {
    const double2 a0 = C[0];
    e2[0] = a0.x * a0.x + a0.y * a0.y;  // alpha_0: final after stage 1
  }
  const bool skip = dims && dims[mat] == 0;  // uniform over the cluster
  const int nsweeps = skip ? 0 : S - 1;
  for (int i = gw; i < nsweeps; i += TW) {
    const int tasks = (S - 1 - i + BWc - 1) / BWc;
    const int prev_tasks = i > 0 ? (S - i + BWc - 1) / BWc : 0;
    volatile int* pflag;  // progress counter of the warp that owns sweep i - 1
    {
      const int gp = (i - 1 + TW) % TW;
      if (CL > 1)
        pflag = cooperative_groups::this_cluster().map_shared_rank(const_cast<int*>(prog), gp / NW) + gp % NW;
      else pflag = prog + gp;
    }
    double taug = 0.0;
#ifdef HX_CHASE_PROFILE
    long long prof_t0_ = clock64();
#endif
    for (int t = 0; t < tasks; ++t) {
      HX_PROF_MARK(0);
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 2, prev_tasks);
        // latency-bound launches (clusters / many sweeps per matrix) poll tightly, throughput-bound ones
        // back off so that waiting warps do not steal issue slots from working ones
        if (lane == 0)
          while (*pflag < need) __nanosleep(CL > 1 || NW >= 6 ? 20 : 200);
        __syncwarp();
        if (CL > 1) __threadfence();
        else __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, S - s);
      const int lb = max(0, min(BWc, S - s - len));
      HX_PROF_MARK(1);  // wait for the previous sweep
      // ---- X and Y tiles (asynchronous, zero-padded); blk = &C[s + lane][s], columns ld apart
      double2* const blk = C + ((size_t)s * ld + s + lane);
      if (len == BWc && (!DUAL || lb == BWc)) {  // full tiles: no padding predicates
        const double2* src = blk;
#pragma unroll 8
        for (int cc = 0; cc < BWc; ++cc, src += ld) bd_cp_async16<L2ONLY>(&W.X[lane][cc], src);
        if (DUAL) {
#pragma unroll 8
          for (int cc = 0; cc < BWc; ++cc, src += ld) bd_cp_async16<L2ONLY>(&W.Y[lane][cc], src);
        }
      } else {
        const double2* src = blk;
#pragma unroll 4
        for (int cc = 0; cc < BWc; ++cc, src += ld) {
          if (lane < len && cc < len) bd_cp_async16<L2ONLY>(&W.X[lane][cc], src);
          else W.X[lane][cc] = zero;
        }
        if (DUAL) {
#pragma unroll 4
          for (int cc = 0; cc < BWc; ++cc, src += ld) {
            if (lane < len && cc < lb) bd_cp_async16<L2ONLY>(&W.Y[lane][cc], src);
            else W.Y[lane][cc] = zero;
          }
        }
      }
      if (t == 0) {
        // right reflector from row i, columns [s, s+len): row i -> (conj beta, 0, ...) = (gamma_i, 0, ...)
        double2 x = zero;
        if (lane < len) {
          const double2* zp = C + (size_t)(s + lane) * ld + i;
          const double2 z = L2ONLY ? __ldcg(zp) : *zp;
          x = make_double2(z.x, -z.y);
        }
        const double sig2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const QuickReflector h = quick_reflector(al, sig2);
        taug = h.tau;
        W.ug[lane] = lane == 0 ? make_double2(1.0, 0.0) : (lane < len ? cmul(x, h.scale) : zero);
        if (lane < len && taug != 0.0)
          C[(size_t)(s + lane) * ld + i] = lane == 0 ? make_double2(h.beta.x, -h.beta.y) : zero;
        if (lane == 0) e2[2 * i + 1] = sig2;
      }
      bd_cp_async_wait_all();
      __syncwarp();
      // ---- X row pass: ty = tau_g (X u)_r, column 0 of X G, left reflector H
      double2 ty;
      {
        double2 a0 = zero, a1 = zero;
#pragma unroll 4
        for (int c = 0; c < BWc; c += 2) {
          const double2 x0 = W.X[lane][c], u0 = W.ug[c], x1 = W.X[lane][c + 1], u1 = W.ug[c + 1];
          a0.x = fma(x0.x, u0.x, fma(-x0.y, u0.y, a0.x));
          a0.y = fma(x0.x, u0.y, fma(x0.y, u0.x, a0.y));
          a1.x = fma(x1.x, u1.x, fma(-x1.y, u1.y, a1.x));
          a1.y = fma(x1.x, u1.y, fma(x1.y, u1.x, a1.y));
        }
        ty = make_double2(taug * (a0.x + a1.x), taug * (a0.y + a1.y));
      }
      const double2 x00 = W.X[lane][0];
      const double2 x0 = make_double2(x00.x - ty.x, x00.y - ty.y);
      const double sh2 = warp_sum(x0.x * x0.x + x0.y * x0.y);
      const double2 ah = make_double2(__shfl_sync(0xffffffffu, x0.x, 0), __shfl_sync(0xffffffffu, x0.y, 0));
      const QuickReflector hh = quick_reflector(ah, sh2);
      const double tauh = hh.tau;
      if (t == 0 && lane == 0) e2[2 * s] = sh2;
      const double2 v = lane == 0 ? make_double2(1.0, 0.0) : cmul(x0, hh.scale);  // zero on padded rows
      W.vh[lane] = v;
      const double2 w = warp_csum(cmul_cj(v, ty));  // v^H (tau_g y)
      __syncwarp();
      HX_PROF_MARK(4);  // X row pass + H
      // ---- X column pass: p = v^H X, b_c = tau_h (p_c - w conj(u_c))
      {
        double2 a0 = zero, a1 = zero;
#pragma unroll 4
        for (int r = 0; r < BWc; r += 2) {
          const double2 v0 = W.vh[r], x0c = W.X[r][lane], v1 = W.vh[r + 1], x1c = W.X[r + 1][lane];
          a0.x = fma(v0.x, x0c.x, fma(v0.y, x0c.y, a0.x));
          a0.y = fma(v0.x, x0c.y, fma(-v0.y, x0c.x, a0.y));
          a1.x = fma(v1.x, x1c.x, fma(v1.y, x1c.y, a1.x));
          a1.y = fma(v1.x, x1c.y, fma(-v1.y, x1c.x, a1.y));
        }
        const double2 u = W.ug[lane];
        const double2 wu = make_double2(w.x * u.x + w.y * u.y, w.y * u.x - w.x * u.y);  // w conj(u)
        W.cb[lane] = make_double2(tauh * (a0.x + a1.x - wu.x), tauh * (a0.y + a1.y - wu.y));
      }
      __syncwarp();
      HX_PROF_MARK(5);  // X column pass
      // ---- X: fused rank-2 row update, straight to HBM: X' = X - ty conj(u) - v b
      if (lane < len) {
        double2* dst = blk;
#pragma unroll 4
        for (int c = 0; c < BWc; ++c, dst += ld) {
          const double2 u = W.ug[c], b = W.cb[c];
          double2 z = W.X[lane][c];
          z.x -= (ty.x * u.x + ty.y * u.y) + (v.x * b.x - v.y * b.y);
          z.y -= (ty.y * u.x - ty.x * u.y) + (v.x * b.y + v.y * b.x);
          if (c == 0 && tauh != 0.0) z = lane == 0 ? hh.beta : zero;
          if (c < len) *dst = z;
        }
      }
      HX_PROF_MARK(6);  // X update + stores
      double next_tau = 0.0;
      if (lb > 0) {
        if (!DUAL) {  // Y into the (now free) tile buffer
          __syncwarp();
          const double2* src = blk + (size_t)len * ld;
          if (len == BWc && lb == BWc) {
#pragma unroll 8
            for (int cc = 0; cc < BWc; ++cc, src += ld) bd_cp_async16<L2ONLY>(&W.X[lane][cc], src);
          } else {
#pragma unroll 4
            for (int cc = 0; cc < BWc; ++cc, src += ld) {
              if (lane < len && cc < lb) bd_cp_async16<L2ONLY>(&W.X[lane][cc], src);
              else W.X[lane][cc] = zero;
            }
          }
          bd_cp_async_wait_all();
          __syncwarp();
        }
        HX_PROF_MARK(7);  // Y tile (single-tile variant)
        double2(*Y)[BWc + 1] = Yt();
        // ---- Y column pass: q = v^H Y, row 0 of H Y -> next right reflector G'
        double2 q;
        {
          double2 a0 = zero, a1 = zero;
#pragma unroll 4
          for (int r = 0; r < BWc; r += 2) {
            const double2 v0 = W.vh[r], y0c = Y[r][lane], v1 = W.vh[r + 1], y1c = Y[r + 1][lane];
            a0.x = fma(v0.x, y0c.x, fma(v0.y, y0c.y, a0.x));
            a0.y = fma(v0.x, y0c.y, fma(-v0.y, y0c.x, a0.y));
            a1.x = fma(v1.x, y1c.x, fma(v1.y, y1c.y, a1.x));
            a1.y = fma(v1.x, y1c.y, fma(-v1.y, y1c.x, a1.y));
          }
          q = make_double2(a0.x + a1.x, a0.y + a1.y);
        }
        const double2 y0 = Y[0][lane];
        const double2 xg = make_double2(y0.x - tauh * q.x, -(y0.y - tauh * q.y));  // conj(row 0 of H Y)
        const double sg2 = warp_sum(xg.x * xg.x + xg.y * xg.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, xg.x, 0), __shfl_sync(0xffffffffu, xg.y, 0));
        const QuickReflector hg = quick_reflector(al, sg2);
        next_tau = hg.tau;
        const double2 u2 = lane == 0 ? make_double2(1.0, 0.0) : cmul(xg, hg.scale);  // zero on padded columns
        const double2 qu = warp_csum(cmul(q, u2));                                    // (v^H Y) u'
        __syncwarp();  // everyone is done with ug (X update) and cb
        W.ug[lane] = u2;
        W.cb[lane] = make_double2(tauh * q.x, tauh * q.y);  // d_c
        __syncwarp();
        HX_PROF_MARK(8);  // Y column pass + G'
        // ---- Y row pass: f = tau_g' (Y u' - tau_h v (q . u')), Y' = Y - v d - f conj(u'), to HBM
        if (lane < len) {
          double2 a0 = zero, a1 = zero;
#pragma unroll 4
          for (int c = 0; c < BWc; c += 2) {
            const double2 y0c = Y[lane][c], u0 = W.ug[c], y1c = Y[lane][c + 1], u1 = W.ug[c + 1];
            a0.x = fma(y0c.x, u0.x, fma(-y0c.y, u0.y, a0.x));
            a0.y = fma(y0c.x, u0.y, fma(y0c.y, u0.x, a0.y));
            a1.x = fma(y1c.x, u1.x, fma(-y1c.y, u1.y, a1.x));
            a1.y = fma(y1c.x, u1.y, fma(y1c.y, u1.x, a1.y));
          }
          const double2 vq = cmul(v, qu);
          const double2 f = make_double2(next_tau * (a0.x + a1.x - tauh * vq.x), next_tau * (a0.y + a1.y - tauh * vq.y));
          const bool row0 = lane == 0 && next_tau != 0.0;
          double2* dst = blk + (size_t)len * ld;
#pragma unroll 4
          for (int c = 0; c < BWc; ++c, dst += ld) {
            const double2 u = W.ug[c], d = W.cb[c];
            double2 z = Y[lane][c];
            z.x -= (v.x * d.x - v.y * d.y) + (f.x * u.x + f.y * u.y);
            z.y -= (v.x * d.y + v.y * d.x) + (f.y * u.x - f.x * u.y);
            if (row0) z = c == 0 ? make_double2(hg.beta.x, -hg.beta.y) : zero;  // (conj beta', 0, ...)
            if (c < lb) *dst = z;
          }
        }
      }
      HX_PROF_MARK(9);  // Y row pass + update + stores
      taug = next_tau;
      if (CL > 1) __threadfence();
      else __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[warp] = i * 65536 + t + 1;
      HX_PROF_MARK(10);  // fence + publish
    }
  }
  if (CL > 1) cooperative_groups::this_cluster().sync();  // remote pollers may still read our counters
}

// ---------------------------------------------------------------------------------------------------
// Real variant for the batches whose band is real (periodic gauge at time-reversal-invariant k, see
// bd_assemble_kernel): same sweep / task / progress-flag structure as bd_chase_kernel (one warp per
// sweep, single tile buffer), real reflectors, real tiles (half the shared memory per warp, a quarter of
// the arithmetic).  Only the real parts of the double2 band are read (8-byte cp.async) and written.
// Poll interval of a waiting sweep in the real chase (ns; HX_CHASE_SPIN_NS).
__constant__ unsigned g_spin_ns = 20;

struct QuickReflectorR {
  double tau, scale, beta;
};
__device__ __forceinline__ QuickReflectorR quick_reflector_r(double alpha, double sig2) {
  QuickReflectorR h;
  if (!(sig2 >= HX_REFLECTOR_TINY)) {
    h.tau = h.scale = h.beta = 0.0;
    return h;
  }
  const double aa = fabs(alpha), ph = alpha < 0.0 ? -1.0 : 1.0;
  if (aa * aa < 1e-280 && alpha != 0.0) {
    const double sigma = sqrt(sig2), mag = aa + sigma;
    h.tau = mag / sigma;
    h.scale = ph / mag;
    h.beta = -ph * sigma;
    return h;
  }
  const double rs = rsqrt(sig2), sigma = sig2 * rs, mag = aa + sigma;
  h.tau = mag * rs;
  h.scale = ph * __drcp_rn(mag);
  h.beta = -ph * sigma;
  return h;
}

// Compact real band of the real chase: element (r, c) with c - 63 <= r <= c + 31 (the upper band of width
// 32 plus the bulges of the X and Y tiles) at B[c * RB_LD + r - c + RB_OFF]; stepping one column right
// along a row is a stride of RB_LD - 1.
constexpr int RB_LD = 96, RB_OFF = 63;

// Tile rows of stride BWc + 2 (even): a lane's row is 16-byte aligned, so the row passes and the
// broadcast vectors use 128-bit shared loads (half the LDS instructions of a stride-(BWc + 1) tile; the
// column passes stay conflict-free, the 8-byte tile fills see 2-way conflicts).
template <int BWc>
struct __align__(16) BdChaseSmemR {
  double X[BWc][BWc + 2];  // X, then Y (zero-padded)
  double ug[BWc], vh[BWc], cb[BWc];
};

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// Two warp sums in one reduction round (the shuffles of the two values pipeline).
__device__ __forceinline__ void warp_sum2(double& a, double& b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
}

__device__ __forceinline__ void bd_cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}

// CL > 1: the sweeps of one matrix are dealt round-robin to the warps of a CL-CTA cluster (CL x NW sweeps
// in flight on CL SMs, for launches with few matrices); progress counters are read across the cluster
// through DSMEM, the band goes through L2 (ld.global.cg: another SM's stores are not visible in this SM's
// L1) and the fences are device-scope.
template <int NW, int BWc, int CL = 1>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NW * 32, 1)
    bd_chase_real_kernel(double2* ws, size_t stride, size_t band_off, size_t tgk_off, int S, const int* dims) {
  extern __shared__ __align__(16) unsigned char bd_smem[];
  BdChaseSmemR<BWc>* all = reinterpret_cast<BdChaseSmemR<BWc>*>(bd_smem);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  BdChaseSmemR<BWc>& W = all[warp];
  const int rank = CL > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int gw = rank * NW + warp;  // global warp (sweep slot) of the cluster
  constexpr int TW = CL * NW;
  const int64_t mat = blockIdx.x / CL;
  double2* base = ws + (size_t)mat * stride;
  // compact real band (bd_band_extract_kernel): element (r, c), c - 63 <= r <= c + 31, at B[c * RB_LD + r - c + 63]
  double* B = reinterpret_cast<double*>(base + band_off);
  double* diag = reinterpret_cast<double*>(base + tgk_off);
  double* e2 = diag + 2 * S;
  for (int q = threadIdx.x + rank * blockDim.x; q < 2 * S; q += blockDim.x * CL) {
    diag[q] = 0.0;
    e2[q] = 0.0;
  }
  if (lane == 0) prog[warp] = -1;
  if constexpr (CL > 1) {
    __threadfence();
    cooperative_groups::this_cluster().sync();
  } else {
    __syncthreads();
  }
  if (rank == 0 && threadIdx.x == 0) {
    const double a0 = B[RB_OFF];
    e2[0] = a0 * a0;  // alpha_0: final after stage 1
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
    double taug = 0.0;
    for (int t = 0; t < tasks; ++t) {
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 2, prev_tasks);
        if (lane == 0)
          while (*pflag < need) __nanosleep(g_spin_ns);
        __syncwarp();
        if constexpr (CL > 1) __threadfence();
        else __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, S - s);
      const int lb = max(0, min(BWc, S - s - len));
      // ---- X tile (zero-padded): element (s + lane, s + cc) at blk[cc * (RB_LD - 1)]
      double* const blk = B + ((size_t)s * RB_LD + lane + RB_OFF);
      {
        const double* src = blk;
        if (CL > 1) {  // L2-coherent loads (the band is written by other SMs of the cluster)
#pragma unroll 8
          for (int cc = 0; cc < BWc; ++cc, src += RB_LD - 1)
            W.X[lane][cc] = (len == BWc || (lane < len && cc < len)) ? __ldcg(src) : 0.0;
        } else if (len == BWc) {
#pragma unroll 8
          for (int cc = 0; cc < BWc; ++cc, src += RB_LD - 1) bd_cp_async8(&W.X[lane][cc], src);
        } else {
#pragma unroll 4
          for (int cc = 0; cc < BWc; ++cc, src += RB_LD - 1) {
            if (lane < len && cc < len) bd_cp_async8(&W.X[lane][cc], src);
            else W.X[lane][cc] = 0.0;
          }
        }
      }
      if (t == 0) {
        // right reflector from row i, columns [s, s+len): row i -> (beta, 0, ...)
        double* const rowi = B + ((size_t)(s + lane) * RB_LD + i - (s + lane) + RB_OFF);  // (i, s + lane)
        const double x = lane < len ? (CL > 1 ? __ldcg(rowi) : *rowi) : 0.0;
        const double sig2 = warp_sum(x * x);
        const QuickReflectorR h = quick_reflector_r(__shfl_sync(0xffffffffu, x, 0), sig2);
        taug = h.tau;
        W.ug[lane] = lane == 0 ? 1.0 : (lane < len ? x * h.scale : 0.0);
        if (lane < len && taug != 0.0) *rowi = lane == 0 ? h.beta : 0.0;
        if (lane == 0) e2[2 * i + 1] = sig2;
      }
      bd_cp_async_wait_all();
      __syncwarp();
      // ---- X row pass: ty = tau_g (X u)_r; column 0 of X G -> left reflector H
      double ty;
      {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int c = 0; c < BWc; c += 2) {
          const double2 x = lds2(&W.X[lane][c]), u = lds2(&W.ug[c]);
          a0 = fma(x.x, u.x, a0);
          a1 = fma(x.y, u.y, a1);
        }
        ty = taug * (a0 + a1);
      }
      const double x0 = W.X[lane][0] - ty;
      // one reduction round for |x0|^2 and sum_{r>=1} x0_r ty_r: w = v^T (tau_g y) = ty_0 + scale * that
      double sh2 = x0 * x0, xt = lane == 0 ? 0.0 : x0 * ty;
      warp_sum2(sh2, xt);
      const QuickReflectorR hh = quick_reflector_r(__shfl_sync(0xffffffffu, x0, 0), sh2);
      const double tauh = hh.tau;
      if (t == 0 && lane == 0) e2[2 * s] = sh2;
      const double v = lane == 0 ? 1.0 : x0 * hh.scale;  // zero on padded rows
      W.vh[lane] = v;
      const double w = fma(hh.scale, xt, __shfl_sync(0xffffffffu, ty, 0));
      __syncwarp();
      // ---- X column pass: p = v^T X, b_c = tau_h (p_c - w u_c)
      {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int r = 0; r < BWc; r += 2) {
          const double2 vv = lds2(&W.vh[r]);
          a0 = fma(vv.x, W.X[r][lane], a0);
          a1 = fma(vv.y, W.X[r + 1][lane], a1);
        }
        W.cb[lane] = tauh * (a0 + a1 - w * W.ug[lane]);
      }
      __syncwarp();
      // ---- X: fused rank-2 row update, straight to HBM: X' = X - ty u^T - v b^T
      if (lane < len) {
        double* dst = blk;
#pragma unroll 4
        for (int c = 0; c < BWc; c += 2, dst += 2 * (RB_LD - 1)) {
          const double2 x = lds2(&W.X[lane][c]), u = lds2(&W.ug[c]), b = lds2(&W.cb[c]);
          double z0 = fma(-v, b.x, fma(-ty, u.x, x.x));
          const double z1 = fma(-v, b.y, fma(-ty, u.y, x.y));
          if (c == 0 && tauh != 0.0) z0 = lane == 0 ? hh.beta : 0.0;
          if (c < len) dst[0] = z0;
          if (c + 1 < len) dst[RB_LD - 1] = z1;
        }
      }
      double next_tau = 0.0;
      if (lb > 0) {
        __syncwarp();
        {
          const double* src = blk + (size_t)len * (RB_LD - 1);  // (s + lane, s + len + cc)
          if (CL > 1) {
#pragma unroll 8
            for (int cc = 0; cc < BWc; ++cc, src += RB_LD - 1)
              W.X[lane][cc] = ((len == BWc && lb == BWc) || (lane < len && cc < lb)) ? __ldcg(src) : 0.0;
          } else if (len == BWc && lb == BWc) {
#pragma unroll 8
            for (int cc = 0; cc < BWc; ++cc, src += RB_LD - 1) bd_cp_async8(&W.X[lane][cc], src);
          } else {
#pragma unroll 4
            for (int cc = 0; cc < BWc; ++cc, src += RB_LD - 1) {
              if (lane < len && cc < lb) bd_cp_async8(&W.X[lane][cc], src);
              else W.X[lane][cc] = 0.0;
            }
          }
          bd_cp_async_wait_all();
          __syncwarp();
        }
        // ---- Y column pass: q = v^T Y; row 0 of H Y -> next right reflector G'
        double q;
        {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
          for (int r = 0; r < BWc; r += 2) {
            const double2 vv = lds2(&W.vh[r]);
            a0 = fma(vv.x, W.X[r][lane], a0);
            a1 = fma(vv.y, W.X[r + 1][lane], a1);
          }
          q = a0 + a1;
        }
        const double xg = W.X[0][lane] - tauh * q;  // row 0 of H Y
        // one reduction round for |xg|^2 and sum_{c>=1} q_c xg_c: qu = (v^T Y) u' = q_0 + scale * that
        double sg2 = xg * xg, qx = lane == 0 ? 0.0 : q * xg;
        warp_sum2(sg2, qx);
        const QuickReflectorR hg = quick_reflector_r(__shfl_sync(0xffffffffu, xg, 0), sg2);
        next_tau = hg.tau;
        const double u2 = lane == 0 ? 1.0 : xg * hg.scale;  // zero on padded columns
        const double qu = fma(hg.scale, qx, __shfl_sync(0xffffffffu, q, 0));
        __syncwarp();  // everyone is done with ug (X update) and cb
        W.ug[lane] = u2;
        W.cb[lane] = tauh * q;  // d_c
        __syncwarp();
        // ---- Y row pass: f = tau_g' (Y u' - tau_h v (q . u')), Y' = Y - v d^T - f u'^T, to HBM
        if (lane < len) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
          for (int c = 0; c < BWc; c += 2) {
            const double2 x = lds2(&W.X[lane][c]), u = lds2(&W.ug[c]);
            a0 = fma(x.x, u.x, a0);
            a1 = fma(x.y, u.y, a1);
          }
          const double f = next_tau * (a0 + a1 - tauh * v * qu);
          const bool row0 = lane == 0 && next_tau != 0.0;
          double* dst = blk + (size_t)len * (RB_LD - 1);
#pragma unroll 4
          for (int c = 0; c < BWc; c += 2, dst += 2 * (RB_LD - 1)) {
            const double2 x = lds2(&W.X[lane][c]), u = lds2(&W.ug[c]), b = lds2(&W.cb[c]);
            double z0 = fma(-f, u.x, fma(-v, b.x, x.x)), z1 = fma(-f, u.y, fma(-v, b.y, x.y));
            if (row0) {
              z0 = c == 0 ? hg.beta : 0.0;
              z1 = 0.0;
            }
            if (c < lb) dst[0] = z0;
            if (c + 1 < lb) dst[RB_LD - 1] = z1;
          }
        }
      }
      taug = next_tau;
      if constexpr (CL > 1) __threadfence();
      else __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[warp] = i * 65536 + t + 1;
    }
  }
  if constexpr (CL > 1) cooperative_groups::this_cluster().sync();  // remote pollers may still read our counters
}

// ---------------------------------------------------------------------------------------------------
// Register-row variant of the real chase (HX_CHASE_REG, default on): the lane's row of the X tile (then of the
// Y tile) is loaded from the band straight into 32 registers (coalesced: a tile column is 32 consecutive
// doubles of the compact band), the row passes and the rank-2 row updates run on those registers, and the tile
// goes to shared memory once, TRANSPOSED (Xt[c][r], stride 33), only for the column pass (lane = column).
// Against bd_chase_real_kernel (tile in shared memory, read by every pass): the shared-memory data pipe - the
// measured limit of that kernel, 67-77 % of peak with 4-way conflicted 8-byte tile fills - carries about a
// third of the wavefronts per task (fills conflict-free, row passes read only the broadcast vectors).
struct __align__(16) BdChaseSmemRR {
  double ug[32], vh[32], cb[32];
  double Xt[32][33];  // X^T (then Y^T): Xt[c][r] = tile (r, c)
};

template <int CL>
__device__ __forceinline__ double ld_band(const double* p) {
  if constexpr (CL > 1) return __ldcg(p);  // written by other SMs of the cluster: through L2
  else return *p;
}

// Row `lane` of a 32 x 32 tile of the compact band into registers: r[cc] = (s + lane, c0 + cc) at p[cc * (RB_LD - 1)];
// columns >= ncols (and every column when ncols = 0: padded rows) read as zero.
template <int CL>
__device__ __forceinline__ void load_row(double (&r)[32], const double* p, bool full, int ncols) {
  if (full) {
#pragma unroll
    for (int cc = 0; cc < 32; ++cc) r[cc] = ld_band<CL>(p + cc * (RB_LD - 1));
  } else {
#pragma unroll
    for (int cc = 0; cc < 32; ++cc) r[cc] = cc < ncols ? ld_band<CL>(p + cc * (RB_LD - 1)) : 0.0;
  }
}

// Register budget: 128 per thread (4 CTAs of 4 warps per SM for the many-matrix launches).
template <int NW, int CL = 1>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NW * 32, NW == 4 ? 4 : (NW <= 2 ? 8 : 1))
    bd_chase_realr_kernel(double2* ws, size_t stride, size_t band_off, size_t tgk_off, int S, const int* dims) {
  constexpr int BWc = 32;
  extern __shared__ __align__(16) unsigned char bd_smem[];
  BdChaseSmemRR* all = reinterpret_cast<BdChaseSmemRR*>(bd_smem);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  BdChaseSmemRR& W = all[warp];
  const int rank = CL > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int gw = rank * NW + warp;
  constexpr int TW = CL * NW;
  const int64_t mat = blockIdx.x / CL;
  double2* base = ws + (size_t)mat * stride;
  double* B = reinterpret_cast<double*>(base + band_off);
  double* diag = reinterpret_cast<double*>(base + tgk_off);
  double* e2 = diag + 2 * S;
  for (int q = threadIdx.x + rank * blockDim.x; q < 2 * S; q += blockDim.x * CL) {
    diag[q] = 0.0;
    e2[q] = 0.0;
  }
  if (lane == 0) prog[warp] = -1;
  if constexpr (CL > 1) {
    __threadfence();
    cooperative_groups::this_cluster().sync();
  } else {
    __syncthreads();
  }
  if (rank == 0 && threadIdx.x == 0) {
    const double a0 = B[RB_OFF];
    e2[0] = a0 * a0;  // alpha_0: final after stage 1
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
    double taug = 0.0;
    for (int t = 0; t < tasks; ++t) {
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 2, prev_tasks);
        if (lane == 0)
          while (*pflag < need) __nanosleep(g_spin_ns);
        __syncwarp();
        if constexpr (CL > 1) __threadfence();
        else __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, S - s);
      const int lb = max(0, min(BWc, S - s - len));
      // element (s + lane, s + cc) at blk[cc * (RB_LD - 1)]
      double* const blk = B + ((size_t)s * RB_LD + lane + RB_OFF);
      double xr[BWc];
      load_row<CL>(xr, blk, len == BWc, lane < len ? len : 0);
      if (t == 0) {
        // right reflector from row i, columns [s, s+len): row i -> (beta, 0, ...)
        double* const rowi = B + ((size_t)(s + lane) * RB_LD + i - (s + lane) + RB_OFF);  // (i, s + lane)
        const double x = lane < len ? ld_band<CL>(rowi) : 0.0;
        const double sig2 = warp_sum(x * x);
        const QuickReflectorR h = quick_reflector_r(__shfl_sync(0xffffffffu, x, 0), sig2);
        taug = h.tau;
        W.ug[lane] = lane == 0 ? 1.0 : (lane < len ? x * h.scale : 0.0);
        if (lane < len && taug != 0.0) *rowi = lane == 0 ? h.beta : 0.0;
        if (lane == 0) e2[2 * i + 1] = sig2;
      }
#pragma unroll
      for (int cc = 0; cc < BWc; ++cc) W.Xt[cc][lane] = xr[cc];
      __syncwarp();
      // ---- X row pass (registers): ty = tau_g (X u)_r; column 0 of X G -> left reflector H
      double ty;
      {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int c = 0; c < BWc; c += 2) {
          const double2 u = lds2(&W.ug[c]);
          a0 = fma(xr[c], u.x, a0);
          a1 = fma(xr[c + 1], u.y, a1);
        }
        ty = taug * (a0 + a1);
      }
      const double x0 = xr[0] - ty;
      double sh2 = x0 * x0, xt = lane == 0 ? 0.0 : x0 * ty;
      warp_sum2(sh2, xt);
      const QuickReflectorR hh = quick_reflector_r(__shfl_sync(0xffffffffu, x0, 0), sh2);
      const double tauh = hh.tau;
      if (t == 0 && lane == 0) e2[2 * s] = sh2;
      const double v = lane == 0 ? 1.0 : x0 * hh.scale;  // zero on padded rows
      W.vh[lane] = v;
      const double w = fma(hh.scale, xt, __shfl_sync(0xffffffffu, ty, 0));
      __syncwarp();
      // ---- X column pass (lane = column, X^T in shared memory): b_c = tau_h (v^T X_c - w u_c)
      {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int r = 0; r < BWc; r += 2) {
          const double2 vv = lds2(&W.vh[r]);
          a0 = fma(vv.x, W.Xt[lane][r], a0);
          a1 = fma(vv.y, W.Xt[lane][r + 1], a1);
        }
        W.cb[lane] = tauh * (a0 + a1 - w * W.ug[lane]);
      }
      __syncwarp();
      // ---- X: fused rank-2 row update on the registers, straight to HBM: X' = X - ty u^T - v b^T
      if (lane < len) {
#pragma unroll
        for (int c = 0; c < BWc; c += 2) {
          const double2 u = lds2(&W.ug[c]), b = lds2(&W.cb[c]);
          double z0 = fma(-v, b.x, fma(-ty, u.x, xr[c]));
          const double z1 = fma(-v, b.y, fma(-ty, u.y, xr[c + 1]));
          if (c == 0 && tauh != 0.0) z0 = lane == 0 ? hh.beta : 0.0;
          if (c < len) blk[c * (RB_LD - 1)] = z0;
          if (c + 1 < len) blk[(c + 1) * (RB_LD - 1)] = z1;
          if ((c & 7) == 6) asm volatile("" ::: "memory");  // bound the broadcast loads in flight (registers)
        }
      }
      double next_tau = 0.0;
      if (lb > 0) {
        // (s + lane, s + len + cc)
        load_row<CL>(xr, blk + (size_t)len * (RB_LD - 1), len == BWc && lb == BWc, lane < len ? lb : 0);
#pragma unroll
        for (int cc = 0; cc < BWc; ++cc) W.Xt[cc][lane] = xr[cc];
        __syncwarp();
        // ---- Y column pass: q = v^T Y; row 0 of H Y -> next right reflector G'
        double q;
        {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int r = 0; r < BWc; r += 2) {
            const double2 vv = lds2(&W.vh[r]);
            a0 = fma(vv.x, W.Xt[lane][r], a0);
            a1 = fma(vv.y, W.Xt[lane][r + 1], a1);
          }
          q = a0 + a1;
        }
        const double xg = W.Xt[lane][0] - tauh * q;  // row 0 of H Y
        double sg2 = xg * xg, qx = lane == 0 ? 0.0 : q * xg;
        warp_sum2(sg2, qx);
        const QuickReflectorR hg = quick_reflector_r(__shfl_sync(0xffffffffu, xg, 0), sg2);
        next_tau = hg.tau;
        const double u2 = lane == 0 ? 1.0 : xg * hg.scale;  // zero on padded columns
        const double qu = fma(hg.scale, qx, __shfl_sync(0xffffffffu, q, 0));
        __syncwarp();  // everyone is done with ug (X update) and cb
        W.ug[lane] = u2;
        W.cb[lane] = tauh * q;  // d_c
        __syncwarp();
        // ---- Y row pass (registers): f = tau_g' (Y u' - tau_h v (q . u')), Y' = Y - v d^T - f u'^T, to HBM
        if (lane < len) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int c = 0; c < BWc; c += 2) {
            const double2 u = lds2(&W.ug[c]);
            a0 = fma(xr[c], u.x, a0);
            a1 = fma(xr[c + 1], u.y, a1);
          }
          const double f = next_tau * (a0 + a1 - tauh * v * qu);
          const bool row0 = lane == 0 && next_tau != 0.0;
          double* const dst = blk + (size_t)len * (RB_LD - 1);
#pragma unroll
          for (int c = 0; c < BWc; c += 2) {
            const double2 u = lds2(&W.ug[c]), b = lds2(&W.cb[c]);
            double z0 = fma(-f, u.x, fma(-v, b.x, xr[c])), z1 = fma(-f, u.y, fma(-v, b.y, xr[c + 1]));
            if (row0) {
              z0 = c == 0 ? hg.beta : 0.0;
              z1 = 0.0;
            }
            if (c < lb) dst[c * (RB_LD - 1)] = z0;
            if (c + 1 < lb) dst[(c + 1) * (RB_LD - 1)] = z1;
            if ((c & 7) == 6) asm volatile("" ::: "memory");
          }
        }
      }
      taug = next_tau;
      if constexpr (CL > 1) __threadfence();
      else __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[warp] = i * 65536 + t + 1;
    }
  }
  if constexpr (CL > 1) cooperative_groups::this_cluster().sync();  // remote pollers may still read our counters
}

template <int NW>
constexpr size_t bd_chase_realr_smem() {
  return NW * sizeof(BdChaseSmemRR) + 64;
}

// Real parts of the upper band (and the zero window around it) of the dense S x S slab C into the compact
// band buffer of the real chase.  One CTA per matrix.
static __global__ void __launch_bounds__(256) bd_band_extract_kernel(double2* ws, size_t stride, size_t c_off,
                                                                      size_t band_off, int S) {
  double2* base = ws + (size_t)blockIdx.x * stride;
  const double2* C = base + c_off;
  double* B = reinterpret_cast<double*>(base + band_off);
  const size_t n = (size_t)S * RB_LD;
  for (size_t p = threadIdx.x; p < n; p += blockDim.x) {
    const int c = (int)(p / RB_LD), r = c + (int)(p % RB_LD) - RB_OFF;
    B[p] = (r >= 0 && r < S) ? C[r + (size_t)c * S].x : 0.0;
  }
}

template <int NW, int BWc>
constexpr size_t bd_chase_real_smem() {
  return NW * sizeof(BdChaseSmemR<BWc>) + 64;
}

// ---------------------------------------------------------------------------------------------------
// Warp-pair variant: every task is split over two warps (64 threads, a pair of one "slot"), halving the
// serial instruction stream of a task (the chase is bound by the latency of one task times the sweep
// stagger, and by the issue rate of the few tasks in flight).  Lane = row in the row-oriented phases
// (each warp takes 16 of the 32 tile columns), lane = column in the column-oriented phases (each warp
// takes 16 of the 32 tile rows); the half sums meet in shared memory behind a 64-thread named barrier.
// Reflectors are built redundantly by both warps from the combined sums (identical values, each warp
// keeps its own copy), so only the partial sums cross warps.  The Y tile is loaded into the X buffer
// after the X update: each warp overwrites exactly the columns it alone reads in the row phases.
template <int BWc>
struct BdPairSmem {
  double2 X[BWc][BWc + 1];  // X, then Y (zero-padded)
  double2 ug[2][BWc];       // right reflector vector, per warp
  double2 vh[2][BWc];       // left reflector vector, per warp
  double2 cb[2][BWc];       // per-column update coefficients, per warp
  double2 part[2][2][BWc];  // [buffer][half][row or column] partial sums (alternating buffers)
};

__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <int NT, int BWc>
__global__ void __launch_bounds__(NT * 64, NT <= 2 ? 4 : 1) bd_chase_pair_kernel(double2* ws, size_t stride, size_t c_off,
                                                                    size_t tgk_off, int S, const int* dims) {
  static_assert(BWc == 32, "lane = row / column of a 32-wide tile");
  static_assert(NT <= 15, "one named barrier per slot");
  constexpr int HW = BWc / 2;
  extern __shared__ __align__(16) unsigned char bd_smem[];
  BdPairSmem<BWc>* all = reinterpret_cast<BdPairSmem<BWc>*>(bd_smem);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NT);
  const int lane = threadIdx.x & 31, slot = threadIdx.x >> 6, h = (threadIdx.x >> 5) & 1;
  const int bar = 1 + slot;
  BdPairSmem<BWc>& W = all[slot];
  double2* const ug = W.ug[h];
  double2* const vh = W.vh[h];
  double2* const cb = W.cb[h];
  const int64_t mat = blockIdx.x;
  double2* base = ws + (size_t)mat * stride;
  double2* C = base + c_off;
  double* diag = reinterpret_cast<double*>(base + tgk_off);
  double* e2 = diag + 2 * S;
  const int ld = S;
  const double2 zero = make_double2(0.0, 0.0);
  for (int q = threadIdx.x; q < 2 * S; q += blockDim.x) {
    diag[q] = 0.0;
    e2[q] = 0.0;
  }
  if (threadIdx.x < NT) prog[threadIdx.x] = -1;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double2 a0 = C[0];
    e2[0] = a0.x * a0.x + a0.y * a0.y;  // alpha_0: final after stage 1
  }
  const bool skip = dims && dims[mat] == 0;
  const int nsweeps = skip ? 0 : S - 1;
  const int c0 = h * HW;  // this warp's columns (row phases) / rows (column phases)
  int pb = 0;             // alternating partial-sum buffer
  for (int i = slot; i < nsweeps; i += NT) {
    const int tasks = (S - 1 - i + BWc - 1) / BWc;
    const int prev_tasks = i > 0 ? (S - i + BWc - 1) / BWc : 0;
    volatile int* pflag = prog + (i - 1 + NT) % NT;
    double taug = 0.0;
    for (int t = 0; t < tasks; ++t) {
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 2, prev_tasks);
        if (lane == 0)
          while (*pflag < need) __nanosleep(NT >= 6 ? 20 : 100);
        __syncwarp();
        __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, S - s);
      const int lb = max(0, min(BWc, S - s - len));
      double2* const blk = C + ((size_t)s * ld + s + lane);
      // ---- X tile, this warp's 16 columns
      {
        const double2* src = blk + (size_t)c0 * ld;
        if (len == BWc) {
#pragma unroll
          for (int cc = 0; cc < HW; ++cc, src += ld) bd_cp_async16<false>(&W.X[lane][c0 + cc], src);
        } else {
#pragma unroll 4
          for (int cc = 0; cc < HW; ++cc, src += ld) {
            if (lane < len && c0 + cc < len) bd_cp_async16<false>(&W.X[lane][c0 + cc], src);
            else W.X[lane][c0 + cc] = zero;
          }
        }
      }
      if (t == 0) {
        // right reflector from row i, columns [s, s+len) (both warps, identical values)
        double2 x = zero;
        if (lane < len) {
          const double2 z = C[(size_t)(s + lane) * ld + i];
          x = make_double2(z.x, -z.y);
        }
        const double sig2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const QuickReflector hq = quick_reflector(al, sig2);
        taug = hq.tau;
        ug[lane] = lane == 0 ? make_double2(1.0, 0.0) : (lane < len ? cmul(x, hq.scale) : zero);
        if (h == 0) {
          if (lane < len && taug != 0.0)
            C[(size_t)(s + lane) * ld + i] = lane == 0 ? make_double2(hq.beta.x, -hq.beta.y) : zero;
          if (lane == 0) e2[2 * i + 1] = sig2;
        }
      }
      bd_cp_async_wait_all();
      pair_bar(bar);  // B1: both column halves of X in shared memory
      // ---- X row pass (lane = row): ty = tau_g (X u)_r over both halves
      {
        double2 a0 = zero, a1 = zero;
#pragma unroll
        for (int c = c0; c < c0 + HW; c += 2) {
          const double2 x0 = W.X[lane][c], u0 = ug[c], x1 = W.X[lane][c + 1], u1 = ug[c + 1];
          a0.x = fma(x0.x, u0.x, fma(-x0.y, u0.y, a0.x));
          a0.y = fma(x0.x, u0.y, fma(x0.y, u0.x, a0.y));
          a1.x = fma(x1.x, u1.x, fma(-x1.y, u1.y, a1.x));
          a1.y = fma(x1.x, u1.y, fma(x1.y, u1.x, a1.y));
        }
        W.part[pb][h][lane] = make_double2(a0.x + a1.x, a0.y + a1.y);
      }
      pair_bar(bar);  // B2
      double2 ty;
      {
        const double2 p0 = W.part[pb][0][lane], p1 = W.part[pb][1][lane];
        ty = make_double2(taug * (p0.x + p1.x), taug * (p0.y + p1.y));
      }
      pb ^= 1;
      const double2 x00 = W.X[lane][0];
      const double2 x0 = make_double2(x00.x - ty.x, x00.y - ty.y);
      const double sh2 = warp_sum(x0.x * x0.x + x0.y * x0.y);
      const double2 ah = make_double2(__shfl_sync(0xffffffffu, x0.x, 0), __shfl_sync(0xffffffffu, x0.y, 0));
      const QuickReflector hh = quick_reflector(ah, sh2);
      const double tauh = hh.tau;
      if (t == 0 && h == 0 && lane == 0) e2[2 * s] = sh2;
      const double2 v = lane == 0 ? make_double2(1.0, 0.0) : cmul(x0, hh.scale);  // zero on padded rows
      vh[lane] = v;
      const double2 w = warp_csum(cmul_cj(v, ty));  // v^H (tau_g y)
      __syncwarp();
      // ---- X column pass (lane = column): p = v^H X over this warp's 16 rows
      {
        double2 a0 = zero, a1 = zero;
#pragma unroll
        for (int r = c0; r < c0 + HW; r += 2) {
          const double2 v0 = vh[r], x0c = W.X[r][lane], v1 = vh[r + 1], x1c = W.X[r + 1][lane];
          a0.x = fma(v0.x, x0c.x, fma(v0.y, x0c.y, a0.x));
          a0.y = fma(v0.x, x0c.y, fma(-v0.y, x0c.x, a0.y));
          a1.x = fma(v1.x, x1c.x, fma(v1.y, x1c.y, a1.x));
          a1.y = fma(v1.x, x1c.y, fma(-v1.y, x1c.x, a1.y));
        }
        W.part[pb][h][lane] = make_double2(a0.x + a1.x, a0.y + a1.y);
      }
      pair_bar(bar);  // B3: partials written; both warps are done reading the other half of X
      {
        const double2 p0 = W.part[pb][0][lane], p1 = W.part[pb][1][lane];
        const double2 u = ug[lane];
        const double2 wu = make_double2(w.x * u.x + w.y * u.y, w.y * u.x - w.x * u.y);  // w conj(u)
        cb[lane] = make_double2(tauh * (p0.x + p1.x - wu.x), tauh * (p0.y + p1.y - wu.y));
      }
      pb ^= 1;
      __syncwarp();
      // ---- X: fused rank-2 row update of this warp's columns, straight to HBM:
      //      X' = X - ty conj(u) - v b   (column 0 of row 0 -> beta_h, rest of column 0 -> 0)
      if (lane < len) {
        double2* dst = blk + (size_t)c0 * ld;
#pragma unroll
        for (int c = c0; c < c0 + HW; ++c, dst += ld) {
          const double2 u = ug[c], b = cb[c];
          double2 z = W.X[lane][c];
          z.x = fma(-ty.x, u.x, fma(-ty.y, u.y, fma(-v.x, b.x, fma(v.y, b.y, z.x))));
          z.y = fma(-ty.y, u.x, fma(ty.x, u.y, fma(-v.x, b.y, fma(-v.y, b.x, z.y))));
          if (c == 0 && tauh != 0.0) z = lane == 0 ? hh.beta : zero;
          if (c < len) *dst = z;
        }
      }
      double next_tau = 0.0;
      if (lb > 0) {
        // ---- Y tile into the X buffer, this warp's columns (it alone reads them from here on in row phases)
        {
          __syncwarp();
          const double2* src = blk + (size_t)(len + c0) * ld;
          if (len == BWc && lb == BWc) {
#pragma unroll
            for (int cc = 0; cc < HW; ++cc, src += ld) bd_cp_async16<false>(&W.X[lane][c0 + cc], src);
          } else {
#pragma unroll 4
            for (int cc = 0; cc < HW; ++cc, src += ld) {
              if (lane < len && c0 + cc < lb) bd_cp_async16<false>(&W.X[lane][c0 + cc], src);
              else W.X[lane][c0 + cc] = zero;
            }
          }
          bd_cp_async_wait_all();
        }
        pair_bar(bar);  // B4: both halves of Y loaded
        // ---- Y column pass (lane = column): q = v^H Y over this warp's rows
        {
          double2 a0 = zero, a1 = zero;
#pragma unroll
          for (int r = c0; r < c0 + HW; r += 2) {
            const double2 v0 = vh[r], y0c = W.X[r][lane], v1 = vh[r + 1], y1c = W.X[r + 1][lane];
            a0.x = fma(v0.x, y0c.x, fma(v0.y, y0c.y, a0.x));
            a0.y = fma(v0.x, y0c.y, fma(-v0.y, y0c.x, a0.y));
            a1.x = fma(v1.x, y1c.x, fma(v1.y, y1c.y, a1.x));
            a1.y = fma(v1.x, y1c.y, fma(-v1.y, y1c.x, a1.y));
          }
          W.part[pb][h][lane] = make_double2(a0.x + a1.x, a0.y + a1.y);
        }
        pair_bar(bar);  // B5
        double2 q;
        {
          const double2 p0 = W.part[pb][0][lane], p1 = W.part[pb][1][lane];
          q = make_double2(p0.x + p1.x, p0.y + p1.y);
        }
        pb ^= 1;
        const double2 y0 = W.X[0][lane];
        const double2 xg = make_double2(y0.x - tauh * q.x, -(y0.y - tauh * q.y));  // conj(row 0 of H Y)
        const double sg2 = warp_sum(xg.x * xg.x + xg.y * xg.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, xg.x, 0), __shfl_sync(0xffffffffu, xg.y, 0));
        const QuickReflector hg = quick_reflector(al, sg2);
        next_tau = hg.tau;
        const double2 u2 = lane == 0 ? make_double2(1.0, 0.0) : cmul(xg, hg.scale);  // zero on padded columns
        const double2 qu = warp_csum(cmul(q, u2));                                    // (v^H Y) u'
        ug[lane] = u2;  // this warp's copy: its X update (the last reader) is done
        cb[lane] = make_double2(tauh * q.x, tauh * q.y);  // d_c
        __syncwarp();
        // ---- Y row pass (lane = row): f = tau_g' (Y u' - tau_h v (q . u')) over both halves
        {
          double2 a0 = zero, a1 = zero;
#pragma unroll
          for (int c = c0; c < c0 + HW; c += 2) {
            const double2 y0c = W.X[lane][c], u0 = ug[c], y1c = W.X[lane][c + 1], u1 = ug[c + 1];
            a0.x = fma(y0c.x, u0.x, fma(-y0c.y, u0.y, a0.x));
            a0.y = fma(y0c.x, u0.y, fma(y0c.y, u0.x, a0.y));
            a1.x = fma(y1c.x, u1.x, fma(-y1c.y, u1.y, a1.x));
            a1.y = fma(y1c.x, u1.y, fma(y1c.y, u1.x, a1.y));
          }
          W.part[pb][h][lane] = make_double2(a0.x + a1.x, a0.y + a1.y);
        }
        pair_bar(bar);  // B6
        double2 f;
        {
          const double2 p0 = W.part[pb][0][lane], p1 = W.part[pb][1][lane];
          const double2 vq = cmul(v, qu);
          f = make_double2(next_tau * (p0.x + p1.x - tauh * vq.x), next_tau * (p0.y + p1.y - tauh * vq.y));
        }
        pb ^= 1;
        // ---- Y' = Y - v d - f conj(u') on this warp's columns, to HBM; row 0 -> (conj beta', 0, ...)
        if (lane < len) {
          const bool row0 = lane == 0 && next_tau != 0.0;
          double2* dst = blk + (size_t)(len + c0) * ld;
#pragma unroll
          for (int c = c0; c < c0 + HW; ++c, dst += ld) {
            const double2 u = ug[c], dd = cb[c];
            double2 z = W.X[lane][c];
            z.x = fma(-v.x, dd.x, fma(v.y, dd.y, fma(-f.x, u.x, fma(-f.y, u.y, z.x))));
            z.y = fma(-v.x, dd.y, fma(-v.y, dd.x, fma(-f.y, u.x, fma(f.x, u.y, z.y))));
            if (row0) z = c == 0 ? make_double2(hg.beta.x, -hg.beta.y) : zero;
            if (c < lb) *dst = z;
          }
        }
      }
      taug = next_tau;
      __threadfence_block();
      pair_bar(bar);  // B7: both warps' stores done (and the X buffer free for the next task)
      if (h == 0 && lane == 0) prog[slot] = i * 65536 + t + 1;
    }
  }
}

template <int NT, int BWc>
constexpr size_t bd_chase_pair_smem() {
  return NT * sizeof(BdPairSmem<BWc>) + 64;
}

template <int NW, int BWc, bool DUAL>
constexpr size_t bd_chase_smem() {
  return NW * sizeof(BdChaseSmem<BWc, DUAL>) + 64;
}

}  // namespace hx
