// Stage 2 of the Hermitian banded path: band (lower, width BW) -> real symmetric tridiagonal by
// Householder bulge chasing, pipelined over sweeps.
//
// Sweep i annihilates column i below the subdiagonal and chases the bulge down the band in tasks
// t = 0, 1, ...; task t works on the diagonal block D = A[s:s+len, s:s+len] (s = i+1+t*BW) and the
// block below it B = A[s+len : s+len+lb, s:s+len]:
//     D <- H D H                   (two-sided: p = D v, w = tau p - tau^2/2 (v^H p) v, D -= v w^H + w v^H)
//     B <- H' B H                  (H' from column 0 of B H; fused into one rank-2 row update:
//                                   with q = tau B v, pB = v'^H B, wq = v'^H q, z = tau' (pB - wq conj(v)),
//                                   B'' = B - q v^H - v' z^T, column 0 -> (beta', 0, ...))
//     H' is carried to task t+1.
// Task t of sweep i touches rows/columns [s, s+2 BW); sweep i+1 may run task t once sweep i has completed
// task t+1.  One warp owns the sweeps i = w (mod NW) of its CTA's matrix and waits on a per-warp
// progress counter in shared memory (no CTA-wide barriers).  Tiles are zero padded to BW x BW so every
// loop is a fixed, compact 32-iteration loop (the fully predicated unrolled form was instruction-cache
// bound), lane = row for row passes and updates (stores coalesced per column), lane = column for the
// column pass.
#pragma once
#include "hx_dense.cuh"

namespace hx {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// warp sum of conj(a) * b
__device__ __forceinline__ double2 warp_csum_hx(double2 a, double2 b) {
  return make_double2(warp_sum(a.x * b.x + a.y * b.y), warp_sum(a.x * b.y - a.y * b.x));
}

// DUAL: D and B tiles staged together; otherwise one tile buffer (B loaded after the D update): half the
// shared memory per warp, twice the warps (sweeps in flight) per SM.
template <int BWc, bool DUAL>
struct ChaseWarpSmem {
  double2 D[BWc][BWc + 1];              // full Hermitian diagonal block (zero padded)
  double2 B[DUAL ? BWc : 1][BWc + 1];   // block below (zero padded)
  double2 v[BWc];           // current reflector (v[0] = 1, zero padded)
  double2 w[BWc];           // two-sided update vector
  double2 vp[BWc];          // next reflector
  double2 z[BWc];           // column coefficients of the B update
};

template <int NW, int BWc, bool DUAL>
__global__ void __launch_bounds__(NW * 32, 1) bulge_chase_pipe_kernel(double2* ws, size_t stride, size_t a_off,
                                                                       size_t dg_off, int N, const int* dims) {
  extern __shared__ __align__(16) unsigned char chase_smem[];
  ChaseWarpSmem<BWc, DUAL>* all = reinterpret_cast<ChaseWarpSmem<BWc, DUAL>*>(chase_smem);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);  // per warp: sweep*65536 + tasks done
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ChaseWarpSmem<BWc, DUAL>& S = all[warp];
  double2(*Bt)[BWc + 1] = DUAL ? S.B : S.D;
  double2* base = ws + (size_t)blockIdx.x * stride;
  double2* A = base + a_off;
  double* diag = reinterpret_cast<double*>(base + dg_off);
  double* e2 = diag + N;
  const int lda = N;
  const int d = dims ? dims[blockIdx.x] : N;
  const double2 zero = make_double2(0.0, 0.0);
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
          while (prog[pw] < need) __nanosleep(20);
        __syncwarp();
        __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, d - s);
      const int lb = max(0, min(BWc, d - s - len));
      // ---- D (lower triangle) and B tiles, asynchronously; colp = &A[s + lane][s], columns lda apart
      double2* const colp = A + ((size_t)s * lda + s + lane);
      {
        const double2* src = colp;
#pragma unroll 4
        for (int c = 0; c < BWc; ++c, src += lda) {
          if (c < len && lane >= c && lane < len) cp_async16(&S.D[lane][c], src);
          else S.D[lane][c] = zero;
        }
        if (DUAL) {
          src = colp + len;
#pragma unroll 4
          for (int c = 0; c < BWc; ++c, src += lda) {
            if (c < len && lane < lb) cp_async16(&S.B[lane][c], src);
            else S.B[lane][c] = zero;
          }
        }
      }
      if (t == 0) {
        // reflector from column i, rows s .. s+len-1
        double2 x = zero;
        if (lane < len) x = A[s + lane + (size_t)i * lda];
        const double sig2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 alpha = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const QuickReflector h = quick_reflector(alpha, sig2);
        tau = h.tau;
        S.v[lane] = lane == 0 ? make_double2(1.0, 0.0) : (lane < len ? cmul(x, h.scale) : zero);
        if (lane < len && tau != 0.0) A[s + lane + (size_t)i * lda] = lane == 0 ? h.beta : zero;
        if (lane == 0) {
          diag[i] = A[i + (size_t)i * lda].x;
          e2[i] = sig2;
        }
      }
      cp_async_wait_all();
      __syncwarp();
      // mirror the strictly upper part of D from its lower triangle
#pragma unroll 4
      for (int c = 0; c < BWc; ++c)
        if (c > lane) {
          const double2 u = S.D[c][lane];
          S.D[lane][c] = make_double2(u.x, -u.y);
        }
      __syncwarp();
      // ---- D: p = D v (lane = row), cval = v^H p, w = tau p - tau^2/2 cval v
      double2 p;
      {
        double2 a0 = zero, a1 = zero;
#pragma unroll 4
        for (int c = 0; c < BWc; c += 2) {
          const double2 x0 = S.D[lane][c], v0 = S.v[c], x1 = S.D[lane][c + 1], v1 = S.v[c + 1];
          a0.x = fma(x0.x, v0.x, fma(-x0.y, v0.y, a0.x));
          a0.y = fma(x0.x, v0.y, fma(x0.y, v0.x, a0.y));
          a1.x = fma(x1.x, v1.x, fma(-x1.y, v1.y, a1.x));
          a1.y = fma(x1.x, v1.y, fma(x1.y, v1.x, a1.y));
        }
        p = make_double2(a0.x + a1.x, a0.y + a1.y);
      }
      const double2 vr = S.v[lane];
      const double cval = warp_sum(vr.x * p.x + vr.y * p.y);
      const double hc = 0.5 * tau * tau * cval;
      const double2 wr = make_double2(tau * p.x - hc * vr.x, tau * p.y - hc * vr.y);
      S.w[lane] = wr;
      __syncwarp();
      // ---- D -= v w^H + w v^H ; lower triangle straight to HBM (coalesced per column)
      if (lane < len) {
        double2* dst = colp;
#pragma unroll 4
        for (int c = 0; c < BWc; ++c, dst += lda) {
          const double2 vc = S.v[c], wc = S.w[c];
          double2 z = S.D[lane][c];
          z.x -= (vr.x * wc.x + vr.y * wc.y) + (wr.x * vc.x + wr.y * vc.y);
          z.y -= (vr.y * wc.x - vr.x * wc.y) + (wr.y * vc.x - wr.x * vc.y);
          if (c == lane) z.y = 0.0;
          if (c <= lane) *dst = z;
        }
      }
      if (lb > 0) {
        if (!DUAL) {  // B into the (now free) tile buffer
          __syncwarp();
          const double2* src = colp + len;
#pragma unroll 4
          for (int c = 0; c < BWc; ++c, src += lda) {
            if (c < len && lane < lb) cp_async16(&S.D[lane][c], src);
            else S.D[lane][c] = zero;
          }
          cp_async_wait_all();
          __syncwarp();
        }
        // ---- B: q = tau B v (lane = row); x0 = column 0 of B - q v^H; H'
        double2 q;
        {
          double2 a0 = zero, a1 = zero;
#pragma unroll 4
          for (int c = 0; c < BWc; c += 2) {
            const double2 x0 = Bt[lane][c], v0 = S.v[c], x1 = Bt[lane][c + 1], v1 = S.v[c + 1];
            a0.x = fma(x0.x, v0.x, fma(-x0.y, v0.y, a0.x));
            a0.y = fma(x0.x, v0.y, fma(x0.y, v0.x, a0.y));
            a1.x = fma(x1.x, v1.x, fma(-x1.y, v1.y, a1.x));
            a1.y = fma(x1.x, v1.y, fma(x1.y, v1.x, a1.y));
          }
          q = make_double2(tau * (a0.x + a1.x), tau * (a0.y + a1.y));
        }
        const double2 b00 = Bt[lane][0];
        const double2 x0 = make_double2(b00.x - q.x, b00.y - q.y);  // (B - q v^H)[r][0], v_0 = 1
        const double sg2 = warp_sum(x0.x * x0.x + x0.y * x0.y);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, x0.x, 0), __shfl_sync(0xffffffffu, x0.y, 0));
        const QuickReflector hp = quick_reflector(al, sg2);
        const double2 vpr = lane == 0 ? make_double2(1.0, 0.0) : cmul(x0, hp.scale);  // zero on padded rows
        S.vp[lane] = vpr;
        const double2 wq = warp_csum_hx(vpr, q);  // v'^H q
        __syncwarp();
        // ---- column pass (lane = column): z_c = tau' (v'^H B[:, c] - wq conj(v_c))
        {
          double2 a0 = zero, a1 = zero;
#pragma unroll 4
          for (int r = 0; r < BWc; r += 2) {
            const double2 p0 = S.vp[r], b0 = Bt[r][lane], p1 = S.vp[r + 1], b1 = Bt[r + 1][lane];
            a0.x = fma(p0.x, b0.x, fma(p0.y, b0.y, a0.x));
            a0.y = fma(p0.x, b0.y, fma(-p0.y, b0.x, a0.y));
            a1.x = fma(p1.x, b1.x, fma(p1.y, b1.y, a1.x));
            a1.y = fma(p1.x, b1.y, fma(-p1.y, b1.x, a1.y));
          }
          const double2 vc = S.v[lane];
          const double2 wv = make_double2(wq.x * vc.x + wq.y * vc.y, wq.y * vc.x - wq.x * vc.y);  // wq conj(v_c)
          S.z[lane] = make_double2(hp.tau * (a0.x + a1.x - wv.x), hp.tau * (a0.y + a1.y - wv.y));
        }
        __syncwarp();
        // ---- B'' = B - q v^H - v' z^T (lane = row), column 0 -> (beta', 0, ...); straight to HBM
        if (lane < lb) {
          double2* dst = colp + len;
#pragma unroll 4
          for (int c = 0; c < BWc; ++c, dst += lda) {
            const double2 vc = S.v[c], zc = S.z[c];
            double2 y = Bt[lane][c];
            y.x -= (q.x * vc.x + q.y * vc.y) + (vpr.x * zc.x - vpr.y * zc.y);
            y.y -= (q.y * vc.x - q.x * vc.y) + (vpr.x * zc.y + vpr.y * zc.x);
            if (c == 0 && hp.tau != 0.0) y = lane == 0 ? hp.beta : zero;
            if (c < len) *dst = y;
          }
        }
        __syncwarp();
        // carry H' to the next task of this sweep
        S.v[lane] = vpr;
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

template <int NW, int BWc, bool DUAL>
constexpr size_t chase_smem_bytes() {
  return NW * sizeof(ChaseWarpSmem<BWc, DUAL>) + 64;
}

// ---------------------------------------------------------------------------------------------------
// Register-row Hermitian chase on a compact lower band (HX_HCHASE_REG, default on) - the complex counterpart of
// sym_chase_realr_kernel (hx_gram.cuh).  Element (r, c), c <= r <= c + 63 (band of width 32 plus the bulge of the
// tile below the diagonal tile) at Bs[c * HB_LD + r - c] (double2): 1 KB per column instead of the 16 N bytes of
// the dense slab, so the bands of a launch stay in L2 and a tile column is one contiguous 512-byte run.  The
// lane's row of the diagonal tile D (lower triangle from the band; the mirrored part through the transposed
// shared-memory copy) and then of the tile B below it live in 32 complex registers; p = D v, q = tau B v and both
// rank-2 updates run on registers, shared memory carries the broadcast vectors and the transposed tile of the
// column pass.  Same tasks, pipeline and progress flags as bulge_chase_pipe_kernel above.
constexpr int HB_LD = 64;

struct __align__(16) HermChaseSmemR {
  double2 v[32], w[32], vp[32], z[32];
  double2 Xt[32][33];  // Xt[c][r] = tile (r, c)
};

// Lower band (width 32) of the leading d x d block of the dense slab A (ld N) into the compact band.
static __global__ void __launch_bounds__(256) herm_band_extract_kernel(double2* ws, size_t stride, size_t a_off,
                                                                        size_t band_off, int N, const int* dims) {
  double2* base = ws + (size_t)blockIdx.x * stride;
  const double2* A = base + a_off;
  double2* B = base + band_off;
  const int d = dims ? dims[blockIdx.x] : N;
  const size_t n = (size_t)N * HB_LD;
  for (size_t p = threadIdx.x; p < n; p += blockDim.x) {
    const int c = (int)(p / HB_LD), j = (int)(p % HB_LD), r = c + j;
    B[p] = (j <= 32 && r < d) ? A[r + (size_t)c * N] : make_double2(0.0, 0.0);
  }
}

__device__ __forceinline__ void warp_sum3(double& a, double& b, double& c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
}

__device__ __forceinline__ double2 lds_c(const double2* p) { return *p; }

template <int NW>
__global__ void __launch_bounds__(NW * 32, NW >= 8 ? 1 : (NW >= 4 ? 2 : (NW >= 2 ? 4 : 8)))
    herm_chase_r_kernel(double2* ws, size_t stride, size_t band_off, size_t dg_off, int N, const int* dims) {
  constexpr int BWc = 32, RS = HB_LD - 1;  // RS: one column to the right along a row
  extern __shared__ __align__(16) unsigned char hcr_raw[];
  HermChaseSmemR* all = reinterpret_cast<HermChaseSmemR*>(hcr_raw);
  volatile int* prog = reinterpret_cast<volatile int*>(all + NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  HermChaseSmemR& W = all[warp];
  double2* base = ws + (size_t)blockIdx.x * stride;
  double2* B = base + band_off;
  double* diag = reinterpret_cast<double*>(base + dg_off);
  double* e2 = diag + N;
  const int d = dims ? dims[blockIdx.x] : N;
  const double2 zero = make_double2(0.0, 0.0);
  if (lane == 0) prog[warp] = -1;
  __syncthreads();
  if (d <= 0) return;
  const int nsweeps = d - 1;
  for (int i = warp; i < nsweeps; i += NW) {
    const int tasks = (d - 1 - i + BWc - 1) / BWc;
    const int prev_tasks = i > 0 ? (d - i + BWc - 1) / BWc : 0;
    volatile int* pflag = prog + (i - 1 + NW) % NW;
    double tau = 0.0;
    double2 vr = zero;
    for (int t = 0; t < tasks; ++t) {
      if (i > 0) {
        const int need = (i - 1) * 65536 + min(t + 2, prev_tasks);
        if (lane == 0)
          while (*pflag < need) __nanosleep(20);
        __syncwarp();
        __threadfence_block();
      }
      const int s = i + 1 + t * BWc;
      const int len = min(BWc, d - s);
      const int lb = max(0, min(BWc, d - s - len));
      double2* const blk = B + ((size_t)s * HB_LD + lane);  // (s + lane, s + c), c <= lane, at blk[c * RS]
      double2 xr[BWc];
      {
        const int nc = lane < len ? lane + 1 : 0;  // lower triangle of the diagonal tile
#pragma unroll
        for (int cc = 0; cc < BWc; ++cc) xr[cc] = cc < nc ? blk[cc * RS] : zero;
      }
      if (t == 0) {
        // reflector from column i, rows [s, s + len): column i -> (beta, 0, ...)
        double2* const coli = B + ((size_t)i * HB_LD + 1 + lane);  // (s + lane, i)
        const double2 x = lane < len ? *coli : zero;
        const double sig2 = warp_sum(x.x * x.x + x.y * x.y);
        const double2 alpha = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
        const QuickReflector h = quick_reflector(alpha, sig2);
        tau = h.tau;
        vr = lane == 0 ? make_double2(1.0, 0.0) : (lane < len ? cmul(x, h.scale) : zero);
        W.v[lane] = vr;
        if (lane < len && tau != 0.0) *coli = lane == 0 ? h.beta : zero;
        if (lane == 0) {
          diag[i] = B[(size_t)i * HB_LD].x;
          e2[i] = sig2;
        }
      }
#pragma unroll
      for (int cc = 0; cc < BWc; ++cc) W.Xt[cc][lane] = xr[cc];
      __syncwarp();
      // mirrored part of the lane's row: D[lane][c] = conj(D[c][lane]) for c > lane
#pragma unroll
      for (int cc = 1; cc < BWc; ++cc)
        if (cc > lane) {
          const double2 u = W.Xt[lane][cc];
          xr[cc] = make_double2(u.x, -u.y);
        }
      // ---- p = D v (registers), cval = v^H p, w = tau p - tau^2/2 cval v
      double2 p;
      {
        double2 a0 = zero, a1 = zero;
#pragma unroll
        for (int c = 0; c < BWc; c += 2) {
          const double2 v0 = lds_c(&W.v[c]), v1 = lds_c(&W.v[c + 1]);
          a0.x = fma(xr[c].x, v0.x, fma(-xr[c].y, v0.y, a0.x));
          a0.y = fma(xr[c].x, v0.y, fma(xr[c].y, v0.x, a0.y));
          a1.x = fma(xr[c + 1].x, v1.x, fma(-xr[c + 1].y, v1.y, a1.x));
          a1.y = fma(xr[c + 1].x, v1.y, fma(xr[c + 1].y, v1.x, a1.y));
        }
        p = make_double2(a0.x + a1.x, a0.y + a1.y);
      }
      const double cval = warp_sum(vr.x * p.x + vr.y * p.y);
      const double hc = 0.5 * tau * tau * cval;
      const double2 wr = make_double2(tau * p.x - hc * vr.x, tau * p.y - hc * vr.y);
      W.w[lane] = wr;
      __syncwarp();
      // ---- D -= v w^H + w v^H on the lower triangle, straight to the band
      if (lane < len) {
#pragma unroll
        for (int c = 0; c < BWc; ++c) {
          const double2 vc = lds_c(&W.v[c]), wc = lds_c(&W.w[c]);
          double2 zz = xr[c];
          zz.x -= (vr.x * wc.x + vr.y * wc.y) + (wr.x * vc.x + wr.y * vc.y);
          zz.y -= (vr.y * wc.x - vr.x * wc.y) + (wr.y * vc.x - wr.x * vc.y);
          if (c == lane) zz.y = 0.0;
          if (c <= lane) blk[c * RS] = zz;
          if ((c & 7) == 7) asm volatile("" ::: "memory");  // bound the broadcast loads in flight (registers)
        }
      }
      if (lb > 0) {
        // tile below: (s + 32 + lane, s + c) at blk[32 + c * RS] (len == 32 here)
        double2* const blk2 = blk + BWc;
        {
          const bool rowok = lane < lb;
#pragma unroll
          for (int cc = 0; cc < BWc; ++cc) xr[cc] = rowok ? blk2[cc * RS] : zero;
        }
#pragma unroll
        for (int cc = 0; cc < BWc; ++cc) W.Xt[cc][lane] = xr[cc];
        // ---- q = tau B v (registers); x0 = column 0 of B - q v^H; H'
        double2 q;
        {
          double2 a0 = zero, a1 = zero;
#pragma unroll
          for (int c = 0; c < BWc; c += 2) {
            const double2 v0 = lds_c(&W.v[c]), v1 = lds_c(&W.v[c + 1]);
            a0.x = fma(xr[c].x, v0.x, fma(-xr[c].y, v0.y, a0.x));
            a0.y = fma(xr[c].x, v0.y, fma(xr[c].y, v0.x, a0.y));
            a1.x = fma(xr[c + 1].x, v1.x, fma(-xr[c + 1].y, v1.y, a1.x));
            a1.y = fma(xr[c + 1].x, v1.y, fma(xr[c + 1].y, v1.x, a1.y));
          }
          q = make_double2(tau * (a0.x + a1.x), tau * (a0.y + a1.y));
        }
        const double2 x0 = make_double2(xr[0].x - q.x, xr[0].y - q.y);  // (B - q v^H)[r][0], v_0 = 1
        // one reduction round: |x0|^2 and S = sum_{r>=1} conj(x0_r) q_r; v'^H q = q_0 + conj(scale') S
        double sg2 = x0.x * x0.x + x0.y * x0.y;
        double sx = lane == 0 ? 0.0 : x0.x * q.x + x0.y * q.y, sy = lane == 0 ? 0.0 : x0.x * q.y - x0.y * q.x;
        warp_sum3(sg2, sx, sy);
        const double2 al = make_double2(__shfl_sync(0xffffffffu, x0.x, 0), __shfl_sync(0xffffffffu, x0.y, 0));
        const QuickReflector hp = quick_reflector(al, sg2);
        const double2 vpr = lane == 0 ? make_double2(1.0, 0.0) : cmul(x0, hp.scale);  // zero on padded rows
        const double2 q0 = make_double2(__shfl_sync(0xffffffffu, q.x, 0), __shfl_sync(0xffffffffu, q.y, 0));
        // conj(scale') * S
        const double2 wq = make_double2(q0.x + hp.scale.x * sx + hp.scale.y * sy, q0.y + hp.scale.x * sy - hp.scale.y * sx);
        W.vp[lane] = vpr;
        __syncwarp();
        // ---- column pass (lane = column): z_c = tau' (v'^H B[:, c] - wq conj(v_c))
        {
          double2 a0 = zero, a1 = zero;
#pragma unroll
          for (int r = 0; r < BWc; r += 2) {
            const double2 p0 = lds_c(&W.vp[r]), b0 = W.Xt[lane][r], p1 = lds_c(&W.vp[r + 1]), b1 = W.Xt[lane][r + 1];
            a0.x = fma(p0.x, b0.x, fma(p0.y, b0.y, a0.x));
            a0.y = fma(p0.x, b0.y, fma(-p0.y, b0.x, a0.y));
            a1.x = fma(p1.x, b1.x, fma(p1.y, b1.y, a1.x));
            a1.y = fma(p1.x, b1.y, fma(-p1.y, b1.x, a1.y));
          }
          const double2 vc = W.v[lane];
          const double2 wv = make_double2(wq.x * vc.x + wq.y * vc.y, wq.y * vc.x - wq.x * vc.y);  // wq conj(v_c)
          W.z[lane] = make_double2(hp.tau * (a0.x + a1.x - wv.x), hp.tau * (a0.y + a1.y - wv.y));
        }
        __syncwarp();
        // ---- B'' = B - q v^H - v' z^T (registers), column 0 -> (beta', 0, ...); to the band
        if (lane < lb) {
          const bool col0 = hp.tau != 0.0;
#pragma unroll
          for (int c = 0; c < BWc; ++c) {
            const double2 vc = lds_c(&W.v[c]), zc = lds_c(&W.z[c]);
            double2 y = xr[c];
            y.x -= (q.x * vc.x + q.y * vc.y) + (vpr.x * zc.x - vpr.y * zc.y);
            y.y -= (q.y * vc.x - q.x * vc.y) + (vpr.x * zc.y + vpr.y * zc.x);
            if (c == 0 && col0) y = lane == 0 ? hp.beta : zero;
            blk2[c * RS] = y;
            if ((c & 7) == 7) asm volatile("" ::: "memory");
          }
        }
        __syncwarp();  // every lane is done with v
        W.v[lane] = vpr;
        vr = vpr;
        tau = hp.tau;
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[warp] = i * 65536 + t + 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) diag[d - 1] = B[(size_t)(d - 1) * HB_LD].x;
}

template <int NW>
constexpr size_t herm_chase_r_smem() {
  return NW * sizeof(HermChaseSmemR) + 64;
}

}  // namespace hx
