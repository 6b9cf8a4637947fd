// Gram path of the shared-memory bipartite tier (graphene, sublattice size S in (32, 64], IDOS only):
// sigma(C)^2 are the eigenvalues of G = C^H C (n x n, n = min(nA, nB)), so ONE Hermitian tridiagonalisation of G
// replaces the Golub-Kahan bidiagonalisation of C (hx_bidiag.cuh bidiag_tgk_reg): one reflector and two CTA
// barriers per step instead of two reflectors and four barriers, 48 instead of 64 complex FMAs per thread and
// step, and a tridiagonal of dimension S instead of the TGK's 2 S for the Sturm counts.  The eigenvalue stage is
// the mu = sigma^2 zone path of the banded Gram tier (launch_gram_idos, hx_kernels.cu); the host takes this
// path under the same condition (gram_zones_ok: no transition zone of the energy grid near lambda = 0).
// Replaces for these batches the eigenvalue solve of the reference's per-sample job (spectrum.py:100-117 through
// runner.py:114-129).
//
// Layout: 256 threads, thread (a, b) = (lane & 15, 2 warp + (lane >> 4)) owns the 4 x 4 elements
// G[a + 16 i][b + 16 k] (cyclic: the active trailing block stays spread over every thread).  G is formed in
// registers from the sparse columns of the dense C in shared memory (<= SG_NZ nonzeros per column: the kept
// neighbours of a site).  Step j (column j, rows j + 1 ..):
//   owners of column j (one half-warp) build v, tau;                                   barrier A
//   s_c = v^H G[:, c] by 16 register FMAs + a reduce-scatter over the 16 lanes a (shuffles); p = tau conj(s)
//   (G Hermitian), the half-warp's part of v^H p;                                      barrier B
//   w = p - (tau / 2)(v^H p) v;  G -= v w^H + w v^H on registers.
// Phases T = j / 16 are templated: register blocks i < T, k < T are finished and skipped statically.
#pragma once
#include "hx_bidiag.cuh"

namespace hx {

constexpr int SG_NZ = 3;  // nonzeros kept per column of C (honeycomb: <= 3 distinct neighbours)

template <bool REAL>
struct SgElem {
  using E = double2;
};
template <>
struct SgElem<true> {
  using E = double;
};

__device__ __forceinline__ double sg_zero(double) { return 0.0; }
__device__ __forceinline__ double2 sg_zero(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double sg_one(double) { return 1.0; }
__device__ __forceinline__ double2 sg_one(double2) { return make_double2(1.0, 0.0); }
__device__ __forceinline__ double sg_norm2(double x) { return x * x; }
__device__ __forceinline__ double sg_norm2(double2 x) { return fma(x.x, x.x, x.y * x.y); }
__device__ __forceinline__ bool sg_nonzero(double x) { return x != 0.0; }
__device__ __forceinline__ bool sg_nonzero(double2 x) { return x.x != 0.0 || x.y != 0.0; }
__device__ __forceinline__ double sg_real(double x) { return x; }
__device__ __forceinline__ double sg_real(double2 x) { return x.x; }
// acc += conj(u) x
__device__ __forceinline__ void sg_acc_cj(double& acc, double u, double x) { acc = fma(u, x, acc); }
__device__ __forceinline__ void sg_acc_cj(double2& acc, double2 u, double2 x) {
  acc.x = fma(u.x, x.x, fma(u.y, x.y, acc.x));
  acc.y = fma(u.x, x.y, fma(-u.y, x.x, acc.y));
}
// x -= v conj(w)
__device__ __forceinline__ void sg_sub_cj(double& x, double v, double w) { x = fma(-v, w, x); }
__device__ __forceinline__ void sg_sub_cj(double2& x, double2 v, double2 w) {
  x.x = fma(-v.x, w.x, fma(-v.y, w.y, x.x));
  x.y = fma(-v.y, w.x, fma(v.x, w.y, x.y));
}
// p - h v (h real)
__device__ __forceinline__ double sg_axpy(double p, double h, double v) { return fma(-h, v, p); }
__device__ __forceinline__ double2 sg_axpy(double2 p, double h, double2 v) {
  return make_double2(fma(-h, v.x, p.x), fma(-h, v.y, p.y));
}
// Re(conj(v) p)
__device__ __forceinline__ double sg_redot(double v, double p) { return v * p; }
__device__ __forceinline__ double sg_redot(double2 v, double2 p) { return fma(v.x, p.x, v.y * p.y); }

__device__ __forceinline__ double sg_shfl(double x, int src) { return __shfl_sync(0xffffffffu, x, src); }
__device__ __forceinline__ double2 sg_shfl(double2 x, int src) {
  return make_double2(__shfl_sync(0xffffffffu, x.x, src), __shfl_sync(0xffffffffu, x.y, src));
}

struct SgReflR {
  double tau, scale;
};
// real reflector for x with x_0 = alpha, |x|^2 = sig2: H = I - tau v v^T, v_0 = 1, v_i = x_i scale (the real
// form of quick_reflector, hx_dense.cuh)
__device__ __forceinline__ SgReflR sg_reflector(double alpha, double sig2) {
  if (!(sig2 >= HX_REFLECTOR_TINY)) return SgReflR{0.0, 0.0};
  const double aa = fabs(alpha), ph = alpha < 0.0 ? -1.0 : 1.0;
  if (aa * aa < 1e-280 && alpha != 0.0) {
    const double sigma = sqrt(sig2), mag = aa + sigma;
    return SgReflR{mag / sigma, ph / mag};
  }
  const double rs = rsqrt(sig2), sigma = sig2 * rs, mag = aa + sigma;
  return SgReflR{mag * rs, ph * __drcp_rn(mag)};
}
struct SgReflC {
  double tau;
  double2 scale;
};
__device__ __forceinline__ SgReflC sg_reflector(double2 alpha, double sig2) {
  const QuickReflector h = quick_reflector(alpha, sig2);
  return SgReflC{h.tau, h.scale};
}
__device__ __forceinline__ double sg_scale(double x, double s) { return x * s; }
__device__ __forceinline__ double2 sg_scale(double2 x, double2 s) { return cmul(x, s); }

// scratch (doubles): v [64 E], p [64 E], tau, 16 dot partials
template <bool REAL>
constexpr int sg_scratch_doubles() {
  return (REAL ? 64 : 128) * 2 + 2 + 16;
}

template <bool REAL>
struct SgScratch {
  using E = typename SgElem<REAL>::E;
  E* vbuf;
  E* pbuf;
  double* stau;
  double* dbuf;
};

template <bool REAL, int T>
static __device__ __forceinline__ void sg_phase(typename SgElem<REAL>::E (&m)[4][4], int n, double* diag, double* e2,
                                                const SgScratch<REAL>& sc) {
  using E = typename SgElem<REAL>::E;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane & 15, hb = lane >> 4, b = 2 * warp + hb;
  const unsigned FULL = 0xffffffffu;
  constexpr int T1 = T < 3 ? T + 1 : 3;
  const int jend = min(16 * T + 16, n - 1);
  for (int j = 16 * T; j < jend; ++j) {
    const int jl = j & 15;
    // ---------------- reflector from column j, rows j + 1 .. (owners: b == jl, one half-warp of warp jl >> 1)
    if (warp == (jl >> 1)) {
      double part = 0.0;
#pragma unroll
      for (int i = T; i < 4; ++i)
        if (i > T || a > jl) part += sg_norm2(m[i][T]);
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) part += __shfl_xor_sync(FULL, part, o);
      const int r1 = j + 1;
      const int src = 16 * (jl & 1) + (r1 & 15);
      const E alpha = sg_shfl((r1 >> 4) == T ? m[T][T] : m[T1][T], src);
      const auto h = sg_reflector(alpha, part);
      if (hb == (jl & 1)) {
#pragma unroll
        for (int i = T; i < 4; ++i) {
          const int r = a + 16 * i;
          sc.vbuf[r] = r <= j ? sg_zero(E{}) : (r == r1 ? sg_one(E{}) : sg_scale(m[i][T], h.scale));
        }
        if (a == jl) {
          *sc.stau = h.tau;
          e2[j] = part;
          diag[j] = sg_real(m[T][T]);
        }
      }
    }
    __syncthreads();  // A: v, tau
    const double tau = *sc.stau;
    E vr[4], vc[4], pc[4];
#pragma unroll
    for (int i = T; i < 4; ++i) vr[i] = sc.vbuf[a + 16 * i];
#pragma unroll
    for (int k = T; k < 4; ++k) vc[k] = sc.vbuf[b + 16 * k];
    {
      // s_c = sum_r conj(v_r) G[r][c] over the thread's rows, then over the 16 lanes a of the half-warp
      constexpr int NV = REAL ? 4 : 8;
      double v[NV];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        E acc = sg_zero(E{});
        if (k >= T)
#pragma unroll
          for (int i = T; i < 4; ++i) sg_acc_cj(acc, vr[i], m[i][k]);
        if constexpr (REAL) {
          v[k] = acc;
        } else {
          v[2 * k] = acc.x;
          v[2 * k + 1] = acc.y;
        }
      }
      const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
      if constexpr (REAL) {
        // 4 values: the lane ends with the sum of value (a >> 2) & 3 = column class k
        double w2[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) w2[t] = (b3 ? v[t + 2] : v[t]) + __shfl_xor_sync(FULL, b3 ? v[t] : v[t + 2], 8);
        double w1 = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(FULL, b2 ? w2[0] : w2[1], 4);
        w1 += __shfl_xor_sync(FULL, w1, 2);
        w1 += __shfl_xor_sync(FULL, w1, 1);
        if (!(a & 3)) {
          const int c = b + 16 * (a >> 2);
          sc.pbuf[c] = c > j ? tau * w1 : 0.0;
        }
      } else {
        // 8 values: the lane ends with the sum of value (a >> 1) & 7 = (column class, re / im)
        double w4[4], w2[2];
#pragma unroll
        for (int t = 0; t < 4; ++t) w4[t] = (b3 ? v[t + 4] : v[t]) + __shfl_xor_sync(FULL, b3 ? v[t] : v[t + 4], 8);
#pragma unroll
        for (int t = 0; t < 2; ++t)
          w2[t] = (b2 ? w4[t + 2] : w4[t]) + __shfl_xor_sync(FULL, b2 ? w4[t] : w4[t + 2], 4);
        double w1 = (b1 ? w2[1] : w2[0]) + __shfl_xor_sync(FULL, b1 ? w2[0] : w2[1], 2);
        w1 += __shfl_xor_sync(FULL, w1, 1);
        if (!(a & 1)) {
          const int p = a >> 1, c = b + 16 * (p >> 1);
          // p_c = tau conj(s_c)
          reinterpret_cast<double*>(sc.pbuf)[2 * c + (p & 1)] = c > j ? ((p & 1) ? -tau * w1 : tau * w1) : 0.0;
        }
      }
      __syncwarp();
      double dot = 0.0;
#pragma unroll
      for (int k = T; k < 4; ++k) {
        pc[k] = sc.pbuf[b + 16 * k];
        dot += sg_redot(vc[k], pc[k]);
      }
      if (a == 0) sc.dbuf[b] = dot;
    }
    __syncthreads();  // B: p, dot partials
    {
      const double2* d2 = reinterpret_cast<const double2*>(sc.dbuf);
      double cd[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 x = d2[2 * q], y = d2[2 * q + 1];
        cd[q] = (x.x + x.y) + (y.x + y.y);
      }
      const double cdot = (cd[0] + cd[1]) + (cd[2] + cd[3]);
      const double hc = 0.5 * tau * cdot;
      E wr[4], wc[4];
#pragma unroll
      for (int i = T; i < 4; ++i) wr[i] = sg_axpy(sc.pbuf[a + 16 * i], hc, vr[i]);
#pragma unroll
      for (int k = T; k < 4; ++k) wc[k] = sg_axpy(pc[k], hc, vc[k]);
#pragma unroll
      for (int i = T; i < 4; ++i)
#pragma unroll
        for (int k = T; k < 4; ++k) {
          E x = m[i][k];
          sg_sub_cj(x, vr[i], wc[k]);
          sg_sub_cj(x, wr[i], vc[k]);
          m[i][k] = x;
        }
    }
  }
}

// C (rows x cols, rows >= cols, column-major, ld = lm) in shared memory -> tridiagonal (diag[S], e2[S]) of
// G = C^H C padded with zeros to dimension S.  lrow / lval: scratch lists [64 * SG_NZ].  Returns false when a
// column of C has more than SG_NZ nonzeros (not a nearest-neighbour honeycomb block).
template <bool REAL>
static __device__ bool small_gram_tridiag(const typename SgElem<REAL>::E* Ms, int lm, int rows, int cols, int S,
                                          double* diag, double* e2, double* scratch, int* lrow,
                                          typename SgElem<REAL>::E* lval, int* flag) {
  using E = typename SgElem<REAL>::E;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane & 15, b = 2 * warp + (lane >> 4);
  SgScratch<REAL> sc;
  sc.vbuf = reinterpret_cast<E*>(scratch);
  sc.pbuf = sc.vbuf + 64;
  sc.stau = reinterpret_cast<double*>(sc.pbuf + 64);
  sc.dbuf = sc.stau + 2;
  for (int i = tid; i < 2 * S; i += blockDim.x) diag[i] = 0.0;  // diag and e2 (e2 = diag + S)
  if (tid == 0) *flag = 0;
  __syncthreads();
  // sparse columns of C: four threads per column (16 rows each), merged in row order (deterministic lists)
  {
    const int col = tid & 63, qd = tid >> 6;
    int cnt = 0, xr[SG_NZ];
    E xv[SG_NZ];
#pragma unroll
    for (int q = 0; q < SG_NZ; ++q) {
      xr[q] = 0;
      xv[q] = sg_zero(E{});
    }
    if (col < cols) {
      const int x1 = min(rows, 16 * qd + 16);
      for (int x = 16 * qd; x < x1; ++x) {
        const E val = Ms[x + (size_t)col * lm];
        if (sg_nonzero(val)) {
#pragma unroll
          for (int q = 0; q < SG_NZ; ++q)
            if (q == cnt) {
              xr[q] = x;
              xv[q] = val;
            }
          ++cnt;
        }
      }
    }
    int* qcnt = reinterpret_cast<int*>(scratch);  // [4][64], before the reflector buffers are in use
    qcnt[qd * 64 + col] = cnt;
    for (int q = tid; q < 64 * SG_NZ; q += blockDim.x) {
      lrow[q] = 0;
      lval[q] = sg_zero(E{});
    }
    __syncthreads();
    int off = 0;
    for (int q = 0; q < qd; ++q) off += qcnt[q * 64 + col];
    if (off + cnt > SG_NZ) *flag = 1;
#pragma unroll
    for (int q = 0; q < SG_NZ; ++q)
      if (q < cnt && off + q < SG_NZ) {
        lrow[col * SG_NZ + off + q] = xr[q];
        lval[col * SG_NZ + off + q] = xv[q];
      }
  }
  __syncthreads();
  if (*flag) return false;
  // G[r][c] = sum_x conj(C[x][r]) C[x][c] over the nonzeros x of column r
  E m[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = a + 16 * i;
    int xr[SG_NZ];
    E xv[SG_NZ];
#pragma unroll
    for (int q = 0; q < SG_NZ; ++q) {
      xr[q] = lrow[r * SG_NZ + q];
      xv[q] = lval[r * SG_NZ + q];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = b + 16 * k;
      E acc = sg_zero(E{});
      if (r < cols && c < cols) {
#pragma unroll
        for (int q = 0; q < SG_NZ; ++q) sg_acc_cj(acc, xv[q], Ms[xr[q] + (size_t)c * lm]);
        if constexpr (!REAL)
          if (r == c) acc.y = 0.0;
      }
      m[i][k] = acc;
    }
  }
  const int n = cols;
  sg_phase<REAL, 0>(m, n, diag, e2, sc);
  if (n > 17) sg_phase<REAL, 1>(m, n, diag, e2, sc);
  if (n > 33) sg_phase<REAL, 2>(m, n, diag, e2, sc);
  if (n > 49) sg_phase<REAL, 3>(m, n, diag, e2, sc);
  // last diagonal element
  if (n >= 1) {
    const int r = n - 1, ib = r >> 4;
    if (a == (r & 15) && b == (r & 15)) {
      double dv = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i == ib) dv = sg_real(m[i][i]);
      diag[r] = dv;
    }
  }
  __syncthreads();
  return true;
}

}  // namespace hx
