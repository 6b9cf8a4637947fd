// Block-level building blocks of the per-matrix pipeline (one CTA per (mask, k) Bloch matrix):
//   compaction (tbmodel.py:233-239) -> Bloch assembly (tbmodel.py:246-270, _kernels.py:62-65)
//   -> Householder tridiagonalisation (what LAPACK zhetrd does inside zheevd/zhegv)
//   -> Sturm bisection (all eigenvalues) -> IDOS accumulation (_kernels.py:68-101, qoi.py:96-108).
#pragma once
#include <float.h>
#include <stdint.h>

#include "hx_common.cuh"

#define HX_TRI_MAXN 160  // largest dimension handled by tridiag_packed (shared-memory tier)

namespace hx {

// ---------------------------------------------------------------------------------------------
// Block reductions (all threads receive the result). `red` needs 33 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();  // protect red from a previous use
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];  // fixed order: deterministic
  return s;
}

// ---------------------------------------------------------------------------------------------
// Vacancy compaction: new_idx[r] = rank of dof r among kept dofs, -1 if removed.  Returns d.
// `cnt` needs ceil(N/32) ints.  Kept dofs stay in natural order (cumsum(keep)-1).
static __device__ int block_compact(const CellDev& c, const uint64_t* mask, int* new_idx, int* cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nch = (c.N + 31) >> 5;
  for (int ch = warp; ch < nch; ch += nw) {
    const int r = (ch << 5) + lane;
    bool keep = false;
    if (r < c.N) {
      const int u = c.unit_of_dof[r];
      keep = (u < 0) || !((mask[u >> 6] >> (u & 63)) & 1ull);
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) cnt[ch] = __popc(b);
  }
  __syncthreads();
  for (int ch = warp; ch < nch; ch += nw) {
    int off = 0;
    for (int q = 0; q < ch; ++q) off += cnt[q];
    const int r = (ch << 5) + lane;
    bool keep = false;
    if (r < c.N) {
      const int u = c.unit_of_dof[r];
      keep = (u < 0) || !((mask[u >> 6] >> (u & 63)) & 1ull);
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    if (r < c.N) new_idx[r] = keep ? off + __popc(b & ((1u << lane) - 1u)) : -1;
  }
  int d = 0;
  for (int q = 0; q < nch; ++q) d += cnt[q];
  __syncthreads();
  return d;
}

// ---------------------------------------------------------------------------------------------
// Bloch element of one coupling list: acc = sum over instances of row r with target c, in the
// reference's instance order, of amp * (cos(phi) + i sin(phi)), phi = disp . k (_kernels.py:63-65).
__device__ __forceinline__ double2 row_target_sum(const int32_t* ptr, const int32_t* col, const double2* amp,
                                                  const double2* disp, int r, int c, double2 k) {
  double2 acc = make_double2(0.0, 0.0);
  for (int e = ptr[r]; e < ptr[r + 1]; ++e) {
    if (col[e] != c) continue;
    const double2 dv = disp[e];
    const double ph = __dadd_rn(__dmul_rn(dv.x, k.x), __dmul_rn(dv.y, k.y));
    double sn, cs;
    sincos(ph, &sn, &cs);
    const double2 a = amp[e];
    acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(a.x, cs), __dmul_rn(a.y, sn)));
    acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(a.x, sn), __dmul_rn(a.y, cs)));
  }
  return acc;
}

// Hermitian part 0.5*(A + A^H) of the accumulated Bloch sum at compacted (i > j) = dofs (r > c).
__device__ __forceinline__ double2 herm_element(const int32_t* ptr, const int32_t* col, const double2* amp,
                                                const double2* disp, int r, int c, double2 k) {
  const double2 a = row_target_sum(ptr, col, amp, disp, r, c, k);
  const double2 b = row_target_sum(ptr, col, amp, disp, c, r, k);
  return make_double2(0.5 * __dadd_rn(a.x, b.x), 0.5 * __dsub_rn(a.y, b.y));
}

// Visit every distinct partner dof c < r (kept) of row r: own targets, then sources pointing at r.
template <class F>
__device__ __forceinline__ void for_each_lower_partner(const int32_t* ptr, const int32_t* col, const int32_t* tptr,
                                                       const int32_t* tinst, const int32_t* src, const int* new_idx,
                                                       int r, F&& f) {
  const int i = new_idx[r];
  for (int e = ptr[r]; e < ptr[r + 1]; ++e) {
    const int c = col[e];
    if (c >= r || new_idx[c] < 0) continue;
    bool dup = false;
    for (int e2 = ptr[r]; e2 < e; ++e2) dup |= (col[e2] == c);
    if (!dup) f(c, i, new_idx[c]);
  }
  for (int t = tptr[r]; t < tptr[r + 1]; ++t) {
    const int c = src[tinst[t]];
    if (c >= r || new_idx[c] < 0) continue;
    bool dup = false;
    for (int e2 = ptr[r]; e2 < ptr[r + 1]; ++e2) dup |= (col[e2] == c);
    for (int t2 = tptr[r]; t2 < t; ++t2) dup |= (src[tinst[t2]] == c);
    if (!dup) f(c, i, new_idx[c]);
  }
}

// Diagonal value of the assembled operator for kept dof r.
__device__ __forceinline__ double diag_value(const CellDev& c, int r, bool overlap) {
  if (overlap) return 1.0;                      // S diagonal := 1 (tbmodel.py:269)
  if (c.pencil == 1) return 0.0;                // T of the commuting pencil has zero diagonal
  return c.onsite[r];                           // H diagonal := on-site (tbmodel.py:260)
}

// Assemble into real-packed Hermitian storage R (d x d, row stride ld):
//   R[i*ld+k] (i>k) = Re A_ik, R[k*ld+i] = Im A_ik, R[i*ld+i] = A_ii.
static __device__ void assemble_packed(const CellDev& c, const int* new_idx, int d, double2 k, double* R, int ld) {
  for (int p = threadIdx.x; p < d * ld; p += blockDim.x) R[p] = 0.0;
  __syncthreads();
  for (int r = threadIdx.x; r < c.N; r += blockDim.x) {
    const int i = new_idx[r];
    if (i < 0) continue;
    R[i * ld + i] = diag_value(c, r, false);
    for_each_lower_partner(c.h_ptr, c.h_col, c.ht_ptr, c.ht_inst, c.h_src, new_idx, r, [&](int cc, int ii, int jj) {
      const double2 h = herm_element(c.h_ptr, c.h_col, c.h_amp, c.h_disp, r, cc, k);
      R[ii * ld + jj] = h.x;
      R[jj * ld + ii] = h.y;
    });
  }
  __syncthreads();
}

// Assemble into full column-major complex storage A (d x d, leading dim lda), both triangles.
static __device__ void assemble_full(const CellDev& c, const int* new_idx, int d, double2 k, double2* A, int64_t lda,
                              bool overlap) {
  const int32_t* ptr = overlap ? c.s_ptr : c.h_ptr;
  const int32_t* col = overlap ? c.s_col : c.h_col;
  const double2* amp = overlap ? c.s_amp : c.h_amp;
  const double2* disp = overlap ? c.s_disp : c.h_disp;
  const int32_t* tptr = overlap ? c.st_ptr : c.ht_ptr;
  const int32_t* tinst = overlap ? c.st_inst : c.ht_inst;
  const int32_t* src = overlap ? c.s_src : c.h_src;
  for (int64_t p = threadIdx.x; p < (int64_t)d * d; p += blockDim.x) {
    const int64_t col_ = p / d, row = p - col_ * d;
    A[row + col_ * lda] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < c.N; r += blockDim.x) {
    const int i = new_idx[r];
    if (i < 0) continue;
    A[i + (int64_t)i * lda] = make_double2(diag_value(c, r, overlap), 0.0);
    if (ptr == nullptr) continue;
    for_each_lower_partner(ptr, col, tptr, tinst, src, new_idx, r, [&](int cc, int ii, int jj) {
      const double2 h = herm_element(ptr, col, amp, disp, r, cc, k);
      A[ii + (int64_t)jj * lda] = h;
      A[jj + (int64_t)ii * lda] = make_double2(h.x, -h.y);
    });
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// Householder reflector with real tau (Hermitian H = I - tau v v^H, v0 = 1) mapping x (length m,
// x0 = alpha) onto beta e1 with |beta| = sigma.  Returns tau and the complex scale 1/v0.
struct Reflector {
  double tau;
  double2 scale;  // multiply x_i (i >= 1) by this to get v_i
  double e2;      // |beta|^2 = sigma^2: squared off-diagonal of the tridiagonal
};

// Columns whose squared norm is below HX_REFLECTOR_TINY are treated as exactly zero (identity reflector):
// their entries (< 1e-100 for O(1) matrices) are noise left by earlier reflections, and below ~1e-154 the
// squares underflow into the denormal range, where the norm loses its precision and a reflector built
// from it is no longer unitary (tau inconsistent with |v|^2) - measured: 6e-8 loss of unitarity in a
// row panel of a vacancy-rich graphene cell.
#define HX_REFLECTOR_TINY 1e-200

__device__ __forceinline__ Reflector make_reflector(double2 alpha, double sigma2) {
  Reflector h;
  h.e2 = sigma2;
  if (!(sigma2 >= HX_REFLECTOR_TINY)) {
    h.tau = 0.0;
    h.scale = make_double2(0.0, 0.0);
    return h;
  }
  const double sigma = sqrt(sigma2);
  const double aa = hypot(alpha.x, alpha.y);
  double2 ph = aa > 0.0 ? make_double2(alpha.x / aa, alpha.y / aa) : make_double2(1.0, 0.0);
  const double mag = aa + sigma;  // |v0|
  h.tau = mag / sigma;
  // 1/v0 = conj(ph)/mag
  h.scale = make_double2(ph.x / mag, -ph.y / mag);
  return h;
}

// Householder reflector for x with x_0 = alpha, |x|^2 = sig2 (same convention as make_reflector):
// H = I - tau v v^H, v_0 = 1, v_i = x_i * scale, H x = beta e_0, beta = -phase(alpha) sqrt(sig2).
// Division-free (rsqrt + one reciprocal) to keep the chase's critical path and code size short.
struct QuickReflector {
  double tau;
  double2 scale, beta;
};
__device__ __forceinline__ QuickReflector quick_reflector(double2 alpha, double sig2) {
  QuickReflector h;
  if (!(sig2 >= HX_REFLECTOR_TINY)) {
    h.tau = 0.0;
    h.scale = make_double2(0.0, 0.0);
    h.beta = make_double2(0.0, 0.0);
    return h;
  }
  const double a2 = alpha.x * alpha.x + alpha.y * alpha.y;
  if (a2 < 1e-280 && (alpha.x != 0.0 || alpha.y != 0.0)) {
    // (near-)underflow: squares lose their precision / the phase of alpha; divide the careful way
    const double sigma = sqrt(sig2), aa = hypot(alpha.x, alpha.y);
    const double2 ph = aa > 0.0 ? make_double2(alpha.x / aa, alpha.y / aa) : make_double2(1.0, 0.0);
    const double mag = aa + sigma;
    h.tau = mag / sigma;
    h.scale = make_double2(ph.x / mag, -ph.y / mag);
    h.beta = make_double2(-ph.x * sigma, -ph.y * sigma);
    return h;
  }
  const double rs = rsqrt(sig2), sigma = sig2 * rs;
  double2 ph = make_double2(1.0, 0.0);
  double aa = 0.0;
  if (a2 > 0.0) {
    const double ra = rsqrt(a2);
    aa = a2 * ra;
    ph = make_double2(alpha.x * ra, alpha.y * ra);
  }
  const double mag = aa + sigma, rm = __drcp_rn(mag);
  h.tau = mag * rs;
  h.scale = make_double2(ph.x * rm, -ph.y * rm);
  h.beta = make_double2(-ph.x * sigma, -ph.y * sigma);
  return h;
}

// Tridiagonalise the d x d Hermitian matrix held in real-packed storage R (smem), unblocked, with
// three CTA barriers per column: the next column's norm is accumulated while the trailing update is
// applied, the Hermitian matrix-vector product uses P threads per row (shuffle-combined), and the
// rank-2 update forms w = tau*y - hc*v on the fly.  Outputs diag[d] and e2[d-1] (squared
// off-diagonals).  v, y: complex scratch [d] in smem; red: 128 doubles (double-buffered partials).
static __device__ void tridiag_packed(double* R, int ld, int d, double* diag, double* e2, double2* v, double2* y,
                                      double* red) {
  const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = bd >> 5;
  double part = 0.0;
  for (int i = 1 + tid; i < d; i += bd) {
    const double xr = R[i * ld], xi = R[i];
    part += xr * xr + xi * xi;
  }
  int par = 0;
  for (int j = 0; j + 2 < d; ++j) {
    const int b = j + 1, m = d - b;
    double* rb = red + par * 64;
    // ---- B1: column norm (partials accumulated by the previous update sweep)
    part = warp_sum(part);
    if (lane == 0) rb[warp] = part;
    __syncthreads();
    double sig2 = 0.0;
    for (int w = 0; w < nw; ++w) sig2 += rb[w];
    const double2 alpha = make_double2(R[b * ld + j], R[j * ld + b]);
    const Reflector h = make_reflector(alpha, sig2);
    if (tid == 0) {
      diag[j] = R[j * ld + j];
      e2[j] = h.e2;
    }
    par ^= 1;
    if (h.tau == 0.0) {
      // column already reduced: next norm from the unchanged trailing matrix
      part = 0.0;
      for (int i = 1 + tid; i < m; i += bd) {
        const double xr = R[(b + i) * ld + b], xi = R[b * ld + b + i];
        part += xr * xr + xi * xi;
      }
      continue;
    }
    // ---- B2: v (v0 = 1)
    for (int i = tid; i < m; i += bd) {
      const double2 x = make_double2(R[(b + i) * ld + j], R[j * ld + b + i]);
      v[i] = i == 0 ? make_double2(1.0, 0.0) : cmul(x, h.scale);
    }
    __syncthreads();
    // ---- B3: y = A22 v (P threads per row), c = v^H y
    int P = 1;
    while (P < 8 && 2 * P * m <= bd) P *= 2;
    const int rows_per_pass = bd / P;
    double cpart = 0.0;
    for (int row0 = 0; row0 < m; row0 += rows_per_pass) {
      const int i = row0 + tid / P, kp = tid % P;
      double yr0 = 0.0, yi0 = 0.0, yr1 = 0.0, yi1 = 0.0;
      if (i < m) {
        const int gi = b + i;
        int k = kp;
        for (; k + P < m; k += 2 * P) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int kk = k + u * P, gk = b + kk;
            const double p = R[gi * ld + gk], q = R[gk * ld + gi];
            const double re = kk < i ? p : (kk > i ? q : p);
            const double im = kk < i ? q : (kk > i ? -p : 0.0);
            const double2 vk = v[kk];
            if (u == 0) {
              yr0 = fma(re, vk.x, fma(-im, vk.y, yr0));
              yi0 = fma(re, vk.y, fma(im, vk.x, yi0));
            } else {
              yr1 = fma(re, vk.x, fma(-im, vk.y, yr1));
              yi1 = fma(re, vk.y, fma(im, vk.x, yi1));
            }
          }
        }
        if (k < m) {
          const int gk = b + k;
          const double p = R[gi * ld + gk], q = R[gk * ld + gi];
          const double re = k < i ? p : (k > i ? q : p);
          const double im = k < i ? q : (k > i ? -p : 0.0);
          const double2 vk = v[k];
          yr0 = fma(re, vk.x, fma(-im, vk.y, yr0));
          yi0 = fma(re, vk.y, fma(im, vk.x, yi0));
        }
      }
      double yr = yr0 + yr1, yim = yi0 + yi1;
      for (int o = 1; o < P; o <<= 1) {
        yr += __shfl_xor_sync(0xffffffffu, yr, o);
        yim += __shfl_xor_sync(0xffffffffu, yim, o);
      }
      if (kp == 0 && i < m) {
        y[i] = make_double2(yr, yim);
        const double2 vi = v[i];
        cpart += vi.x * yr + vi.y * yim;
      }
    }
    cpart = warp_sum(cpart);
    if (lane == 0) rb[32 + warp] = cpart;
    __syncthreads();
    double cval = 0.0;
    for (int w = 0; w < nw; ++w) cval += rb[32 + w];
    const double hc = 0.5 * h.tau * h.tau * cval;
    const double tau = h.tau;
    // ---- update A22 -= v w^H + w v^H (w = tau y - hc v), accumulating the next column's norm
    // Position (i, k) of the packed array holds Re A_ik (i >= k) or Im A_ki (i < k); with
    // a = v_i conj(w_k) + w_i conj(v_k) the update is R -= Re(a) (i >= k) or R += Im(a) (i < k), i.e.
    // R -= vi.x*X1 + vi.y*X2 + wi.x*X3 + wi.y*X4 with X = (wk.x, wk.y, vk.x, vk.y) or
    // (wk.y, -wk.x, vk.y, -vk.x).  Each lane keeps its columns' (v_k, w_k) in registers.
    part = 0.0;
    constexpr int KC = (HX_TRI_MAXN + 31) / 32;
    double2 vks[KC], wks[KC];
#pragma unroll
    for (int t = 0; t < KC; ++t) {
      const int k = lane + 32 * t;
      const double2 vk = k < m ? v[k] : make_double2(0.0, 0.0);
      const double2 yk = k < m ? y[k] : make_double2(0.0, 0.0);
      vks[t] = vk;
      wks[t] = make_double2(tau * yk.x - hc * vk.x, tau * yk.y - hc * vk.y);
    }
    for (int i = warp; i < m; i += nw) {
      const double2 vi = v[i], yi = y[i];
      const double2 wi = make_double2(tau * yi.x - hc * vi.x, tau * yi.y - hc * vi.y);
      double* row = R + (b + i) * ld + b;
#pragma unroll
      for (int t = 0; t < KC; ++t) {
        const int k = lane + 32 * t;
        if (k < m) {
          const bool low = i >= k;
          const double2 vk = vks[t], wk = wks[t];
          const double x1 = low ? wk.x : wk.y, x2 = low ? wk.y : -wk.x;
          const double x3 = low ? vk.x : vk.y, x4 = low ? vk.y : -vk.x;
          const double delta = fma(vi.x, x1, fma(vi.y, x2, fma(wi.x, x3, wi.y * x4)));
          const double val = row[k] - delta;
          row[k] = val;
          if ((k == 0 && i >= 1) || (i == 0 && k >= 1)) part = fma(val, val, part);
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (d >= 2) {
      const double xr = R[(d - 1) * ld + d - 2], xi = R[(d - 2) * ld + d - 1];
      diag[d - 2] = R[(d - 2) * ld + d - 2];
      e2[d - 2] = xr * xr + xi * xi;
    }
    diag[d - 1] = R[(d - 1) * ld + d - 1];
  }
  __syncthreads();
}

// Same on full column-major complex storage in global memory (both triangles kept current).
static __device__ void tridiag_full(double2* A, int64_t lda, int d, double* diag, double* e2, double2* v, double2* y,
                             double* red) {
  const int tid = threadIdx.x, bd = blockDim.x;
  for (int j = 0; j + 2 < d; ++j) {
    const int b = j + 1, m = d - b;
    double2* col = A + (int64_t)j * lda + b;
    double part = 0.0;
    for (int i = tid; i < m; i += bd) {
      const double2 x = col[i];
      part += x.x * x.x + x.y * x.y;
    }
    const double sig2 = block_sum(part, red);
    const double2 alpha = col[0];
    const Reflector h = make_reflector(alpha, sig2);
    if (tid == 0) {
      diag[j] = A[j + (int64_t)j * lda].x;
      e2[j] = h.e2;
    }
    if (h.tau == 0.0) {
      __syncthreads();
      continue;
    }
    for (int i = tid; i < m; i += bd) v[i] = i == 0 ? make_double2(1.0, 0.0) : cmul(col[i], h.scale);
    __syncthreads();
    double cpart = 0.0;
    double2* A22 = A + (int64_t)b * lda + b;
    for (int i = tid; i < m; i += bd) {
      double yr = 0.0, yim = 0.0;
      for (int k = 0; k < m; ++k) {
        const double2 a = A22[i + (int64_t)k * lda];
        const double2 vk = v[k];
        yr += a.x * vk.x - a.y * vk.y;
        yim += a.x * vk.y + a.y * vk.x;
      }
      y[i] = make_double2(yr, yim);
      const double2 vi = v[i];
      cpart += vi.x * yr + vi.y * yim;
    }
    const double cval = block_sum(cpart, red);
    const double hc = 0.5 * h.tau * h.tau * cval;
    for (int i = tid; i < m; i += bd) {
      const double2 yi = y[i], vi = v[i];
      y[i] = make_double2(h.tau * yi.x - hc * vi.x, h.tau * yi.y - hc * vi.y);
    }
    __syncthreads();
    // A22 -= v w^H + w v^H ; element (i, k) column-major, i fastest for coalescing
    for (int64_t p = tid; p < (int64_t)m * m; p += bd) {
      const int k = (int)(p / m), i = (int)(p - (int64_t)k * m);
      const double2 vi = v[i], wi = y[i], vk = v[k], wk = y[k];
      // v_i conj(w_k) + w_i conj(v_k)
      const double re = vi.x * wk.x + vi.y * wk.y + wi.x * vk.x + wi.y * vk.y;
      const double im = (vi.y * wk.x - vi.x * wk.y) + (wi.y * vk.x - wi.x * vk.y);
      double2 a = A22[i + (int64_t)k * lda];
      a.x -= re;
      a.y -= im;
      A22[i + (int64_t)k * lda] = a;
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (d >= 2) {
      const double2 x = A[(d - 1) + (int64_t)(d - 2) * lda];
      diag[d - 2] = A[(d - 2) + (int64_t)(d - 2) * lda].x;
      e2[d - 2] = x.x * x.x + x.y * x.y;
    }
    diag[d - 1] = A[(d - 1) + (int64_t)(d - 1) * lda].x;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// Sturm count: number of eigenvalues of the symmetric tridiagonal (diag, e2) strictly below x
// (LAPACK dlaebz-style recurrence with pivmin safeguard).
__device__ __forceinline__ int sturm_count(const double* diag, const double* e2, int d, double x, double pivmin) {
  double q = diag[0] - x;
  if (fabs(q) <= pivmin) q = -pivmin;
  int cnt = q < 0.0;
  for (int i = 1; i < d; ++i) {
    q = (diag[i] - x) - e2[i - 1] / q;
    if (fabs(q) <= pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// 1/q to full double precision without the division routine: MUFU reciprocal seed + two Newton steps.
// |q| >= pivmin = DBL_MIN * max(1, max e2) keeps q normal and e2/q finite (dstebz's pivmin argument).
__device__ __forceinline__ double sturm_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = fma(r, fma(-q, r, 1.0), r);
  r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

// Sturm count (number of eigenvalues < x); ZD: zero diagonal (TGK matrix).
//
// HX_STURM_POLY (default): the scaled determinant recurrence P_i = (a_i - x) P_{i-1} - e2_{i-1} P_{i-2}
// (P_{-1} = 1); the count is the number of sign changes P_{i-1} -> P_i, i.e. of negative q_i = P_i / P_{i-1} of
// the dstebz recurrence.  The dependency chain is ONE fused multiply-add per row (the product e2 P_{i-2} is off
// the chain) instead of a reciprocal with two Newton steps plus an fma (~10x the latency, ~2x the FP64
// instructions); every 4 rows both values are rescaled by an exact power of two (max in [1, 2): no overflow for
// any row growth factor below 1e75, signs untouched).  An exact zero P_i takes the role of dstebz's q = -pivmin:
// it is replaced by -2^-200 P_{i-1}, counted as negative, and P_{i+1} = -e2 P_{i-1} + ... restarts the sequence.
#ifndef HX_STURM_POLY
#define HX_STURM_POLY 1
#endif

// Scale so that max(|p0|, |p1|) is in [1, 2): sc = 2^(1023 - E) from the exponent field of the maximum.
__device__ __forceinline__ double sturm_scale_of(double p0, double p1) {
  const int hi = __double2hiint(fmax(fabs(p0), fabs(p1)));
  return __hiloint2double(0x7fe00000 - (hi & 0x7ff00000), 0);
}

// 1 if a and b have different signs (sign bits).
__device__ __forceinline__ int sturm_sign_change(double a, double b) {
  return (int)((unsigned)(__double2hiint(a) ^ __double2hiint(b)) >> 31);
}

template <bool ZD>
__device__ __forceinline__ int sturm_count_fast(const double* __restrict__ diag, const double* __restrict__ e2, int d,
                                                double x, double pivmin) {
#if HX_STURM_POLY
  (void)pivmin;
  double p1 = 1.0, p0 = (ZD ? 0.0 : diag[0]) - x;
  if (p0 == 0.0) p0 = -0x1p-200;
  int cnt = p0 < 0.0;
  for (int i = 1; i < d; ++i) {
    const double ep = e2[i - 1] * p1;
    double pn = fma((ZD ? 0.0 : diag[i]) - x, p0, -ep);
    if (pn == 0.0) pn = -0x1p-200 * p0;
    cnt += sturm_sign_change(pn, p0);
    p1 = p0;
    p0 = pn;
    if ((i & 3) == 0) {
      const double sc = sturm_scale_of(p0, p1);
      p0 *= sc;
      p1 *= sc;
    }
  }
  return cnt;
#else
  double q = (ZD ? 0.0 : diag[0]) - x;
  if (fabs(q) <= pivmin) q = -pivmin;
  int cnt = q < 0.0;
  for (int i = 1; i < d; ++i) {
    q = fma(-e2[i - 1], sturm_rcp(q), (ZD ? 0.0 : diag[i]) - x);
    if (fabs(q) <= pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
#endif
}

// All eigenvalues of the tridiagonal by bisection to ~2 ulp; out[idx] ascending.  red: 96 doubles.
static __device__ void bisect_all(const double* diag, const double* e2, int d, double* out, double* red) {
  const int tid = threadIdx.x, bd = blockDim.x;
  double lo_p = DBL_MAX, hi_p = -DBL_MAX, emax = 0.0;
  for (int i = tid; i < d; i += bd) {
    const double el = i > 0 ? sqrt(e2[i - 1]) : 0.0;
    const double er = i + 1 < d ? sqrt(e2[i]) : 0.0;
    lo_p = fmin(lo_p, diag[i] - el - er);
    hi_p = fmax(hi_p, diag[i] + el + er);
    if (i + 1 < d) emax = fmax(emax, e2[i]);
  }
  // block min/max via the sum helper pattern
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  lo_p = warp_min(lo_p);
  hi_p = warp_max(hi_p);
  emax = warp_max(emax);
  __syncthreads();
  if (lane == 0) {
    red[warp] = lo_p;
    red[32 + warp] = hi_p;
    red[64 + warp] = emax;
  }
  __syncthreads();
  double gl = DBL_MAX, gu = -DBL_MAX, em = 0.0;
  for (int w = 0; w < nw; ++w) {
    gl = fmin(gl, red[w]);
    gu = fmax(gu, red[32 + w]);
    em = fmax(em, red[64 + w]);
  }
  const double pivmin = DBL_MIN * fmax(1.0, em);
  const double tnorm = fmax(fabs(gl), fabs(gu));
  const double ulp = DBL_EPSILON;
  gl = gl - 2.1 * tnorm * ulp * d - 4.2 * pivmin;
  gu = gu + 2.1 * tnorm * ulp * d + 4.2 * pivmin;
  for (int idx = tid; idx < d; idx += bd) {
    double lo = gl, hi = gu;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      const double tol = 2.0 * ulp * fmax(fabs(lo), fabs(hi)) + pivmin;
      if (hi - lo <= tol || mid <= lo || mid >= hi) break;
      if (sturm_count(diag, e2, d, mid, pivmin) > idx) hi = mid;
      else lo = mid;
    }
    out[idx] = 0.5 * (lo + hi);
  }
  __syncthreads();
}

// Map eigenvalues of T through the commuting pencil and return them ascending in `out`.
__device__ __forceinline__ double pencil_map(const CellDev& c, double lam) {
  if (c.pencil != 1) return lam;
  return (c.eps0 + c.t * lam) / (1.0 + c.s * lam);
}

// ---------------------------------------------------------------------------------------------
// IDOS contribution of one state energy E (unit weight) to the per-sample accumulators:
// diff[lo] += 1 (full weight for m >= lo) and fixed-point g(x) for the transition band,
// with the reference's index arithmetic (_kernels.py:68-88): lo = ceil((E + delta - e0)/step),
// m0 = floor((E - delta - e0)/step) + 1, x = (E - (e0 + step*m))/delta, g = 0.5 + x(-1.125 + 0.625x^2).
__device__ __forceinline__ void idos_state(const GridDev& g, double E, int* diff, unsigned long long* trans,
                                           int mult = 1) {
  const double ulo = __ddiv_rn(__dsub_rn(__dadd_rn(E, g.delta), g.e0), g.step);
  long long lo = (long long)ceil(ulo);
  if (lo < 0) lo = 0;
  if (lo < g.npts) atomicAdd(diff + lo, mult);
  const double um0 = __ddiv_rn(__dsub_rn(__dsub_rn(E, g.delta), g.e0), g.step);
  long long m0 = (long long)floor(um0) + 1;
  if (m0 < 0) m0 = 0;
  const long long m1 = lo < g.npts ? lo : g.npts;
  const double scale = ldexp(1.0, g.shift);
  for (long long m = m0; m < m1; ++m) {
    const double em = __dadd_rn(g.e0, __dmul_rn(g.step, (double)m));
    const double x = __ddiv_rn(__dsub_rn(E, em), g.delta);
    const double gx = __dadd_rn(0.5, __dmul_rn(x, __dadd_rn(-1.125, __dmul_rn(__dmul_rn(0.625, x), x))));
    const long long fx = __double2ll_rn(gx * scale);
    atomicAdd(trans + m, (unsigned long long)(fx * mult));
  }
}

// Sharp count contribution: weight at m >= floor((E - e0)/step) + 1 (_kernels.py:91-101).
__device__ __forceinline__ void sharp_state(const GridDev& g, double E, int* diff, int mult = 1) {
  long long idx = (long long)floor(__ddiv_rn(__dsub_rn(E, g.e0), g.step)) + 1;
  if (idx < 0) idx = 0;
  if (idx < g.npts) atomicAdd(diff + idx, mult);
}

// ---------------------------------------------------------------------------------------------
// General pencil: S (in B) = L L^H (lower, in place), A <- L^-1 A L^-H.  Returns false if S is not PD.
static __device__ __noinline__ bool chol_reduce_full(double2* A, double2* B, int64_t lda, int d, double* red) {
  __shared__ int not_pd;
  if (threadIdx.x == 0) not_pd = 0;
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    const double s = B[j + (int64_t)j * lda].x;
    if (!(s > 0.0) || !isfinite(s)) {
      if (threadIdx.x == 0) not_pd = 1;
      break;
    }
    const double ljj = sqrt(s);
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < d; i += blockDim.x) {
      double2 b = B[i + (int64_t)j * lda];
      B[i + (int64_t)j * lda] = make_double2(b.x / ljj, b.y / ljj);
    }
    if (threadIdx.x == 0) B[j + (int64_t)j * lda] = make_double2(ljj, 0.0);
    __syncthreads();
    const int m = d - j - 1;
    for (int64_t p = threadIdx.x; p < (int64_t)m * m; p += blockDim.x) {
      const int kq = (int)(p / m), iq = (int)(p - (int64_t)kq * m);
      if (iq < kq) continue;
      const int i = j + 1 + iq, k = j + 1 + kq;
      const double2 li = B[i + (int64_t)j * lda], lk = B[k + (int64_t)j * lda];
      double2 b = B[i + (int64_t)k * lda];
      // b -= li * conj(lk)
      b.x -= li.x * lk.x + li.y * lk.y;
      b.y -= li.y * lk.x - li.x * lk.y;
      B[i + (int64_t)k * lda] = b;
    }
    __syncthreads();
  }
  __syncthreads();
  if (not_pd) return false;
  // X = L^-1 A (forward substitution per column)
  for (int col = threadIdx.x; col < d; col += blockDim.x) {
    double2* x = A + (int64_t)col * lda;
    for (int i = 0; i < d; ++i) {
      double2 acc = x[i];
      for (int k = 0; k < i; ++k) {
        const double2 l = B[i + (int64_t)k * lda], xk = x[k];
        acc.x -= l.x * xk.x - l.y * xk.y;
        acc.y -= l.x * xk.y + l.y * xk.x;
      }
      const double lii = B[i + (int64_t)i * lda].x;
      x[i] = make_double2(acc.x / lii, acc.y / lii);
    }
  }
  __syncthreads();
  // A <- A^H (in place conjugate transpose)
  for (int64_t p = threadIdx.x; p < (int64_t)d * d; p += blockDim.x) {
    const int k = (int)(p / d), i = (int)(p - (int64_t)k * d);
    if (i > k) {
      const double2 a = A[i + (int64_t)k * lda], b = A[k + (int64_t)i * lda];
      A[i + (int64_t)k * lda] = make_double2(b.x, -b.y);
      A[k + (int64_t)i * lda] = make_double2(a.x, -a.y);
    } else if (i == k) {
      A[i + (int64_t)i * lda].y = -A[i + (int64_t)i * lda].y;
    }
  }
  __syncthreads();
  for (int col = threadIdx.x; col < d; col += blockDim.x) {
    double2* x = A + (int64_t)col * lda;
    for (int i = 0; i < d; ++i) {
      double2 acc = x[i];
      for (int k = 0; k < i; ++k) {
        const double2 l = B[i + (int64_t)k * lda], xk = x[k];
        acc.x -= l.x * xk.x - l.y * xk.y;
        acc.y -= l.x * xk.y + l.y * xk.x;
      }
      const double lii = B[i + (int64_t)i * lda].x;
      x[i] = make_double2(acc.x / lii, acc.y / lii);
    }
  }
  __syncthreads();
  // Hermitian part (the reduced matrix is Hermitian up to rounding)
  for (int64_t p = threadIdx.x; p < (int64_t)d * d; p += blockDim.x) {
    const int k = (int)(p / d), i = (int)(p - (int64_t)k * d);
    if (i > k) {
      const double2 a = A[i + (int64_t)k * lda], b = A[k + (int64_t)i * lda];
      const double2 h = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
      A[i + (int64_t)k * lda] = h;
      A[k + (int64_t)i * lda] = make_double2(h.x, -h.y);
    } else if (i == k) {
      A[i + (int64_t)i * lda].y = 0.0;
    }
  }
  __syncthreads();
  return true;
}

}  // namespace hx
