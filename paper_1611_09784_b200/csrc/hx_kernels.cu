// Per-matrix kernels of the hexmc hot path on sm_100a.
//
//  * small_tridiag_kernel: one CTA per (mask, k) Bloch matrix, everything in shared memory
//    (N <= HX_SMEM_MAX_N): compaction -> assembly -> Householder tridiagonalisation -> (diag, e2).
//  * global_tridiag_kernel: same with the matrix in an HBM workspace slice (fallback tier, and the
//    general (H, S) pencil via Cholesky).  The large-N two-stage path lives in hx_band.cu.
//  * eig_idos_kernel: one THREAD per eigenvalue of every matrix in the batch (Sturm bisection),
//    pencil map, the reference IDOS functional (fixed-point accumulation) and the eigenvalue output.
//  * finalize_kernel: prefix-sum of the integer full-weight counts + fixed-point transition sums
//    -> per-mask IDOS curves (qoi.py:96-102: values = counts / area, weights 1/nk).
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>

#include <cmath>
#include <stdint.h>

#include "hx_bidiag.cuh"
#include "hx_dense.cuh"
#include "hx_kernels.cuh"
#include "hx_smallgram.cuh"

namespace hx {

static __device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) small_tridiag_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                            const uint64_t* __restrict__ masks, double* tri,
                                                            int* dims, int* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = c.N;
  const int ld = N | 1;  // odd row stride: conflict-free column walks
  const int64_t mat = blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  double* R = reinterpret_cast<double*>(smem_raw);
  double2* v = reinterpret_cast<double2*>(R + (((size_t)N * ld + 1) & ~(size_t)1));
  double2* y = v + N;
  double* red = reinterpret_cast<double*>(y + N);      // 128
  int* new_idx = reinterpret_cast<int*>(red + 128);     // N
  int* cnt = new_idx + N;                              // ceil(N/32)
  double* diag = tri + mat * 2 * N;
  double* e2 = diag + N;

  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (threadIdx.x == 0) {
    dims[mat] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  if (d == 0) return;
  assemble_packed(c, new_idx, d, kpts[kk], R, ld);
  tridiag_packed(R, ld, d, diag, e2, v, y, red);
}

// Bipartite (graphene) variant: bidiagonalise the nA x nB block C instead of tridiagonalising T.
// klist (optional): this launch covers the k-points klist[0..nks) of every mask (block = mask * nks + i),
// written at the batch's matrix index mask * nk + klist[i].  real: those k-points make the periodic-gauge
// block exactly real (hx_capi k_is_real) - real Golub-Kahan on doubles (bidiag_tgk(_warp)_real).
__global__ void __launch_bounds__(256) small_bidiag_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                           const uint64_t* __restrict__ masks, double* tri, int* dims,
                                                           int* status, const int* __restrict__ klist, int nks,
                                                           int real) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = c.N, S = c.nsub;
  int64_t mk, mat;
  int kk;
  if (klist) {
    mk = blockIdx.x / nks;
    kk = klist[blockIdx.x - mk * nks];
    mat = mk * nk + kk;
  } else {
    mat = blockIdx.x;
    mk = mat / nk;
    kk = (int)(mat - mk * nk);
  }
  const int lm = real ? (blockDim.x == 32 ? bidiag_ld_real_warp(S) : bidiag_ld_real(S)) : bidiag_ld(S);
  double2* M = reinterpret_cast<double2*>(smem_raw);
  double* Mr = reinterpret_cast<double*>(smem_raw);
  double2* u = M + (size_t)lm * S;
  double2* s = u + S + 1;
  double* ur = Mr + (size_t)lm * S;
  double* red = real ? ur + S + 1 : reinterpret_cast<double*>(s + S + 1);  // 128
  int* idx_a = reinterpret_cast<int*>(red + 128);                           // N
  int* idx_b = idx_a + N;                                                   // N
  int* cnt = idx_b + N;                                                     // 2 ceil(N/32)
  double* diag = tri + mat * 2 * N;
  double* e2 = diag + N;
  const int2 nn = block_compact_bipartite(c, masks + mk * c.words, idx_a, idx_b, cnt);
  const int d = nn.x + nn.y;
  if (threadIdx.x == 0) {
    dims[mat] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  if (d == 0) return;
  const bool transpose = nn.x < nn.y;
  const int rows = transpose ? nn.y : nn.x, cols = transpose ? nn.x : nn.y;
  if (real) {
    assemble_bipartite(c, idx_a, idx_b, kpts[kk], M, lm, rows, cols, transpose, true, Mr);
    if (blockDim.x == 32) bidiag_tgk_warp_real(Mr, lm, rows, cols, diag, e2, ur);
    else bidiag_tgk_real(Mr, lm, rows, cols, diag, e2, ur, red);
    return;
  }
  assemble_bipartite(c, idx_a, idx_b, kpts[kk], M, lm, rows, cols, transpose);
  if (blockDim.x == 32) bidiag_tgk_warp(M, lm, rows, cols, diag, e2, u);
  else bidiag_tgk(M, lm, rows, cols, diag, e2, u, s, red);
}

// Complex k-points with S <= 64: the matrix in registers of 256 threads (bidiag_tgk_reg); the assembly
// still goes through shared memory.
__global__ void __launch_bounds__(BIDIAG_REG_THREADS, 2)
    small_bidiag_reg_kernel(CellDev c, const double2* __restrict__ kpts, int nk, const uint64_t* __restrict__ masks,
                            double* tri, int* dims, int* status, const int* __restrict__ klist, int nks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = c.N, S = c.nsub;
  int64_t mk, mat;
  int kk;
  if (klist) {
    mk = blockIdx.x / nks;
    kk = klist[blockIdx.x - mk * nks];
    mat = mk * nk + kk;
  } else {
    mat = blockIdx.x;
    mk = mat / nk;
    kk = (int)(mat - mk * nk);
  }
  const int lm = bidiag_ld(S);
  double2* M = reinterpret_cast<double2*>(smem_raw);
  double* scratch = reinterpret_cast<double*>(M + (size_t)lm * S);
  int* idx_a = reinterpret_cast<int*>(scratch + BIDIAG_REG_SCRATCH);
  int* idx_b = idx_a + N;
  int* cnt = idx_b + N;
  double* diag = tri + mat * 2 * N;
  double* e2 = diag + N;
  const int2 nn = block_compact_bipartite(c, masks + mk * c.words, idx_a, idx_b, cnt);
  const int d = nn.x + nn.y;
  if (threadIdx.x == 0) {
    dims[mat] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  if (d == 0) return;
  const bool transpose = nn.x < nn.y;
  const int rows = transpose ? nn.y : nn.x, cols = transpose ? nn.x : nn.y;
  assemble_bipartite(c, idx_a, idx_b, kpts[kk], M, lm, rows, cols, transpose);
  bidiag_tgk_reg(M, lm, rows, cols, diag, e2, scratch);
}

// Real k-points (periodic gauge at TRIM k) with S <= 64: bidiag_tgk_reg_real.
__global__ void __launch_bounds__(BIDIAG_REG_THREADS, 3)
    small_bidiag_reg_real_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                 const uint64_t* __restrict__ masks, double* tri, int* dims, int* status,
                                 const int* __restrict__ klist, int nks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = c.N, S = c.nsub;
  const int64_t mk = blockIdx.x / nks;
  const int kk = klist[blockIdx.x - mk * nks];
  const int64_t mat = mk * nk + kk;
  const int lm = bidiag_ld_real(S);
  double* Mr = reinterpret_cast<double*>(smem_raw);
  double* scratch = Mr + (size_t)lm * S;
  int* idx_a = reinterpret_cast<int*>(scratch + BIDIAG_REG_SCRATCH_REAL);
  int* idx_b = idx_a + N;
  int* cnt = idx_b + N;
  double* diag = tri + mat * 2 * N;
  double* e2 = diag + N;
  const int2 nn = block_compact_bipartite(c, masks + mk * c.words, idx_a, idx_b, cnt);
  const int d = nn.x + nn.y;
  if (threadIdx.x == 0) {
    dims[mat] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  if (d == 0) return;
  const bool transpose = nn.x < nn.y;
  const int rows = transpose ? nn.y : nn.x, cols = transpose ? nn.x : nn.y;
  assemble_bipartite(c, idx_a, idx_b, kpts[kk], nullptr, lm, rows, cols, transpose, true, Mr);
  bidiag_tgk_reg_real(Mr, lm, rows, cols, diag, e2, scratch);
}

// Gram path of the S in (32, 64] tiers (hx_smallgram.cuh): compaction -> dense C in shared memory -> G = C^H C in
// registers -> Hermitian tridiagonalisation; output (diag[S], e2[S]) of G padded to S at tri + mat * 2N, read by
// launch_gram_idos with a cell of N = S.  dims = kept dimension nA + nB as in the TGK kernels.
template <bool REAL>
static __device__ __forceinline__ void small_gram_body(const CellDev& c, const double2* __restrict__ kpts, int nk,
                                                       const uint64_t* __restrict__ masks, double* tri, int* dims,
                                                       int* status, const int* __restrict__ klist, int nks) {
  using E = typename SgElem<REAL>::E;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = c.N, S = c.nsub;
  int64_t mk, mat;
  int kk;
  if (klist) {
    mk = blockIdx.x / nks;
    kk = klist[blockIdx.x - mk * nks];
    mat = mk * nk + kk;
  } else {
    mat = blockIdx.x;
    mk = mat / nk;
    kk = (int)(mat - mk * nk);
  }
  const int lm = REAL ? bidiag_ld_real(S) : bidiag_ld(S);
  E* M = reinterpret_cast<E*>(smem_raw);
  double* scratch = reinterpret_cast<double*>(M + (size_t)lm * S);
  E* lval = reinterpret_cast<E*>(scratch + sg_scratch_doubles<REAL>());
  int* lrow = reinterpret_cast<int*>(lval + 64 * SG_NZ);
  int* flag = lrow + 64 * SG_NZ;
  int* idx_a = flag + 2;
  int* idx_b = idx_a + N;
  int* cnt = idx_b + N;
  double* diag = tri + mat * 2 * N;
  double* e2 = diag + S;
  const int2 nn = block_compact_bipartite(c, masks + mk * c.words, idx_a, idx_b, cnt);
  const int d = nn.x + nn.y;
  if (threadIdx.x == 0) {
    dims[mat] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  if (d == 0) return;
  const bool transpose = nn.x < nn.y;
  const int rows = transpose ? nn.y : nn.x, cols = transpose ? nn.x : nn.y;
  if constexpr (REAL)
    assemble_bipartite(c, idx_a, idx_b, kpts[kk], nullptr, lm, rows, cols, transpose, true, M);
  else
    assemble_bipartite(c, idx_a, idx_b, kpts[kk], M, lm, rows, cols, transpose);
  if (!small_gram_tridiag<REAL>(M, lm, rows, cols, S, diag, e2, scratch, lrow, lval, flag) && threadIdx.x == 0) {
    dims[mat] = 0;
    status[mat] = 2;  // not a nearest-neighbour block: the host never routes such a model here
  }
}

__global__ void __launch_bounds__(BIDIAG_REG_THREADS, 2)
    small_gram_reg_kernel(CellDev c, const double2* __restrict__ kpts, int nk, const uint64_t* __restrict__ masks,
                          double* tri, int* dims, int* status, const int* __restrict__ klist, int nks) {
  small_gram_body<false>(c, kpts, nk, masks, tri, dims, status, klist, nks);
}

__global__ void __launch_bounds__(BIDIAG_REG_THREADS, 4)
    small_gram_reg_real_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                               const uint64_t* __restrict__ masks, double* tri, int* dims, int* status,
                               const int* __restrict__ klist, int nks) {
  small_gram_body<true>(c, kpts, nk, masks, tri, dims, status, klist, nks);
}

size_t small_gram_reg_smem(int N, int S, bool real) {
  const size_t es = real ? 8 : 16;
  const size_t lm = real ? bidiag_ld_real(S) : bidiag_ld(S);
  return lm * S * es + (size_t)(real ? sg_scratch_doubles<true>() : sg_scratch_doubles<false>()) * 8 +
         64 * SG_NZ * (es + 4) + 8 + (size_t)N * 8 + 2 * ((N + 31) / 32) * 4 + 16;
}

size_t small_bidiag_reg_real_smem(int N, int S) {
  return ((size_t)bidiag_ld_real(S) * S) * 8 + BIDIAG_REG_SCRATCH_REAL * 8 + (size_t)N * 8 +
         2 * ((N + 31) / 32) * 4 + 16;
}

size_t small_bidiag_reg_smem(int N, int S) {
  return ((size_t)bidiag_ld(S) * S) * 16 + BIDIAG_REG_SCRATCH * 8 + (size_t)N * 8 + 2 * ((N + 31) / 32) * 4 + 16;
}

size_t small_bidiag_smem(int N, int S) {
  return ((size_t)bidiag_ld(S) * S + 2 * (S + 1)) * 16 + 128 * 8 + (size_t)N * 8 + 2 * ((N + 31) / 32) * 4 + 16;
}

size_t small_bidiag_smem_real(int N, int S, bool warp) {
  const int lm = warp ? bidiag_ld_real_warp(S) : bidiag_ld_real(S);
  return ((size_t)lm * S + (S + 1)) * 8 + 128 * 8 + (size_t)N * 8 + 2 * ((N + 31) / 32) * 4 + 16;
}

size_t small_tridiag_smem(int N) {
  const int ld = N | 1;
  return (((size_t)N * ld + 1) & ~(size_t)1) * 8 + (size_t)N * 16 * 2 + 128 * 8 + (size_t)N * 4 +
         ((N + 31) / 32) * 4 + 16;
}

// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) global_tridiag_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                             const uint64_t* __restrict__ masks, int64_t mat0,
                                                             unsigned char* ws, size_t ws_stride, double* tri,
                                                             int* dims, int* status) {
  __shared__ double red[96];
  __shared__ int cnt[(HX_MAX_N + 31) / 32];
  const int N = c.N;
  const int64_t mat = mat0 + blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  unsigned char* w = ws + (size_t)blockIdx.x * ws_stride;
  double2* A = reinterpret_cast<double2*>(w);
  double2* B = A + (size_t)N * N;
  const bool general = c.pencil == 2;
  double2* v = general ? B + (size_t)N * N : B;
  double2* y = v + N;
  int* new_idx = reinterpret_cast<int*>(y + N);
  double* diag = tri + (int64_t)blockIdx.x * 2 * N;
  double* e2 = diag + N;

  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (threadIdx.x == 0) {
    dims[blockIdx.x] = d;
    status[mat] = d == 0 ? 3 : 0;
  }
  if (d == 0) return;
  const double2 k = kpts[kk];
  assemble_full(c, new_idx, d, k, A, N, false);
  if (general) {
    assemble_full(c, new_idx, d, k, B, N, true);
    if (!chol_reduce_full(A, B, N, d, red)) {
      if (threadIdx.x == 0) {
        status[mat] = 1;
        dims[blockIdx.x] = 0;
      }
      return;
    }
  }
  tridiag_full(A, N, d, diag, e2, v, y, red);
}

size_t global_ws_stride(int N, bool general) {
  size_t b = (size_t)N * N * 16 * (general ? 2 : 1) + (size_t)N * 16 * 2 + (size_t)N * 4;
  return (b + 255) & ~(size_t)255;
}

// ------------------------------------------------------------------------------------------------
// Early exit of the bisection (no eigenvalue output): an eigenvalue whose bracket [lo, hi] maps entirely
// into one gap between the transition windows contributes a full weight at a determined grid index
// (the index arithmetic of _kernels.py:68-101 is constant over the widened bracket, so the result
// equals the reference's for any eigenvalue in it).  Returns the index or LLONG_MIN if not settled.
static __device__ __forceinline__ long long settle_index(const CellDev& c, const GridDev& g, int sharp, double lo,
                                                         double hi) {
  const double ea = pencil_map(c, lo), eb = pencil_map(c, hi);
  double Ea = fmin(ea, eb), Eb = fmax(ea, eb);
  const double eta = 16.0 * DBL_EPSILON * fmax(1.0, fmax(fabs(Ea), fabs(Eb)));
  Ea -= eta;
  Eb += eta;
  // multiplying by 1/step instead of dividing moves a quotient by <= 2 ulp; the 16-ulp widening above
  // (>= 10 ulp of the quotient) keeps the decision identical to the reference's division
  const double is = g.inv_step;
  if (sharp) {
    const long long ia = (long long)floor((Ea - g.e0) * is), ib = (long long)floor((Eb - g.e0) * is);
    return ia == ib ? ia + 1 : LLONG_MIN;
  }
  const long long la = (long long)ceil((Ea + g.delta - g.e0) * is);
  const long long lb = (long long)ceil((Eb + g.delta - g.e0) * is);
  const long long ma = (long long)floor((Ea - g.delta - g.e0) * is) + 1;
  const long long mb = (long long)floor((Eb - g.delta - g.e0) * is) + 1;
  return (la == lb && ma == mb && ma >= la) ? la : LLONG_MIN;
}

static __device__ __forceinline__ void add_settled(const GridDev& g, int* diff, int64_t mk, long long l, int mult) {
  const long long l0 = l < 0 ? 0 : l;
  if (l0 < g.npts) atomicAdd(diff + mk * (g.npts + 1) + l0, mult);
}

// IDOS contribution (and status) of one eigenvalue lam of T
static __device__ __forceinline__ void add_eigenvalue(const CellDev& c, const GridDev& g, int sharp, int* diff,
                                                      unsigned long long* trans, int* status, int64_t mat, int nk,
                                                      double lam) {
  const double E = pencil_map(c, lam);
  if (!isfinite(E)) atomicCAS(status + mat, 0, 2);
  const int64_t mk = mat / nk;
  const int mult = kmul(g, mat, nk);
  if (sharp) sharp_state(g, E, diff + mk * (g.npts + 1), mult);
  else idos_state(g, E, diff + mk * (g.npts + 1), trans + mk * g.npts, mult);
}

// One thread per (matrix, eigenvalue index) - for TGK tridiagonals one thread per +-pair: it bisects
// lambda_{d-1-j} >= 0 and also accounts for -lambda_{d-1-j} = lambda_j.  tri: per matrix `tri_stride`
// doubles, diag at 0 and e2 at +N (N = c.N).  Matrices with dims == 0 (all vacant / failed) contribute
// nothing.
template <bool TGK>
__global__ void __launch_bounds__(128) eig_idos_kernel(CellDev c, int nk, GridDev g, int64_t mat0, int64_t nmat,
                                                       const double* __restrict__ tri, size_t tri_stride,
                                                       const int* __restrict__ dims, int* diff,
                                                       unsigned long long* trans, double* eigs, int* status,
                                                       int sharp, RefineItem* refine,
                                                       unsigned long long* refine_count) {
  const int N = c.N;
  const int per = TGK ? (N + 1) / 2 : N;
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lm = slot / per;
  if (lm >= nmat) return;
  const int j = (int)(slot - lm * per);
  const int64_t mat = mat0 + lm;
  const int d = dims[lm];
  double* eig_out = eigs ? eigs + mat * N : nullptr;
  const bool rev = (c.pencil == 1) && (c.t - c.s * c.eps0 < 0.0);
  auto put = [&](int k, double E) {
    if (eig_out) eig_out[rev ? d - 1 - k : k] = E;
  };
  if (eig_out) {  // padding beyond d
    if (j >= d) eig_out[j] = qnan();
    if (TGK && N - 1 - j >= d && N - 1 - j != j) eig_out[N - 1 - j] = qnan();
  }
  // index bisected by this thread and whether its mirror is also ours
  int idx;
  bool mirror = false;
  if (TGK) {
    if (2 * j + 1 > d) return;  // j >= ceil(d/2)
    idx = d - 1 - j;
    if (idx == j) {  // odd d: the middle eigenvalue of a symmetric spectrum is exactly 0
      if (diff) add_eigenvalue(c, g, sharp, diff, trans, status, mat, nk, 0.0);
      put(j, pencil_map(c, 0.0));
      return;
    }
    mirror = true;
  } else {
    if (j >= d) return;
    idx = j;
  }
  const double* diag = tri + lm * tri_stride;
  const double* e2 = diag + N;
  // Gershgorin interval and pivmin (dstebz conventions)
  double gl = 1e308, gu = -1e308, em = 0.0, el = 0.0;
  for (int i = 0; i < d; ++i) {
    const double er2 = i + 1 < d ? e2[i] : 0.0;
    const double er = sqrt(er2);
    const double di = TGK ? 0.0 : diag[i];
    gl = fmin(gl, di - el - er);
    gu = fmax(gu, di + el + er);
    em = fmax(em, er2);
    el = er;
  }
  const double pivmin = DBL_MIN * fmax(1.0, em);
  const double tnorm = fmax(fabs(gl), fabs(gu));
  gl = gl - 2.1 * tnorm * DBL_EPSILON * d - 4.2 * pivmin;
  gu = gu + 2.1 * tnorm * DBL_EPSILON * d + 4.2 * pivmin;
  double lo = gl, hi = gu;
  const bool early = eigs == nullptr && refine != nullptr;
  // settle state: bit 0 = lambda settled, bit 1 = mirror settled (or not needed)
  int done = mirror ? 0 : 2;
  const int64_t mk = mat / nk;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double tol = 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin;
    if (hi - lo <= tol || mid <= lo || mid >= hi) break;
    if (early && it >= 4) {
      if (!(done & 1)) {
        const long long l = settle_index(c, g, sharp, lo, hi);
        if (l != LLONG_MIN) {
          add_settled(g, diff, mk, l, kmul(g, mat, nk));
          done |= 1;
        }
      }
      if (!(done & 2)) {
        const long long l = settle_index(c, g, sharp, -hi, -lo);
        if (l != LLONG_MIN) {
          add_settled(g, diff, mk, l, kmul(g, mat, nk));
          done |= 2;
        }
      }
      if (done == 3) return;
      if (it >= 14) {
        // phase 1 done: hand the bracket to the dense refinement pass (keeps warps free of divergence)
        const unsigned long long pos = atomicAdd(refine_count, 1ull);
        refine[pos] = RefineItem{mat, lm, idx, (~done) & 3, lo, hi, pivmin};
        return;
      }
    }
    if (sturm_count_fast<TGK>(diag, e2, d, mid, pivmin) > idx) hi = mid;
    else lo = mid;
  }
  const double lam = 0.5 * (lo + hi);
  if (diff) {
    if (!(done & 1)) add_eigenvalue(c, g, sharp, diff, trans, status, mat, nk, lam);
    if (!(done & 2)) add_eigenvalue(c, g, sharp, diff, trans, status, mat, nk, -lam);
  } else {
    if (!isfinite(pencil_map(c, lam)) || (mirror && !isfinite(pencil_map(c, -lam)))) atomicCAS(status + mat, 0, 2);
  }
  put(idx, pencil_map(c, lam));
  if (mirror) put(d - 1 - idx, pencil_map(c, -lam));
}

// The refinement only feeds the IDOS (never an eigenvalue output): the smoothed count is a Lipschitz
// function of E (slope <= ~2/delta), so lambda to 1e-13 (vs 2 ulp) moves a curve value by < 1e-10, well
// inside the 1e-9 parity tolerance, and saves ~8 of ~40 bisection steps.
__device__ __forceinline__ double refine_tol(double lo, double hi, double pivmin) {
  const double m = fmax(fabs(lo), fabs(hi));
  return fmax(2.0 * DBL_EPSILON * m + pivmin, 1e-13 * fmax(1.0, m));
}

// G lanes per item: G-point multisection (log2(G+1) bits per Sturm round) for the latency-bound case of
// few items (large matrices); shared by the bisection and the zone refinement passes.
template <bool TGK, bool GRAM = false>
__device__ void refine_multisection(const CellDev& c, int nk, const GridDev& g, const double* __restrict__ tri,
                                    size_t tri_stride, const int* __restrict__ dims, int* diff,
                                    unsigned long long* trans, int* status, int sharp,
                                    const RefineItem* __restrict__ items, unsigned long long n, int G) {
  const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, sub = lane % G, base = lane - sub;
    const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << base;
    const unsigned long long ngroups = nthreads / G;
    const double inv = 1.0 / (double)(G + 1);
    // loop bound uniform over the warp: every lane runs the same number of rounds (shuffles/ballots)
    const unsigned long long g0 = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const unsigned long long wfirst = ((unsigned long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / G;
    for (unsigned long long qw = wfirst; qw < n; qw += ngroups) {
      const unsigned long long q = qw + (g0 - wfirst);
      const bool valid = q < n;
      RefineItem it = items[valid ? q : qw];
      const double* diag = tri + it.lm * tri_stride;
      const double* e2 = diag + c.N;
      const int d = GRAM ? c.N : dims[it.lm];  // Gram mode: the S x S tridiagonal of G, items in mu = sigma^2
      double lo = it.lo, hi = it.hi;
      bool done = false;
      for (int k = 0; k < 200; ++k) {
        const double tol = refine_tol(lo, hi, it.pivmin);
        const double mid = 0.5 * (lo + hi);
        done = done || hi - lo <= tol || mid <= lo || mid >= hi;
        if (__all_sync(0xffffffffu, done)) break;
        // points x_m = lo + (m + 1) (hi - lo) / (G + 1); the first with count > idx brackets lambda
        const double x = fma((double)(sub + 1) * inv, hi - lo, lo);
        bool above = true;
        if (!done) above = (x > lo && x < hi) ? sturm_count_fast<TGK>(diag, e2, d, x, it.pivmin) > it.idx : x >= hi;
        const unsigned b = (__ballot_sync(0xffffffffu, above) & gmask) >> base;
        const int m = b ? __ffs(b) - 1 : G;  // lambda in (x_{m-1}, x_m]
        const double nlo = __shfl_sync(0xffffffffu, x, base + (m == 0 ? 0 : m - 1));
        const double nhi = __shfl_sync(0xffffffffu, x, base + (m == G ? G - 1 : m));
        if (!done) {
          lo = m == 0 ? lo : nlo;
          hi = m == G ? hi : nhi;
        }
      }
      if (valid && sub == 0) {
        const double lam = 0.5 * (lo + hi);
        if constexpr (GRAM) {  // lambda = +-sqrt(mu), sign in flag bit 1
          const double sg = sqrt(fmax(lam, 0.0));
          add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, (it.flags & 2) ? -sg : sg);
        } else {
          if (it.flags & 1) add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, lam);
          if (it.flags & 2) add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, -lam);
        }
      }
    }
}

// Staged G-lane multisection of the zone items (grouped list: zone_count(_gram)_kernel with group =
// blockDim.x / G): every block iteration works on blockDim.x / G consecutive items of ONE matrix, whose tridiagonal
// (2 S doubles) it first copies to shared memory - the Sturm row steps then read shared memory with at most a few
// distinct addresses per warp instead of L2 (ncu on the unstaged kernel: long-scoreboard stalls dominate).  Same
// search as refine_multisection (same points, same counts: the same bits).
template <bool ZD, bool GRAM>
__device__ void refine_multisection_staged(const CellDev& c, int nk, const GridDev& g,
                                           const double* __restrict__ tri, size_t tri_stride,
                                           const int* __restrict__ dims, int* diff, unsigned long long* trans,
                                           int* status, int sharp, const RefineItem* __restrict__ items,
                                           unsigned long long n, int G, double* sm) {
  const int S = c.N;
  const int per_block = blockDim.x / G;
  const unsigned long long stride = (unsigned long long)gridDim.x * per_block;
  const int lane = threadIdx.x & 31, sub = lane % G, base = lane - sub;
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << base;
  const double inv = 1.0 / (double)(G + 1);
  for (unsigned long long qb = (unsigned long long)blockIdx.x * per_block; qb < n; qb += stride) {
    const RefineItem it = items[qb + threadIdx.x / G];  // n is a multiple of per_block
    const int64_t lm0 = items[qb].lm;
    const double* src = tri + lm0 * tri_stride;
    const int d = GRAM ? S : dims[lm0];  // Gram mode: the S x S tridiagonal of G, items in mu = sigma^2
    __syncthreads();  // the previous iteration's readers are done
    for (int i = threadIdx.x; i < 2 * S; i += blockDim.x) sm[i] = src[i];
    __syncthreads();
    const bool valid = it.idx >= 0;
    double lo = it.lo, hi = it.hi;
    bool done = !valid;
    for (int k = 0; k < 200; ++k) {
      const double tol = refine_tol(lo, hi, it.pivmin);
      const double mid = 0.5 * (lo + hi);
      done = done || hi - lo <= tol || mid <= lo || mid >= hi;
      if (__all_sync(0xffffffffu, done)) break;
      const double x = fma((double)(sub + 1) * inv, hi - lo, lo);
      bool above = true;
      if (!done) above = (x > lo && x < hi) ? sturm_count_fast<ZD>(sm, sm + S, d, x, it.pivmin) > it.idx : x >= hi;
      const unsigned b = (__ballot_sync(0xffffffffu, above) & gmask) >> base;
      const int m = b ? __ffs(b) - 1 : G;
      const double nlo = __shfl_sync(0xffffffffu, x, base + (m == 0 ? 0 : m - 1));
      const double nhi = __shfl_sync(0xffffffffu, x, base + (m == G ? G - 1 : m));
      if (!done) {
        lo = m == 0 ? lo : nlo;
        hi = m == G ? hi : nhi;
      }
    }
    if (valid && sub == 0) {
      const double lam = 0.5 * (lo + hi);
      if constexpr (GRAM) {  // lambda = +-sqrt(mu), sign in flag bit 1
        const double sg = sqrt(fmax(lam, 0.0));
        add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, (it.flags & 2) ? -sg : sg);
      } else {
        if (it.flags & 1) add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, lam);
        if (it.flags & 2) add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, -lam);
      }
    }
  }
}

// Phase 2: bisection of the eigenvalues left unsettled by eig_idos_kernel, densely
// packed (every lane of a warp has real work), then the IDOS contribution (+ the TGK mirror).
// Lanes per refinement item (1: per-thread Newton / bisection, 2-8: multisection), a function of the
// matrix dimension alone (never the batch size).
constexpr int g_refine_min_n = 1024;  // N >= this: multisection with 4 lanes per item
__device__ __forceinline__ int refine_lanes(int N) { return N >= g_refine_min_n ? 4 : 1; }

template <bool TGK>
__global__ void __launch_bounds__(128) eig_refine_kernel(CellDev c, int nk, GridDev g, const double* __restrict__ tri,
                                                         size_t tri_stride, const int* __restrict__ dims, int* diff,
                                                         unsigned long long* trans, int* status, int sharp,
                                                         const RefineItem* __restrict__ items,
                                                         const unsigned long long* __restrict__ count) {
  const unsigned long long n = *count;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
  // G lanes per item: G-point multisection (log2(G+1) bits per Sturm round).  The method is a function of
  // the matrix size only (refine_lanes), never of the batch: the refined eigenvalues - and so the curves - are
  // then bitwise independent of how the masks are split into batches, devices or ranks.
  const int G = refine_lanes(c.N);
  if (G > 1) {
    refine_multisection<TGK>(c, nk, g, tri, tri_stride, dims, diff, trans, status, sharp, items, n, G);
    return;
  }
  for (unsigned long long q = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += nthreads) {
    const RefineItem it = items[q];
    const double* diag = tri + it.lm * tri_stride;
    const double* e2 = diag + c.N;
    const int d = dims[it.lm];
    double lo = it.lo, hi = it.hi;
    for (int k = 0; k < 200; ++k) {
      const double mid = 0.5 * (lo + hi);
      const double tol = refine_tol(lo, hi, it.pivmin);
      if (hi - lo <= tol || mid <= lo || mid >= hi) break;
      if (sturm_count_fast<TGK>(diag, e2, d, mid, it.pivmin) > it.idx) hi = mid;
      else lo = mid;
    }
    const double lam = 0.5 * (lo + hi);
    if (it.flags & 1) add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, lam);
    if (it.flags & 2) add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, -lam);
  }
}

// ------------------------------------------------------------------------------------------------
// Zone path of the eigenvalue stage (IDOS only, no eigenvalue output).
//
// Every eigenvalue contributes to the curve through the reference's index arithmetic
// (_kernels.py:68-101): a full weight from lo = ceil((E + delta - e0)/step) on, and transition terms for
// the grid points within delta of E.  Around every grid energy e_m lies a transition zone
// Z_m = [e_m - w - eta, e_m + w + eta] (w = delta, or 0 for the sharp counts; eta = 4e-12 max(1, |E|)
// covers the rounding of the reference's own quotients).  An eigenvalue between Z_{m-1} and Z_m
// contributes exactly a full weight at index m - nothing else depends on where it lies in that gap - so
// the gap populations follow from Sturm counts at the 2 npts zone edges alone (one thread per zone, two
// interleaved recurrences), and only the eigenvalues inside a zone (about 2(w + eta)/step of them) are
// located, by a Newton-accelerated bracketed search from the zone's own bracket (zone_refine_kernel).
// For a matrix of dimension d this costs 2 npts + (zone eigenvalues) x (a few) Sturm counts instead of
// ~d/2 x (8 .. 14) bisection steps plus the refinement of the zone eigenvalues from a full-width start.

// Inverse of pencil_map (E -> lambda) on the branch 1 + s lambda > 0.
__host__ __device__ __forceinline__ double pencil_inv(int pencil, double eps0, double t, double s, double E) {
  if (pencil != 1) return E;
  return (E - eps0) / (t - s * E);
}

// lambda-space bracket [la, lb] of zone m.
__device__ __forceinline__ void zone_bracket(const CellDev& c, const GridDev& g, int sharp, int m, double& la,
                                             double& lb) {
  const double em = __dadd_rn(g.e0, __dmul_rn(g.step, (double)m));
  const double w = sharp ? 0.0 : g.delta;
  double Elo = em - w, Ehi = em + w;
  Elo -= 4e-12 * fmax(1.0, fabs(Elo));
  Ehi += 4e-12 * fmax(1.0, fabs(Ehi));
  const double a = pencil_inv(c.pencil, c.eps0, c.t, c.s, Elo), b = pencil_inv(c.pencil, c.eps0, c.t, c.s, Ehi);
  la = fmin(a, b);
  lb = fmax(a, b);
}

// Two interleaved Sturm counts (the two edges of a zone).
template <bool ZD>
__device__ __forceinline__ void sturm_count_pair(const double* __restrict__ diag, const double* __restrict__ e2, int d,
                                                 double xa, double xb, double pivmin, int& na, int& nb) {
#if HX_STURM_POLY
  (void)pivmin;
  const double a0 = ZD ? 0.0 : diag[0];
  double pa1 = 1.0, pa0 = a0 - xa, pb1 = 1.0, pb0 = a0 - xb;
  if (pa0 == 0.0) pa0 = -0x1p-200;
  if (pb0 == 0.0) pb0 = -0x1p-200;
  int ca = pa0 < 0.0, cb = pb0 < 0.0;
  for (int i = 1; i < d; ++i) {
    const double e = e2[i - 1], a = ZD ? 0.0 : diag[i];
    double pan = fma(a - xa, pa0, -(e * pa1));
    double pbn = fma(a - xb, pb0, -(e * pb1));
    if (pan == 0.0) pan = -0x1p-200 * pa0;
    if (pbn == 0.0) pbn = -0x1p-200 * pb0;
    ca += sturm_sign_change(pan, pa0);
    cb += sturm_sign_change(pbn, pb0);
    pa1 = pa0;
    pa0 = pan;
    pb1 = pb0;
    pb0 = pbn;
    if ((i & 3) == 0) {
      const double sa = sturm_scale_of(pa0, pa1), sb = sturm_scale_of(pb0, pb1);
      pa0 *= sa;
      pa1 *= sa;
      pb0 *= sb;
      pb1 *= sb;
    }
  }
  na = ca;
  nb = cb;
#else
  double qa = (ZD ? 0.0 : diag[0]) - xa, qb = (ZD ? 0.0 : diag[0]) - xb;
  if (fabs(qa) <= pivmin) qa = -pivmin;
  if (fabs(qb) <= pivmin) qb = -pivmin;
  int ca = qa < 0.0, cb = qb < 0.0;
  for (int i = 1; i < d; ++i) {
    const double e = e2[i - 1], a = ZD ? 0.0 : diag[i];
    qa = fma(-e, sturm_rcp(qa), a - xa);
    qb = fma(-e, sturm_rcp(qb), a - xb);
    if (fabs(qa) <= pivmin) qa = -pivmin;
    if (fabs(qb) <= pivmin) qb = -pivmin;
    ca += qa < 0.0;
    cb += qb < 0.0;
  }
  na = ca;
  nb = cb;
#endif
}

template <bool ZD>
__device__ double zone_locate(const double* diag, const double* e2, int d, int idx, double lo, double hi, int clo,
                              int chi, double pivmin);

// Block-wide exclusive scan of the zone item counts nz(m), m < npts, into zoff[0 .. npts] (zoff[npts] = total);
// wsum: 8 ints of shared memory.  Every thread of the block calls it; ends with a barrier.
template <class F>
__device__ __forceinline__ void zone_item_offsets(int npts, int* zoff, int* wsum, F nz_of) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int carry = 0;
  for (int m0 = 0; m0 < npts; m0 += blockDim.x) {
    const int m = m0 + tid;
    const int nz = m < npts ? nz_of(m) : 0;
    int incl = nz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (m < npts) zoff[m] = before + incl - nz;
    for (int w = 0; w < nw; ++w) carry += wsum[w];
    __syncthreads();
  }
  if (tid == 0) zoff[npts] = carry;
  __syncthreads();
}

// One CTA per matrix.  counts[2m] / counts[2m+1]: eigenvalues below the lower / upper lambda edge of zone m
// (dynamic shared memory, 2 npts ints).  rev: E decreases with lambda.
template <bool ZD>
__global__ void __launch_bounds__(256) zone_count_kernel(CellDev c, int nk, GridDev g, int sharp, int rev,
                                                         int64_t mat0, int64_t nmat, const double* __restrict__ tri,
                                                         size_t tri_stride, const int* __restrict__ dims, int* diff,
                                                         RefineItem* refine, unsigned long long* refine_count,
                                                         int fuse, unsigned long long* trans, int* status, int group) {
  // fuse != 0 (per-thread refinement, N < 1024): the block locates its own zone eigenvalues on a shared-memory copy
  // of the tridiagonal (as zone_count_gram_kernel).  Dynamic shared memory: fuse: [2 N] doubles (diag, e2), then
  // ints: [2 npts] counts, fuse: [npts + 1] item offsets, [N] items.
  extern __shared__ __align__(16) unsigned char zraw[];
  __shared__ double red[3][32];
  __shared__ int wsum[8];
  __shared__ unsigned long long list_base;  // group > 0: the matrix's padded range of the item list
  const int64_t lm = blockIdx.x;
  if (lm >= nmat) return;
  const int d = dims[lm];
  if (d <= 0) return;
  const int N = c.N, npts = g.npts;
  double* sd = reinterpret_cast<double*>(zraw);
  int* zc = reinterpret_cast<int*>(zraw + (fuse ? (size_t)2 * N * sizeof(double) : 0));
  int* zoff = zc + 2 * npts;     // fuse only
  int* ilist = zoff + npts + 1;  // fuse only
  const int64_t mat = mat0 + lm;
  const int64_t mk = mat / nk;
  const double* diag = tri + lm * tri_stride;
  const double* e2 = diag + N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // Gershgorin interval and pivmin (dstebz conventions, as eig_idos_kernel)
  double gl = 1e308, gu = -1e308, em = 0.0;
  for (int i = tid; i < d; i += blockDim.x) {
    const double el = i > 0 ? sqrt(e2[i - 1]) : 0.0;
    const double er2 = i + 1 < d ? e2[i] : 0.0;
    const double er = sqrt(er2);
    const double di = ZD ? 0.0 : diag[i];
    gl = fmin(gl, di - el - er);
    gu = fmax(gu, di + el + er);
    em = fmax(em, er2);
    if (fuse) {
      sd[i] = di;
      sd[N + i] = e2[i];
    }
  }
  gl = warp_min(gl);
  gu = warp_max(gu);
  em = warp_max(em);
  if (lane == 0) {
    red[0][warp] = gl;
    red[1][warp] = gu;
    red[2][warp] = em;
  }
  __syncthreads();
  gl = red[0][0];
  gu = red[1][0];
  em = red[2][0];
  for (int w = 1; w < nw; ++w) {
    gl = fmin(gl, red[0][w]);
    gu = fmax(gu, red[1][w]);
    em = fmax(em, red[2][w]);
  }
  const double pivmin = DBL_MIN * fmax(1.0, em);
  const double tnorm = fmax(fabs(gl), fabs(gu));
  gl = gl - 2.1 * tnorm * DBL_EPSILON * d - 4.2 * pivmin;
  gu = gu + 2.1 * tnorm * DBL_EPSILON * d + 4.2 * pivmin;
  for (int m = tid; m < npts; m += blockDim.x) {
    double xa, xb;
    zone_bracket(c, g, sharp, m, xa, xb);
    // two interleaved Sturm recurrences (edges outside the Gershgorin interval are trivial)
    const bool ra = xa > gl && xa < gu, rb = xb > gl && xb < gu;
    int ca = xa <= gl ? 0 : d, cb = xb <= gl ? 0 : d;
    if (ra || rb) {
      int na, nb;
      sturm_count_pair<ZD>(fuse ? sd : diag, fuse ? sd + N : e2, d, xa, xb, pivmin, na, nb);
      if (ra) ca = na;
      if (rb) cb = nb;
    }
    zc[2 * m] = ca;
    zc[2 * m + 1] = max(ca, cb);
  }
  __syncthreads();
  int* drow = diff + mk * (npts + 1);
  if (fuse || group > 0) {
    zone_item_offsets(npts, zoff, wsum, [&](int m) { return zc[2 * m + 1] - zc[2 * m]; });
    if (!fuse) {
      const int total = zoff[npts], padded = (total + group - 1) / group * group;
      if (tid == 0) list_base = atomicAdd(refine_count, (unsigned long long)padded);
      __syncthreads();
      for (int q = total + tid; q < padded; q += blockDim.x)
        refine[list_base + q] = RefineItem{mat, lm, -1, 0, 0.0, 0.0, 0.0};
    }
  }
  for (int m = tid; m < npts; m += blockDim.x) {
    // gap below zone m (in E): settles at index m
    int n;
    if (!rev) n = zc[2 * m] - (m > 0 ? zc[2 * m - 1] : 0);
    else n = (m > 0 ? zc[2 * m - 2] : d) - zc[2 * m + 1];
    if (n > 0) atomicAdd(drow + m, n * kmul(g, mat, nk));
    // eigenvalues inside zone m: refinement items from the zone's own bracket
    const int i0 = zc[2 * m], nz = zc[2 * m + 1] - i0;
    if (nz > 0) {
      if (fuse) {
        const int o = zoff[m];
        for (int k = 0; k < nz; ++k) ilist[o + k] = m | (k << 16);
        continue;
      }
      double xa, xb;
      zone_bracket(c, g, sharp, m, xa, xb);
      const unsigned long long pos =
          group > 0 ? list_base + (unsigned long long)zoff[m] : atomicAdd(refine_count, (unsigned long long)nz);
      for (int k = 0; k < nz; ++k)
        refine[pos + k] = RefineItem{mat, lm, i0 + k, (int)(1u | ((unsigned)k << 2) | ((unsigned)nz << 17)),
                                     fmax(xa, gl), fmin(xb, gu), pivmin};
    }
  }
  if (!fuse) return;
  __syncthreads();
  const int total = zoff[npts];
  for (int q = tid; q < total; q += blockDim.x) {
    const int il = ilist[q], m = il & 0xffff, k = il >> 16;
    double xa, xb;
    zone_bracket(c, g, sharp, m, xa, xb);
    const int i0 = zc[2 * m], nz = zc[2 * m + 1] - i0;
    const double lam = zone_locate<ZD>(sd, sd + N, d, i0 + k, fmax(xa, gl), fmin(xb, gu), i0, i0 + nz, pivmin);
    add_eigenvalue(c, g, sharp, diff, trans, status, mat, nk, lam);
  }
}

// Sturm count below x and, with it, s = d/dx log|det(T - x)| = P'(x) / P(x): the determinant recurrence of
// sturm_count_fast and its derivative P_i' = (a_i - x) P_{i-1}' - P_{i-1} - e2_{i-1} P_{i-2}' (P_{-1}' = 0,
// P_0' = -1) under the same power-of-two scaling; one division at the end.  (HX_STURM_POLY=0: the dstebz quotients
// with s = sum_i q_i'/q_i, q_i' = -1 + e q_{i-1}'/q_{i-1}^2.)
template <bool ZD>
__device__ __forceinline__ int sturm_count_deriv(const double* __restrict__ diag, const double* __restrict__ e2, int d,
                                                 double x, double pivmin, double& s) {
#if HX_STURM_POLY
  (void)pivmin;
  double p1 = 1.0, p0 = (ZD ? 0.0 : diag[0]) - x, d1 = 0.0, d0 = -1.0;
  if (p0 == 0.0) p0 = -0x1p-200;
  int cnt = p0 < 0.0;
  for (int i = 1; i < d; ++i) {
    const double e = e2[i - 1], ax = (ZD ? 0.0 : diag[i]) - x;
    double pn = fma(ax, p0, -(e * p1));
    const double dn = fma(ax, d0, fma(-e, d1, -p0));
    if (pn == 0.0) pn = -0x1p-200 * p0;
    cnt += sturm_sign_change(pn, p0);
    p1 = p0;
    p0 = pn;
    d1 = d0;
    d0 = dn;
    if ((i & 3) == 0) {
      const double sc = sturm_scale_of(p0, p1);
      p0 *= sc;
      p1 *= sc;
      d0 *= sc;
      d1 *= sc;
    }
  }
  s = d0 / p0;
  return cnt;
#else
  double q = (ZD ? 0.0 : diag[0]) - x;
  if (fabs(q) <= pivmin) q = -pivmin;
  int cnt = q < 0.0;
  double r = sturm_rcp(q), dq = -1.0;
  double acc = -r;
  for (int i = 1; i < d; ++i) {
    const double e = e2[i - 1];
    const double er = e * r;
    q = fma(-e, r, (ZD ? 0.0 : diag[i]) - x);
    dq = fma(er * r, dq, -1.0);
    if (fabs(q) <= pivmin) q = -pivmin;
    cnt += q < 0.0;
    r = sturm_rcp(q);
    acc = fma(dq, r, acc);
  }
  s = acc;
  return cnt;
#endif
}

// Eigenvalue idx of the tridiagonal inside [lo, hi] (clo / chi: Sturm counts at lo / hi) to the
// refinement tolerance.  Bisection until the bracket isolates the eigenvalue (chi - clo == 1), then a
// safeguarded Newton iteration on det(T - x) (rtsafe rules: a Newton step is taken only when it stays in
// the bracket and at least halves the previous step, else bisection); every trial point's Sturm count
// shrinks the bracket, and a converged iterate is certified by closing the bracket around it with two
// counts.  Exact (or sub-tolerance) multiple eigenvalues never isolate and finish by bisection.
template <bool ZD>
__device__ double zone_locate(const double* diag, const double* e2, int d, int idx, double lo, double hi, int clo,
                              int chi, double pivmin) {
  for (int it = 0; it < 200 && chi - clo > 1; ++it) {
    if (hi - lo <= refine_tol(lo, hi, pivmin)) return 0.5 * (lo + hi);
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) return mid;
    const int cm = sturm_count_fast<ZD>(diag, e2, d, mid, pivmin);
    if (cm > idx) {
      hi = mid;
      chi = cm;
    } else {
      lo = mid;
      clo = cm;
    }
  }
  double x = 0.5 * (lo + hi), dxold = hi - lo, dx = dxold;
  for (int it = 0; it < 200; ++it) {
    double tol = refine_tol(lo, hi, pivmin);
    if (hi - lo <= tol) break;
    double sd;
    const int cnt = sturm_count_deriv<ZD>(diag, e2, d, x, pivmin, sd);
    if (cnt > idx) hi = x;
    else lo = x;
    tol = refine_tol(lo, hi, pivmin);
    if (hi - lo <= tol) break;
    const double nstep = (sd != 0.0 && isfinite(sd)) ? 1.0 / sd : 0.0;
    if (nstep != 0.0 && fabs(nstep) <= 0.25 * tol) {
      // converged (the step is below the tolerance, possibly below an ulp of x).  The bracket isolates
      // the eigenvalue (one root of det(T - x) in it), so the Newton point is within d |step| of it
      // (Laguerre's bound; in practice ~step^2): accept it.
      const double xc = fmin(fmax(x - nstep, lo), hi);
      if (chi - clo == 1) return xc;
      const double a = fmax(lo, xc - 0.5 * tol), b = fmin(hi, xc + 0.5 * tol);
      if (a > lo) {
        if (sturm_count_fast<ZD>(diag, e2, d, a, pivmin) > idx) hi = a;
        else lo = a;
      }
      if (b < hi && b > lo) {
        if (sturm_count_fast<ZD>(diag, e2, d, b, pivmin) > idx) hi = b;
        else lo = b;
      }
      x = 0.5 * (lo + hi);
      dxold = dx = hi - lo;
      continue;
    }
    const double xn = x - nstep;
    if (nstep == 0.0 || !(xn > lo && xn < hi) || fabs(2.0 * nstep) > fabs(dxold)) {
      dxold = dx;
      dx = 0.5 * (hi - lo);
      x = lo + dx;
      if (x <= lo || x >= hi) break;
      continue;
    }
    dxold = dx;
    dx = nstep;
    x = xn;
  }
  return 0.5 * (lo + hi);
}

template <bool ZD>
__global__ void __launch_bounds__(512) zone_refine_kernel(CellDev c, int nk, GridDev g, const double* __restrict__ tri,
                                                          size_t tri_stride, const int* __restrict__ dims, int* diff,
                                                          unsigned long long* trans, int* status, int sharp,
                                                          const RefineItem* __restrict__ items,
                                                          const unsigned long long* __restrict__ count, int staged,
                                                          int G) {
  extern __shared__ __align__(16) double zsm_stage[];
  const unsigned long long n = *count;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
  // G (launch_eig_idos: a function of the matrix size and the options only, so that results do not depend on the
  // batch composition): 1 = one thread per item, Newton (about 11 Sturm counts on average; staged: grouped list,
  // the matrix in shared memory); > 1 = G-lane multisection with its fixed round count (tridiagonals too large to
  // stage, HX_REFINE_LANES).
  if (G > 1) {
    if (staged)
      refine_multisection_staged<ZD, false>(c, nk, g, tri, tri_stride, dims, diff, trans, status, sharp, items, n, G,
                                            zsm_stage);
    else
      refine_multisection<ZD>(c, nk, g, tri, tri_stride, dims, diff, trans, status, sharp, items, n, G);
    return;
  }
  if (staged) {
    // grouped list: blockDim.x items of one matrix per block iteration, its tridiagonal in shared memory
    const int N = c.N;
    for (unsigned long long qb = (unsigned long long)blockIdx.x * blockDim.x; qb < n; qb += nthreads) {
      const RefineItem it = items[qb + threadIdx.x];
      const int64_t lm0 = items[qb].lm;
      const double* src = tri + lm0 * tri_stride;
      __syncthreads();
      for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) zsm_stage[i] = src[i];
      __syncthreads();
      if (it.idx < 0) continue;
      const unsigned f = (unsigned)it.flags;
      const int k = (int)((f >> 2) & 0x7fffu), nz = (int)(f >> 17);
      const int clo = it.idx - k;
      const double lam =
          zone_locate<ZD>(zsm_stage, zsm_stage + N, dims[lm0], it.idx, it.lo, it.hi, clo, clo + nz, it.pivmin);
      add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, lam);
    }
    return;
  }
  for (unsigned long long q = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += nthreads) {
    const RefineItem it = items[q];
    const double* diag = tri + it.lm * tri_stride;
    // flags: bit 0 set; bits 2..16: k = idx - (count at lo); bits 17..31: eigenvalues in the zone
    const unsigned f = (unsigned)it.flags;
    const int k = (int)((f >> 2) & 0x7fffu), nz = (int)(f >> 17);
    const int clo = it.idx - k;
    const double lam = zone_locate<ZD>(diag, diag + c.N, dims[it.lm], it.idx, it.lo, it.hi, clo, clo + nz, it.pivmin);
    add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, lam);
  }
}

// Host-side applicability of the zone path: non-overlapping zones and an inverse pencil map that is
// monotone (one branch) over the whole energy grid.
static bool zone_path_ok(const CellDev& c, const GridDev& g, int sharp, bool& rev) {
  const double w = sharp ? 0.0 : g.delta;
  const double hi_e = g.e0 + g.step * (g.npts - 1);
  const double margin = 8e-12 * std::max(1.0, std::max(std::fabs(g.e0), std::fabs(hi_e)));
  if (!(2.0 * (w + margin) < 0.95 * g.step)) return false;
  rev = (c.pencil == 1) && (c.t - c.s * c.eps0 < 0.0);
  if (c.pencil == 1) {
    // lambda(E) = (E - eps0) / (t - s E) stays on one branch: t - s E keeps its sign over the grid
    const double a = c.t - c.s * (g.e0 - w - 1.0), b = c.t - c.s * (hi_e + w + 1.0);
    if (!(a * b > 0.0)) return false;
    if ((c.t - c.s * c.eps0) * a <= 0.0) return false;
  }
  return (size_t)g.npts * 2 * sizeof(int) <= 96 * 1024;
}

// ------------------------------------------------------------------------------------------------
// Gram mode of the zone path (graphene IDOS batches reduced through G = C^T C, hx_gram.cuh): the tridiagonal is
// that of G (dimension S = the padded sublattice size: the m = min(nA, nB) values sigma^2 plus S - m zeros), not
// the TGK of C.  The eigenvalues of T = [[0, C], [C^T, 0]] (dimension d = nA + nB) are +-sigma plus d - 2m
// zeros, so for x away from 0
//     count_T(x) = d - S + count_G(x^2)   (x > 0),      count_T(x) = S - count_G(x^2)   (x < 0),
// and the zone eigenvalues are located in mu = sigma^2 (relative accuracy eps in mu = eps/2 in sigma) and mapped
// to lambda = +-sqrt(mu).  The host uses this mode only when no transition zone comes near lambda = 0, where
// sigma^2 loses its relative accuracy (gram_zones_ok).
// fuse != 0 (many-matrix launches, S < 1024): the block also locates its own zone eigenvalues, on a copy of the
// tridiagonal in shared memory (zone_locate with the arguments zone_refine_gram_kernel would pass: the same bits),
// instead of handing them to the global refinement list - the list's items of one warp belong to different
// matrices, so every Sturm row step of zone_refine_gram_kernel was 32 scattered loads (ncu: 10 of 14 stall cycles
// per issue on the long scoreboard, 9 of 32 lanes active).
// Dynamic shared memory: fuse: [2 S] doubles (diag, e2), then ints: [2 npts] T counts at the zone edges,
// [2 npts] Gram counts, fuse: [npts + 1] item offsets, [2 S] items.
__global__ void __launch_bounds__(256) zone_count_gram_kernel(CellDev c, int nk, GridDev g, int sharp, int rev,
                                                              int64_t mat0, int64_t nmat, const double* __restrict__ tri,
                                                              size_t tri_stride, const int* __restrict__ dims,
                                                              int* diff, RefineItem* refine,
                                                              unsigned long long* refine_count, int fuse,
                                                              unsigned long long* trans, int* status, int group) {
  // group > 0 (list mode): the matrix's items go to ONE contiguous range of the list, padded with invalid items
  // (idx < 0) to a multiple of `group` - every block of the staged multisection kernel then works on one matrix
  extern __shared__ __align__(16) unsigned char zraw[];
  __shared__ double red[3][32];
  __shared__ int wsum[8];
  __shared__ unsigned long long list_base;
  const int64_t lm = blockIdx.x;
  if (lm >= nmat) return;
  const int d = dims[lm];
  if (d <= 0) return;
  const int S = c.N, npts = g.npts;
  double* sd = reinterpret_cast<double*>(zraw);
  int* zc = reinterpret_cast<int*>(zraw + (fuse ? (size_t)2 * S * sizeof(double) : 0));
  int* zg = zc + 2 * npts;
  int* zoff = zg + 2 * npts;     // fuse / grouped list
  int* ilist = zoff + npts + 1;  // fuse only
  const int64_t mat = mat0 + lm;
  const int64_t mk = mat / nk;
  const double* diag = tri + lm * tri_stride;
  const double* e2 = diag + S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double gl = 1e308, gu = -1e308, em = 0.0;
  for (int i = tid; i < S; i += blockDim.x) {
    const double el = i > 0 ? sqrt(e2[i - 1]) : 0.0;
    const double er2 = i + 1 < S ? e2[i] : 0.0;
    const double er = sqrt(er2);
    gl = fmin(gl, diag[i] - el - er);
    gu = fmax(gu, diag[i] + el + er);
    em = fmax(em, er2);
    if (fuse) {
      sd[i] = diag[i];
      sd[S + i] = e2[i];
    }
  }
  gl = warp_min(gl);
  gu = warp_max(gu);
  em = warp_max(em);
  if (lane == 0) {
    red[0][warp] = gl;
    red[1][warp] = gu;
    red[2][warp] = em;
  }
  __syncthreads();
  gl = red[0][0];
  gu = red[1][0];
  em = red[2][0];
  for (int w = 1; w < nw; ++w) {
    gl = fmin(gl, red[0][w]);
    gu = fmax(gu, red[1][w]);
    em = fmax(em, red[2][w]);
  }
  const double pivmin = DBL_MIN * fmax(1.0, em);
  const double tnorm = fmax(fabs(gl), fabs(gu));
  gl = gl - 2.1 * tnorm * DBL_EPSILON * S - 4.2 * pivmin;
  gu = gu + 2.1 * tnorm * DBL_EPSILON * S + 4.2 * pivmin;
  const double* cd = fuse ? sd : diag;
  const double* ce2 = fuse ? sd + S : e2;
  for (int m = tid; m < npts; m += blockDim.x) {
    double la, lb;
    zone_bracket(c, g, sharp, m, la, lb);
    const bool pos = la > 0.0;
    const double xa = pos ? la * la : lb * lb, xb = pos ? lb * lb : la * la;  // mu bracket, xa < xb
    const bool ra = xa > gl && xa < gu, rb = xb > gl && xb < gu;
    int ca = xa <= gl ? 0 : S, cb = xb <= gl ? 0 : S;
    if (ra || rb) {
      int na, nb;
      sturm_count_pair<false>(cd, ce2, S, xa, xb, pivmin, na, nb);
      if (ra) ca = na;
      if (rb) cb = nb;
    }
    cb = max(ca, cb);
    zg[2 * m] = ca;
    zg[2 * m + 1] = cb;
    zc[2 * m] = pos ? d - S + ca : S - cb;
    zc[2 * m + 1] = pos ? d - S + cb : S - ca;
  }
  __syncthreads();
  int* drow = diff + mk * (npts + 1);
  if (fuse || group > 0) {
    zone_item_offsets(npts, zoff, wsum, [&](int m) { return zg[2 * m + 1] - zg[2 * m]; });
    if (!fuse) {
      const int total = zoff[npts], padded = (total + group - 1) / group * group;
      if (tid == 0) list_base = atomicAdd(refine_count, (unsigned long long)padded);
      __syncthreads();
      for (int q = total + tid; q < padded; q += blockDim.x)
        refine[list_base + q] = RefineItem{mat, lm, -1, 0, 0.0, 0.0, 0.0};
    }
  }
  for (int m = tid; m < npts; m += blockDim.x) {
    int n;
    if (!rev) n = zc[2 * m] - (m > 0 ? zc[2 * m - 1] : 0);
    else n = (m > 0 ? zc[2 * m - 2] : d) - zc[2 * m + 1];
    if (n > 0) atomicAdd(drow + m, n * kmul(g, mat, nk));
    const int i0 = zg[2 * m], nz = zg[2 * m + 1] - i0;
    if (nz > 0) {
      if (fuse) {
        const int o = zoff[m];
        for (int k = 0; k < nz; ++k) ilist[o + k] = m | (k << 16);
        continue;
      }
      double la, lb;
      zone_bracket(c, g, sharp, m, la, lb);
      const bool pos = la > 0.0;
      const double xa = pos ? la * la : lb * lb, xb = pos ? lb * lb : la * la;
      const unsigned long long p0 =
          group > 0 ? list_base + (unsigned long long)zoff[m] : atomicAdd(refine_count, (unsigned long long)nz);
      for (int k = 0; k < nz; ++k)
        refine[p0 + k] = RefineItem{mat, lm, i0 + k,
                                    (int)(1u | (pos ? 0u : 2u) | ((unsigned)k << 2) | ((unsigned)nz << 17)),
                                    fmax(xa, gl), fmin(xb, gu), pivmin};
    }
  }
  if (!fuse) return;
  __syncthreads();
  const int total = zoff[npts];
  for (int q = tid; q < total; q += blockDim.x) {
    const int il = ilist[q], m = il & 0xffff, k = il >> 16;
    double la, lb;
    zone_bracket(c, g, sharp, m, la, lb);
    const bool pos = la > 0.0;
    const double xa = pos ? la * la : lb * lb, xb = pos ? lb * lb : la * la;
    const int i0 = zg[2 * m], nz = zg[2 * m + 1] - i0;
    const double mu = zone_locate<false>(sd, sd + S, S, i0 + k, fmax(xa, gl), fmin(xb, gu), i0, i0 + nz, pivmin);
    const double sg = sqrt(fmax(mu, 0.0));
    add_eigenvalue(c, g, sharp, diff, trans, status, mat, nk, pos ? sg : -sg);
  }
}

// Gram zone eigenvalues in mu = sigma^2 on G's tridiagonal, lambda = +-sqrt(mu), for the launches that are not fused
// into zone_count_gram_kernel (launch_gram_idos chooses by the matrix size and the options only: batch-independent
// results).  G = 1: the bracketed Newton search of zone_locate, one thread per item - staged: on the grouped list,
// the block's matrix in shared memory (S >= 1024 by default), else on the scattered list with loads from L2
// (HX_ZONE_FUSE=0 / HX_ZONE_STAGE=0: same bits, 5.0 ms on the 64-matrix S = 1024 launch).  G > 1
// (HX_GRAM_REFINE_LANES, or a tridiagonal too large to stage): G-lane multisection, uniform control flow, every
// lane one Sturm count per round (2.1 ms unstaged / 1.45 ms staged with 8 lanes on that launch).
__global__ void __launch_bounds__(512) zone_refine_gram_kernel(CellDev c, int nk, GridDev g,
                                                               const double* __restrict__ tri, size_t tri_stride,
                                                               int* diff, unsigned long long* trans, int* status,
                                                               int sharp, const RefineItem* __restrict__ items,
                                                               const unsigned long long* __restrict__ count, int G,
                                                               int staged) {
  extern __shared__ __align__(16) double zsm_refine[];
  const unsigned long long n = *count;
  if (G > 1) {
    if (staged)
      refine_multisection_staged<false, true>(c, nk, g, tri, tri_stride, nullptr, diff, trans, status, sharp, items, n, G,
                                              zsm_refine);
    else
      refine_multisection<false, true>(c, nk, g, tri, tri_stride, nullptr, diff, trans, status, sharp, items, n, G);
    return;
  }
  const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
  const int S = c.N;
  if (staged) {
    // grouped list (group = blockDim.x): a block iteration = blockDim.x items of one matrix, its tridiagonal staged
    // in shared memory; one thread per item, the bracketed Newton search of zone_locate
    for (unsigned long long qb = (unsigned long long)blockIdx.x * blockDim.x; qb < n; qb += nthreads) {
      const RefineItem it = items[qb + threadIdx.x];
      const double* src = tri + items[qb].lm * tri_stride;
      __syncthreads();
      for (int i = threadIdx.x; i < 2 * S; i += blockDim.x) zsm_refine[i] = src[i];
      __syncthreads();
      if (it.idx < 0) continue;
      const unsigned f = (unsigned)it.flags;
      const int k = (int)((f >> 2) & 0x7fffu), nz = (int)(f >> 17);
      const int clo = it.idx - k;
      const double mu =
          zone_locate<false>(zsm_refine, zsm_refine + S, S, it.idx, it.lo, it.hi, clo, clo + nz, it.pivmin);
      const double sg = sqrt(fmax(mu, 0.0));
      add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, (f & 2u) ? -sg : sg);
    }
    return;
  }
  for (unsigned long long q = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += nthreads) {
    const RefineItem it = items[q];
    const double* diag = tri + it.lm * tri_stride;
    const unsigned f = (unsigned)it.flags;
    const int k = (int)((f >> 2) & 0x7fffu), nz = (int)(f >> 17);
    const int clo = it.idx - k;
    const double mu = zone_locate<false>(diag, diag + S, S, it.idx, it.lo, it.hi, clo, clo + nz, it.pivmin);
    const double sg = sqrt(fmax(mu, 0.0));
    add_eigenvalue(c, g, sharp, diff, trans, status, it.mat, nk, (f & 2u) ? -sg : sg);
  }
}

bool gram_zones_ok(const CellDev& c, const GridDev& g, int sharp, double lam_min) {
  bool rev = false;
  if (c.pencil != 1 || !zone_path_ok(c, g, sharp, rev)) return false;
  for (int m = 0; m < g.npts; ++m) {
    const double em = g.e0 + g.step * m;
    const double w = sharp ? 0.0 : g.delta;
    const double a = pencil_inv(c.pencil, c.eps0, c.t, c.s, em - w - 1e-9),
                 b = pencil_inv(c.pencil, c.eps0, c.t, c.s, em + w + 1e-9);
    if (!(a * b > 0.0) || std::fmin(std::fabs(a), std::fabs(b)) < lam_min) return false;
  }
  return true;
}

// Gram-mode eigenvalue stage (IDOS only): false if the zone path does not apply (the caller uses the TGK path).
bool launch_gram_idos(const CellDev& c, int nk, const GridDev& g, int64_t mat0, int64_t nmat, const double* tri,
                      size_t tri_stride, const int* dims, int* diff, unsigned long long* trans, int* status, int sharp,
                      cudaStream_t st, RefineItem* refine, unsigned long long* refine_count) {
  bool rev = false;
  if (!refine || !refine_count || !diff || !zone_path_ok(c, g, sharp, rev)) return false;
  NvtxRange nvtx_eig("eigenvalue stage (Gram zone path) S=%d nmat=%lld", c.N, (long long)nmat);
  // Refinement of the zone eigenvalues, a function of the matrix size (and the options) only - never of the batch:
  //   S < 1024: one thread per item (zone_locate: isolation + safeguarded Newton), fused into the count kernel on a
  //             shared-memory copy of the tridiagonal (HX_ZONE_FUSE=0: global item list, same bits);
  //   S >= 1024: the same per-thread search on the GROUPED item list, the block's matrix staged in shared memory
  //             (HX_ZONE_STAGE=0: loads from L2, same bits).  Per item ~11 Sturm counts instead of the 8 lanes x 13
  //             rounds of the multisection that the unstaged kernel needed to hide the L2 latency of its scattered
  //             loads (S = 1024, 64 matrices: 2.1 ms; staged multisection 1.45 ms at 67 % issue utilisation);
  //   HX_GRAM_REFINE_LANES = G > 1, or a tridiagonal too large to stage (S > 4096): G-lane multisection.
  const size_t stage_b = (size_t)2 * c.N * sizeof(double);
  const bool can_stage = stage_b <= 64 * 1024;
  const int lanes_opt = (int)opt("HX_GRAM_REFINE_LANES", 0);
  const int G = lanes_opt > 0 ? lanes_opt : (c.N >= 1024 && !can_stage ? 8 : 1);
  const int fuse = G == 1 && c.N < 1024 && opt("HX_ZONE_FUSE", 1) != 0 && g.npts < 65536;
  const int staged = !fuse && c.N >= 1024 && can_stage && 128 % G == 0 && opt("HX_ZONE_STAGE", 1) != 0;
  const int rthreads = !staged ? 128 : (stage_b <= 16 * 1024 ? 128 : (stage_b <= 32 * 1024 ? 256 : 512));
  const int group = staged ? rthreads / G : 0;
  const size_t zsm = (size_t)g.npts * 4 * sizeof(int) + (size_t)(g.npts + 1) * sizeof(int) +
                     (fuse ? (size_t)2 * c.N * (sizeof(double) + sizeof(int)) : 0);
  const int zt = g.npts >= 256 ? 256 : ((g.npts + 31) / 32) * 32;
  if (zsm > 200 * 1024) return false;
  set_smem_attr(zone_count_gram_kernel, zsm);
  if (!fuse) cudaMemsetAsync(refine_count, 0, sizeof(unsigned long long), st);
  zone_count_gram_kernel<<<(unsigned)nmat, zt, zsm, st>>>(c, nk, g, sharp, rev, mat0, nmat, tri, tri_stride, dims,
                                                           diff, refine, refine_count, fuse, trans, status, group);
  count_launch();
  if (!fuse) {
    if (staged) {
      set_smem_attr(zone_refine_gram_kernel, stage_b);
      const int per_sm = (int)std::min<size_t>(2048 / rthreads, (200 * 1024) / stage_b);
      zone_refine_gram_kernel<<<148 * per_sm, rthreads, stage_b, st>>>(c, nk, g, tri, tri_stride, diff, trans, status,
                                                                      sharp, refine, refine_count, G, 1);
    } else {
      zone_refine_gram_kernel<<<148 * 16, 128, 0, st>>>(c, nk, g, tri, tri_stride, diff, trans, status, sharp, refine,
                                                        refine_count, G, 0);
    }
    count_launch();
  }
  return true;
}




void launch_eig_idos(const CellDev& c, int nk, const GridDev& g, int64_t mat0, int64_t nmat, const double* tri,
                     size_t tri_stride, const int* dims, int* diff, unsigned long long* trans, double* eigs,
                     int* status, int sharp, cudaStream_t st, RefineItem* refine, unsigned long long* refine_count,
                     bool tgk) {
  NvtxRange nvtx_eig("eigenvalue stage N=%d nmat=%lld tgk=%d", c.N, (long long)nmat, (int)tgk);
  const int64_t per = tgk ? (c.N + 1) / 2 : c.N;
  const int64_t slots = nmat * per;
  const bool two_pass = refine && refine_count && diff && !eigs;
  if (two_pass) cudaMemsetAsync(refine_count, 0, sizeof(unsigned long long), st);
  bool rev = false;
  // zone path: 2 npts Sturm counts per matrix beat ~d/2 x 10 bisection steps from d ~ 96 on
  if (two_pass && c.N >= opt("HX_ZONE_MIN_N", 96) && zone_path_ok(c, g, sharp, rev)) {
    // per-thread refinement (N < 1024, refine_lanes): fused into the count kernel (HX_ZONE_FUSE=0: the item list)
    // refinement method by matrix size only, as launch_gram_idos: fused below N = 1024, the grouped list with the
    // matrix staged in shared memory from there (per-thread Newton), 4-lane multisection when the tridiagonal does
    // not fit (N > 4096) or with HX_REFINE_LANES = G > 1
    const size_t stage_b = (size_t)2 * c.N * sizeof(double);
    const bool can_stage = stage_b <= 64 * 1024;
    const int lanes_opt = (int)opt("HX_REFINE_LANES", 0);
    const int G = lanes_opt > 0 ? lanes_opt : (c.N >= g_refine_min_n && !can_stage ? 4 : 1);
    const int fuse = G == 1 && c.N < g_refine_min_n && opt("HX_ZONE_FUSE", 1) != 0 && g.npts < 65536;
    const int staged = !fuse && c.N >= g_refine_min_n && can_stage && 128 % G == 0 && opt("HX_ZONE_STAGE", 1) != 0;
    const int rthreads = !staged ? 128 : (stage_b <= 16 * 1024 ? 128 : (stage_b <= 32 * 1024 ? 256 : 512));
    const int group = staged ? rthreads / G : 0;
    const size_t zsm = (size_t)g.npts * 2 * sizeof(int) + (size_t)(g.npts + 1) * sizeof(int) +
                       (fuse ? (size_t)c.N * (2 * sizeof(double) + sizeof(int)) : 0);
    const int zt = g.npts >= 256 ? 256 : ((g.npts + 31) / 32) * 32;
    if (tgk) {
      set_smem_attr(zone_count_kernel<true>, zsm);
      zone_count_kernel<true><<<(unsigned)nmat, zt, zsm, st>>>(c, nk, g, sharp, rev, mat0, nmat, tri, tri_stride, dims,
                                                              diff, refine, refine_count, fuse, trans, status, group);
    } else {
      set_smem_attr(zone_count_kernel<false>, zsm);
      zone_count_kernel<false><<<(unsigned)nmat, zt, zsm, st>>>(c, nk, g, sharp, rev, mat0, nmat, tri, tri_stride, dims,
                                                               diff, refine, refine_count, fuse, trans, status, group);
    }
    count_launch();
    if (fuse) return;
    const int per_sm = staged ? (int)std::min<size_t>(2048 / rthreads, (200 * 1024) / stage_b) : 16;
    const int64_t rblocks = 148 * per_sm;
    const size_t rsm = staged ? stage_b : 0;
    if (tgk) {
      if (staged) set_smem_attr(zone_refine_kernel<true>, rsm);
      zone_refine_kernel<true><<<(unsigned)rblocks, rthreads, rsm, st>>>(c, nk, g, tri, tri_stride, dims, diff, trans,
                                                                        status, sharp, refine, refine_count, staged, G);
    } else {
      if (staged) set_smem_attr(zone_refine_kernel<false>, rsm);
      zone_refine_kernel<false><<<(unsigned)rblocks, rthreads, rsm, st>>>(c, nk, g, tri, tri_stride, dims, diff, trans,
                                                                         status, sharp, refine, refine_count, staged, G);
    }
    count_launch();
    return;
  }
  const unsigned blocks = (unsigned)((slots + 127) / 128);
  RefineItem* rf = two_pass ? refine : nullptr;
  if (tgk)
    eig_idos_kernel<true><<<blocks, 128, 0, st>>>(c, nk, g, mat0, nmat, tri, tri_stride, dims, diff, trans, eigs,
                                                  status, sharp, rf, refine_count);
  else
    eig_idos_kernel<false><<<blocks, 128, 0, st>>>(c, nk, g, mat0, nmat, tri, tri_stride, dims, diff, trans, eigs,
                                                   status, sharp, rf, refine_count);
  count_launch();
  if (two_pass) {
    // at least 148 x 16 blocks: when few items are left (large matrices) each gets a whole warp
    const int64_t rblocks = 148 * 16;
    if (tgk)
      eig_refine_kernel<true><<<(unsigned)rblocks, 128, 0, st>>>(c, nk, g, tri, tri_stride, dims, diff, trans, status,
                                                                 sharp, refine, refine_count);
    else
      eig_refine_kernel<false><<<(unsigned)rblocks, 128, 0, st>>>(c, nk, g, tri, tri_stride, dims, diff, trans,
                                                                  status, sharp, refine, refine_count);
    count_launch();
  }
}

// ------------------------------------------------------------------------------------------------
// Dense H(k), S(k) per (mask, k) into caller buffers (column-major N x N complex, leading d x d
// block valid, rest zero): assemble_bloch (tbmodel.py:277-293) on the device.
__global__ void __launch_bounds__(256) assemble_kernel(CellDev c, const double2* __restrict__ kpts, int nk,
                                                       const uint64_t* __restrict__ masks, double2* H, double2* S,
                                                       int* dims) {
  __shared__ int cnt[(HX_MAX_N + 31) / 32];
  extern __shared__ int new_idx[];
  const int N = c.N;
  const int64_t mat = blockIdx.x;
  const int64_t mk = mat / nk;
  const int kk = (int)(mat - mk * nk);
  double2* h = H + mat * (int64_t)N * N;
  double2* s = S ? S + mat * (int64_t)N * N : nullptr;
  for (int64_t p = threadIdx.x; p < (int64_t)N * N; p += blockDim.x) {
    h[p] = make_double2(0.0, 0.0);
    if (s) s[p] = make_double2(0.0, 0.0);
  }
  const int d = block_compact(c, masks + mk * c.words, new_idx, cnt);
  if (threadIdx.x == 0 && kk == 0) dims[mk] = d;
  if (d == 0) return;
  const double2 k = kpts[kk];
  assemble_full(c, new_idx, d, k, h, N, false);
  if (!s) return;
  if (c.pencil == 2) {
    assemble_full(c, new_idx, d, k, s, N, true);
  } else if (c.pencil == 1) {
    // h holds T: S = I + s T, H = eps0 I + t T
    for (int64_t p = threadIdx.x; p < (int64_t)d * d; p += blockDim.x) {
      const int col = (int)(p / d), row = (int)(p - (int64_t)col * d);
      const double2 tv = h[row + (int64_t)col * N];
      const double dg = row == col ? 1.0 : 0.0;
      s[row + (int64_t)col * N] = make_double2(dg + c.s * tv.x, c.s * tv.y);
      h[row + (int64_t)col * N] = make_double2(dg * c.eps0 + c.t * tv.x, c.t * tv.y);
    }
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) s[i + (int64_t)i * N] = make_double2(1.0, 0.0);
  }
}

// ------------------------------------------------------------------------------------------------
// Standalone matrices (hx_eigvalsh_batch_device): lower triangle of A -> packed smem -> (diag, e2).
__global__ void __launch_bounds__(512) eigvalsh_small_kernel(int n, const double2* __restrict__ A, double* tri,
                                                             int* dims, int* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = n | 1;
  double* R = reinterpret_cast<double*>(smem_raw);
  double2* v = reinterpret_cast<double2*>(R + (((size_t)n * ld + 1) & ~(size_t)1));
  double2* y = v + n;
  double* red = reinterpret_cast<double*>(y + n);
  const double2* a = A + (size_t)blockIdx.x * n * n;
  for (int p = threadIdx.x; p < n * n; p += blockDim.x) {
    const int col = p / n, row = p - col * n;
    const double2 z = a[p];
    if (row > col) {
      R[row * ld + col] = z.x;
      R[col * ld + row] = z.y;
    } else if (row == col) {
      R[row * ld + row] = z.x;
    }
  }
  if (threadIdx.x == 0) {
    status[blockIdx.x] = 0;
    dims[blockIdx.x] = n;
  }
  __syncthreads();
  double* diag = tri + (size_t)blockIdx.x * 2 * n;
  tridiag_packed(R, ld, n, diag, diag + n, v, y, red);
}

__global__ void __launch_bounds__(512) eigvalsh_global_kernel(int n, const double2* __restrict__ A,
                                                              const double2* __restrict__ B, int64_t mat0,
                                                              unsigned char* ws, size_t stride, double* tri,
                                                              int* dims, int* status) {
  __shared__ double red[96];
  const int64_t mat = mat0 + blockIdx.x;
  unsigned char* w = ws + (size_t)blockIdx.x * stride;
  double2* Aw = reinterpret_cast<double2*>(w);
  double2* Bw = Aw + (size_t)n * n;
  double2* v = B ? Bw + (size_t)n * n : Bw;
  double2* y = v + n;
  const double2* a = A + (size_t)mat * n * n;
  for (int64_t p = threadIdx.x; p < (int64_t)n * n; p += blockDim.x) Aw[p] = a[p];
  if (B) {
    const double2* b = B + (size_t)mat * n * n;
    for (int64_t p = threadIdx.x; p < (int64_t)n * n; p += blockDim.x) Bw[p] = b[p];
  }
  if (threadIdx.x == 0) {
    status[mat] = 0;
    dims[blockIdx.x] = n;
  }
  __syncthreads();
  if (B && !chol_reduce_full(Aw, Bw, n, n, red)) {
    if (threadIdx.x == 0) {
      status[mat] = 1;
      dims[blockIdx.x] = 0;
    }
    return;
  }
  double* diag = tri + (size_t)blockIdx.x * 2 * n;
  tridiag_full(Aw, n, n, diag, diag + n, v, y, red);
}

// ------------------------------------------------------------------------------------------------
// curves[mk][m] = (sum_{m' <= m} diff[mk][m'] + trans[mk][m] * 2^-shift) * inv_nk / area
__global__ void finalize_kernel(const int* diff, const unsigned long long* trans, int64_t nmasks, GridDev g,
                                double inv_nk, double inv_area, double* curves) {
  const int64_t mk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (mk >= nmasks) return;
  const int lane = threadIdx.x & 31;
  const int* dr = diff + mk * (g.npts + 1);
  const unsigned long long* tr = trans + mk * g.npts;
  const double sc = ldexp(1.0, -g.shift);
  long long carry = 0;
  for (int base = 0; base < g.npts; base += 32) {
    const int m = base + lane;
    long long x = m < g.npts ? dr[m] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    const long long cnt = carry + x;
    if (m < g.npts) {
      const double frac = (double)(long long)tr[m] * sc;
      curves[mk * g.npts + m] = ((double)cnt + frac) * inv_nk * inv_area;
    }
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

}  // namespace hx
