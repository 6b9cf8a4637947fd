// Kernel declarations shared between the launch layer (hx_capi.cu) and the kernel TUs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "hx_common.cuh"

#define HX_SMEM_MAX_N 160   // largest N held entirely in shared memory (real-packed Hermitian)
#define HX_MAX_N 16384      // envelope of the global-memory path

namespace hx {

// an eigenvalue bracket handed from the bisection pass to the dense refinement pass
struct RefineItem {
  int64_t mat;  // global matrix index (mask * nk + k)
  int64_t lm;   // chunk-local matrix index (tri / dims row)
  int idx;      // eigenvalue index
  int flags;    // bit 0: contribute lambda; bit 1: contribute -lambda (TGK mirror)
  double lo, hi, pivmin;
};

// tridiagonalisation tiers: write (diag[N], e2[N]) per matrix into `tri` (2N doubles per matrix)
__global__ void small_tridiag_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, double* tri,
                                     int* dims, int* status);
size_t small_tridiag_smem(int N);
// klist / nks (optional): the launch covers k-points klist[0..nks) of every mask; real: those k-points make the
// periodic-gauge block real (real Golub-Kahan)
__global__ void small_bidiag_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, double* tri,
                                    int* dims, int* status, const int* klist, int nks, int real);
size_t small_bidiag_smem(int N, int S);
size_t small_bidiag_smem_real(int N, int S, bool warp);
// complex k-points, S <= 64: matrix in registers of 256 threads (hx_bidiag.cuh bidiag_tgk_reg)
constexpr int BIDIAG_REG_THREADS = 256;
__global__ void small_bidiag_reg_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, double* tri,
                                        int* dims, int* status, const int* klist, int nks);
size_t small_bidiag_reg_smem(int N, int S);
// real (TRIM) k-points from klist, S <= 64: matrix in registers of 256 threads (bidiag_tgk_reg_real)
__global__ void small_bidiag_reg_real_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks,
                                             double* tri, int* dims, int* status, const int* klist, int nks);
size_t small_bidiag_reg_real_smem(int N, int S);

// Gram path of the S in (32, 64] tiers (hx_smallgram.cuh): tridiagonal (diag[S], e2[S]) of G = C^H C per matrix at
// tri + mat * 2N, for launch_gram_idos with a cell of N = S; klist == NULL: every k-point
__global__ void small_gram_reg_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, double* tri,
                                      int* dims, int* status, const int* klist, int nks);
__global__ void small_gram_reg_real_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks,
                                           double* tri, int* dims, int* status, const int* klist, int nks);
size_t small_gram_reg_smem(int N, int S, bool real);

__global__ void global_tridiag_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, int64_t mat0,
                                      unsigned char* ws, size_t ws_stride, double* tri, int* dims, int* status);
size_t global_ws_stride(int N, bool general);

// eigenvalues (bisection, thread per eigenvalue) + pencil map + IDOS accumulation + eigenvalue output
__global__ void assemble_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, double2* H, double2* S,
                                int* dims);

__global__ void eigvalsh_small_kernel(int n, const double2* A, double* tri, int* dims, int* status);
__global__ void eigvalsh_global_kernel(int n, const double2* A, const double2* B, int64_t mat0, unsigned char* ws,
                                       size_t stride, double* tri, int* dims, int* status);

__global__ void finalize_kernel(const int* diff, const unsigned long long* trans, int64_t nmasks, GridDev g,
                                double inv_nk, double inv_area, double* curves);

// Eigenvalue stage over `nmat` matrices starting at global index mat0.  With a refinement buffer
// (capacity >= nmat * N items) and no eigenvalue output, eigenvalues that settle into a gap between
// transition windows stop early and the rest are finished by a densely packed second pass.  tgk: the
// tridiagonals are Golub-Kahan (zero diagonal, spectrum symmetric about 0): one thread per +-pair.
// smallest N that takes the zone path of the eigenvalue stage (HX_ZONE_MIN_N; 0 = always)

// Gram mode (hx_kernels.cu): zone path on the tridiagonal of G = C^T C; false if it does not apply.
bool gram_zones_ok(const CellDev& c, const GridDev& g, int sharp, double lam_min);
bool launch_gram_idos(const CellDev& c, int nk, const GridDev& g, int64_t mat0, int64_t nmat, const double* tri,
                      size_t tri_stride, const int* dims, int* diff, unsigned long long* trans, int* status, int sharp,
                      cudaStream_t st, RefineItem* refine, unsigned long long* refine_count);
void launch_eig_idos(const CellDev& c, int nk, const GridDev& g, int64_t mat0, int64_t nmat, const double* tri,
                     size_t tri_stride, const int* dims, int* diff, unsigned long long* trans, double* eigs,
                     int* status, int sharp, cudaStream_t st, RefineItem* refine = nullptr,
                     unsigned long long* refine_count = nullptr, bool tgk = false);

}  // namespace hx
