// Large-N two-stage path (dense -> band -> tridiagonal) for batched Hermitian eigenvalues.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>

#include "hx_common.cuh"
#include "hx_kernels.cuh"

namespace hx {

using Alloc = std::function<void*(size_t)>;

void band_init_attributes();
bool band_path_supported(int N);
const char* band_last_error();

// IDOS batch through the banded path (pencil STANDARD or COMMUTING).
int band_eval(const CellDev& c, const double2* kp, int nk, const uint64_t* masks, int64_t nmasks, const GridDev& g,
              int* diff, unsigned long long* trans, double* eigs, int* status, int sharp, size_t ws_budget,
              const Alloc& alloc, cudaStream_t st, RefineItem* refine, unsigned long long* refine_count);

// Eigenvalues of caller-provided Hermitian matrices (column-major complex, n x n each); B != nullptr: the
// generalized problem A x = lambda B x (Cholesky of B, as the general-pencil tier).
int band_eigvalsh(int n, int64_t batch, const double2* A, const double2* B, double* eigs, int* status,
                  size_t ws_budget, const Alloc& alloc, cudaStream_t st);

// Hermitian two-stage reduction of caller-assembled matrices (the complex Gram path of the bipartite tier): slab
// layout of one n x n matrix (offsets in double2 units) and the reduction dense -> band -> tridiagonal
// (diag[n], e2[n] doubles at dg_off); dims[m] = size of the leading nonzero block of matrix m.
struct HermSlab {
  size_t a_off, scratch_off, scratch_len, dg_off, stride;
};
HermSlab herm_slab(int n);
int herm_reduce(double2* ws, int n, int64_t cnt, const int* dims, cudaStream_t st);

// Bipartite (graphene) banded tier: singular values of the A-B block (hx_bdband.cu).
void bd_init_attributes();
bool bd_path_supported(const CellDev& c);
const char* bd_last_error();
int bd_eval(const CellDev& c, const double2* kp, int nk, const uint64_t* masks, int64_t nmasks, const GridDev& g,
            int* diff, unsigned long long* trans, double* eigs, int* status, int sharp, bool real,
            size_t ws_budget, const Alloc& alloc, cudaStream_t st, RefineItem* refine,
            unsigned long long* refine_count);

}  // namespace hx
