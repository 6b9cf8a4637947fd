// Kernel declarations shared between the launch layer (hx_capi.cu) and the kernel TUs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hx_common.cuh"

#define HX_SMEM_MAX_N 160   // largest N held entirely in shared memory (real-packed Hermitian)
#define HX_MAX_N 16384      // envelope of the global-memory path

namespace hx {

__global__ void fused_smem_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, GridDev g, int* diff,
                                  unsigned long long* trans, double* eigs, int* status, int sharp);
size_t fused_smem_bytes(int N);

__global__ void global_solve_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, GridDev g, int* diff,
                                    unsigned long long* trans, double* eigs, int* status, int64_t mat0,
                                    unsigned char* ws, size_t ws_stride, int sharp);
size_t global_ws_stride(int N, bool general);

__global__ void assemble_kernel(CellDev c, const double2* kpts, int nk, const uint64_t* masks, double2* H, double2* S,
                                int* dims);

__global__ void finalize_kernel(const int* diff, const unsigned long long* trans, int64_t nmasks, GridDev g,
                                double inv_nk, double inv_area, double* curves);

}  // namespace hx
