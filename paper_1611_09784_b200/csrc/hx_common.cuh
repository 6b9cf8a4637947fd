// Shared device helpers for libhx (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdio.h>

namespace hx {

// NVTX range over a host-side submission phase (tier / stage of a batch): shows the (tier, stage) structure of
// a step in Nsight Systems / ncu --nvtx; a no-op without an attached tool.
struct NvtxRange {
  template <class... A>
  explicit NvtxRange(const char* fmt, A... a) {
    char buf[96];
    snprintf(buf, sizeof buf, fmt, a...);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Number of libhx kernel launches issued by this process (reported by bench.py as gpu_launches).
void count_launch(unsigned long long n = 1);

// Tuning / path-selection knobs (HX_*): a value set through hx_set_option() wins, else the environment
// variable of the same name, else `dflt`.  Read at every batch call, so tests can force each kernel
// variant in-process (hx_capi.cu).
long opt(const char* name, long dflt);

// Compiled-cell tables resident in HBM (uploaded once per (model, nu)).
struct CellDev {
  int32_t N;          // total dofs
  int32_t nunits;     // removable units
  int32_t words;      // uint64 words per mask
  int32_t pencil;     // HX_PENCIL_*
  double eps0, t, s;  // commuting-pencil parameters
  double area;
  const int32_t* unit_of_dof;  // [N]
  const double* onsite;        // [N]
  // hopping CSR by source dof, and its transpose (instances grouped by target dof, instance order)
  const int32_t* h_ptr;
  const int32_t* h_col;
  const double2* h_amp;
  const double2* h_disp;
  const int32_t* ht_ptr;   // [N+1]
  const int32_t* ht_inst;  // instance ids with dst == row, ascending
  const int32_t* h_src;    // [nnz] source dof of each instance
  // overlap (HX_PENCIL_GENERAL)
  const int32_t* s_ptr;
  const int32_t* s_col;
  const double2* s_amp;
  const double2* s_disp;
  const int32_t* st_ptr;
  const int32_t* st_inst;
  const int32_t* s_src;
  // bipartite commuting pencil (graphene): every hop joins sublattice 0 and 1 -> T = [[0, C], [C^H, 0]]
  int32_t bipartite;
  int32_t nsub;        // max dofs on one sublattice
  const int32_t* sub;  // [N] sublattice of each dof
  const double2* pos;  // [N] Cartesian site position of each dof (periodic gauge), or nullptr
};

struct GridDev {
  double e0, step, delta;
  int32_t npts;
  int32_t shift;     // fixed-point fraction bits of the transition accumulator
  double inv_step;   // 1 / step: only for the (eta-widened) early-settle test, never for contributions
  const int* kmult;  // device: multiplicity of each k-point of the batch (time-reversal pairs), or nullptr
};

// Multiplicity of matrix `mat` (= mask * nk + k) in the IDOS sums.
__device__ __forceinline__ int kmul(const GridDev& g, int64_t mat, int nk) {
  return g.kmult ? g.kmult[mat % nk] : 1;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Warp-level sum of a double.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Dynamic shared memory limit of a kernel.  (Forcing the maximum shared-memory carveout as well was
// measured slower: the bulge chase and the rank update lose more to the smaller L1 than they gain from
// extra resident CTAs.)
// The limit is only ever RAISED, under a lock, per (device, kernel) (raise_smem_attr, hx_capi.cu): contexts on
// several host threads launch the same kernels with different dynamic sizes (e.g. the zone kernels stage tridiagonals
// of different S); setting the exact size per launch let one thread lower the limit between another thread's
// set and launch ("invalid argument" on that launch).
void raise_smem_attr(const void* kernel, size_t bytes);
template <typename K>
inline void set_smem_attr(K* kernel, size_t bytes) {
  raise_smem_attr(reinterpret_cast<const void*>(kernel), bytes);
}

}  // namespace hx
