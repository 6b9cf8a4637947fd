// C-ABI layer of libhx.so (see include/hx.h for the contract and the reference seams replaced).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/hx.h"
#include "hx_band.cuh"
#include "hx_dense.cuh"
#include "hx_kernels.cuh"
#include "hx_rng.cuh"
#include "hx_fixed.cuh"

#include <atomic>

namespace hx {
static std::atomic<unsigned long long> g_launches{0};
void count_launch(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void raise_smem_attr(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> limit;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = limit[{dev, kernel}];
  if (bytes > cur) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cur = bytes;
  }
}

namespace {
std::mutex g_opt_mu;
std::map<std::string, long> g_opts;
}  // namespace

long opt(const char* name, long dflt) {
  {
    std::lock_guard<std::mutex> lk(g_opt_mu);
    auto it = g_opts.find(name);
    if (it != g_opts.end()) return it->second;
  }
  const char* e = getenv(name);
  return e && e[0] ? atol(e) : dflt;
}
}  // namespace hx

namespace {

// general pencils above the shared-memory tier: Cholesky + the two-stage banded path (HX_GENERAL_BAND=0: the
// single-CTA global-memory kernel)
bool general_band() { return hx::opt("HX_GENERAL_BAND", 1) != 0; }

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define HX_CUDA(call)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return fail(HX_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int grow(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max(bytes, (size_t)4096);
    if (cudaMalloc(&p, want) != cudaSuccess) return -1;
    cap = want;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Pinned host staging buffer: host-API copies go through it so that they are true asynchronous DMA on the
// context's stream (pageable copies are staged by the driver and were measured to hold a small tier's
// results back until the concurrent large tier finished).  `ev` marks the last copy that reads it.
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  int grow(size_t bytes) {
    if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return -1;
    cudaEventSynchronize(ev);  // the previous copy from / to this buffer has completed
    if (bytes <= cap) return 0;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max(bytes, (size_t)4096);
    if (cudaHostAlloc(&p, want, cudaHostAllocPortable) != cudaSuccess) return -1;
    cap = want;
    return 0;
  }
  void release() {
    if (p) cudaFreeHost(p);
    if (ev) cudaEventDestroy(ev);
    p = nullptr;
    ev = nullptr;
    cap = 0;
  }
};

}  // namespace

struct hx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  DevBuf kpts, kmult, diff, trans, ws, masks, curves, eigs, status, band, tri, refine;
  HostBuf h_kpts, h_io;  // pinned staging: k-points (+ lists, multiplicities); masks in / curves + status out
  size_t ws_budget = (size_t)24 << 30;  // HBM workspace budget for the global / banded paths
  int bd_min_n = HX_SMEM_MAX_N;          // bipartite cells with N above this take the banded SVD tier
  int bidiag_warp_max_s = 32;            // shared-memory bidiagonalisation: one warp per matrix up to this S
  int bidiag_threads = 256;              // ... and a CTA of this size above it
  int bidiag_real_warp_max_s = 64;       // real (time-reversal-invariant) k-points: one warp per matrix up to this S
  bool bidiag_reg = true;                // register-resident reduction for complex S in (warp max, 64]
  bool bidiag_real = true;               // real Golub-Kahan for those k-points (HX_BIDIAG_REAL=0 disables)
  bool use_bipartite = true;            // graphene: singular values of the A-B block (HX_NO_BIPARTITE=1 disables)
  size_t ws_budget_default = ws_budget;
};

namespace {
// Path-selection knobs of a context, re-read from the option registry at every batch call (hx::opt).
void refresh_opts(hx_ctx* ctx) {
  ctx->use_bipartite = hx::opt("HX_NO_BIPARTITE", 0) == 0;
  ctx->bd_min_n = (int)hx::opt("HX_BD_MIN_N", HX_SMEM_MAX_N);
  ctx->bidiag_warp_max_s = (int)hx::opt("HX_BIDIAG_WARP_MAX_S", 32);
  ctx->bidiag_threads = (int)hx::opt("HX_BIDIAG_THREADS", 256);
  ctx->bidiag_real = hx::opt("HX_BIDIAG_REAL", 1) != 0;
  ctx->bidiag_reg = hx::opt("HX_BIDIAG_REG", 1) != 0;
  ctx->bidiag_real_warp_max_s = (int)hx::opt("HX_BIDIAG_REAL_WARP_MAX_S", 64);
  // experiments: workspace chunk budget in MB (L2-resident chunks)
  const long wb = hx::opt("HX_WS_BUDGET_MB", 0);
  ctx->ws_budget = wb > 0 ? (size_t)wb << 20 : ctx->ws_budget_default;
}
}  // namespace

struct hx_cell {
  hx_ctx* ctx = nullptr;
  hx::CellDev dev{};
  std::vector<void*> allocs;
  // periodic-gauge realness: real amplitudes and the lattice translation R of every hop (host copy)
  bool real_amps = false;
  std::vector<double> lat;  // [2 * nnz] R = disp - (pos_dst - pos_src)
};

namespace {
// All k-points make the periodic-gauge matrix real: exp(2i k.R) = 1 for every hop's lattice translation.
bool batch_is_real(const hx_cell* cell, const double* kpoints, int nk) {
  if (!cell->real_amps || !cell->dev.pos || cell->lat.empty()) return false;
  const size_t nnz = cell->lat.size() / 2;
  for (int k = 0; k < nk; ++k)
    for (size_t e = 0; e < nnz; ++e) {
      const double ph = 2.0 * (kpoints[2 * k] * cell->lat[2 * e] + kpoints[2 * k + 1] * cell->lat[2 * e + 1]);
      if (std::fabs(std::sin(ph)) > 1e-9 || std::cos(ph) < 0.0) return false;
    }
  return true;
}

// One k-point makes the periodic-gauge matrix real (per-k version of batch_is_real).
bool k_is_real(const hx_cell* cell, const double* kpoints, int k) {
  if (!cell->real_amps || !cell->dev.pos || cell->lat.empty()) return false;
  const size_t nnz = cell->lat.size() / 2;
  for (size_t e = 0; e < nnz; ++e) {
    const double ph = 2.0 * (kpoints[2 * k] * cell->lat[2 * e] + kpoints[2 * k + 1] * cell->lat[2 * e + 1]);
    if (std::fabs(std::sin(ph)) > 1e-9 || std::cos(ph) < 0.0) return false;
  }
  return true;
}
}  // namespace

namespace {

int set_device(hx_ctx* ctx) {
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return fail(HX_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return 0;
}

template <class T>
int upload(hx_cell* cell, const T* host, size_t n, const T** out) {
  *out = nullptr;
  if (host == nullptr || n == 0) return 0;
  void* p = nullptr;
  HX_CUDA(cudaMalloc(&p, n * sizeof(T)));
  cell->allocs.push_back(p);
  HX_CUDA(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
  *out = static_cast<const T*>(p);
  return 0;
}

// Transposed instance lists: for each target dof, the instance ids pointing at it (ascending).
void transpose_csr(int N, const int32_t* ptr, const int32_t* col, std::vector<int32_t>& tptr,
                   std::vector<int32_t>& tinst, std::vector<int32_t>& src) {
  const int nnz = ptr[N];
  tptr.assign(N + 1, 0);
  src.resize(nnz);
  for (int r = 0; r < N; ++r)
    for (int e = ptr[r]; e < ptr[r + 1]; ++e) {
      src[e] = r;
      tptr[col[e] + 1]++;
    }
  for (int r = 0; r < N; ++r) tptr[r + 1] += tptr[r];
  tinst.assign(nnz, 0);
  std::vector<int32_t> fill(tptr.begin(), tptr.end() - 1);
  for (int e = 0; e < nnz; ++e) tinst[fill[col[e]]++] = e;
}

// periodic-gauge real arithmetic for TRIM batches (HX_NO_REAL=1 disables)
bool real_batches() { return hx::opt("HX_NO_REAL", 0) == 0; }

int fixed_point_shift(int64_t nk, int N) {
  const double terms = (double)nk * (double)(N + 1) + 1.0;
  int need = (int)std::ceil(std::log2(terms));
  return std::min(52, 62 - need);
}

}  // namespace

extern "C" {

int hx_abi_version(void) { return HX_ABI_VERSION; }

int hx_set_option(const char* name, int64_t value) {
  if (!name || std::strncmp(name, "HX_", 3) != 0) return fail(HX_E_ARG, "option names start with HX_");
  std::lock_guard<std::mutex> lk(hx::g_opt_mu);
  hx::g_opts[name] = (long)value;
  return 0;
}

int hx_clear_option(const char* name) {
  std::lock_guard<std::mutex> lk(hx::g_opt_mu);
  if (name) hx::g_opts.erase(name);
  else hx::g_opts.clear();
  return 0;
}

int hx_get_option(const char* name, int64_t dflt, int64_t* out) {
  if (!name || !out) return fail(HX_E_ARG, "null argument");
  *out = hx::opt(name, (long)dflt);
  return 0;
}

int hx_kernel_launches(uint64_t* out) {
  if (!out) return fail(HX_E_ARG, "null out");
  *out = hx::g_launches.load();
  return 0;
}

const char* hx_last_error(void) { return g_err.c_str(); }

int hx_device_count(int32_t* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return fail(HX_E_NODEV, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *out = n;
  return 0;
}

int hx_ctx_create(int32_t device, hx_ctx** out) { return hx_ctx_create_priority(device, 0, out); }

int hx_ctx_create_priority(int32_t device, int32_t priority, hx_ctx** out) {
  if (!out) return fail(HX_E_ARG, "hx_ctx_create: null out");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(HX_E_NODEV, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(HX_E_ARG, "device index out of range");
  hx_ctx* ctx = new hx_ctx();
  ctx->device = device;
  if (set_device(ctx)) {
    delete ctx;
    return HX_E_CUDA;
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    delete ctx;
    return fail(HX_E_NODEV, "libhx is built for sm_100a (B200); found sm_" + std::to_string(prop.major) +
                                std::to_string(prop.minor));
  }
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  const int prio = std::max(hi_prio, std::min(lo_prio, (int)priority));
  if (cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, prio) != cudaSuccess) {
    delete ctx;
    return fail(HX_E_CUDA, "cudaStreamCreate failed");
  }
  size_t freeb = 0, total = 0;
  cudaMemGetInfo(&freeb, &total);
  hx::set_smem_attr(hx::small_bidiag_kernel, 200 * 1024);
  hx::set_smem_attr(hx::small_bidiag_reg_kernel, (int)hx::small_bidiag_reg_smem(128, 64));
  hx::set_smem_attr(hx::small_bidiag_reg_real_kernel, (int)hx::small_bidiag_reg_real_smem(128, 64));
  hx::set_smem_attr(hx::small_gram_reg_kernel, (int)hx::small_gram_reg_smem(128, 64, false));
  hx::set_smem_attr(hx::small_gram_reg_real_kernel, (int)hx::small_gram_reg_smem(128, 64, true));
  ctx->ws_budget = std::min(ctx->ws_budget, freeb / 3);
  ctx->ws_budget_default = ctx->ws_budget;
  refresh_opts(ctx);
  hx::set_smem_attr(hx::small_tridiag_kernel, (int)hx::small_tridiag_smem(HX_SMEM_MAX_N));
  hx::set_smem_attr(hx::eigvalsh_small_kernel, (int)hx::small_tridiag_smem(HX_SMEM_MAX_N));
  hx::band_init_attributes();
  hx::bd_init_attributes();
  *out = ctx;
  return 0;
}

int hx_ctx_destroy(hx_ctx* ctx) {
  if (!ctx) return 0;
  set_device(ctx);
  for (DevBuf* b : {&ctx->kpts, &ctx->kmult, &ctx->diff, &ctx->trans, &ctx->ws, &ctx->masks, &ctx->curves, &ctx->eigs,
                    &ctx->status, &ctx->band, &ctx->tri, &ctx->refine})
    b->release();
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->h_kpts.release();
  ctx->h_io.release();
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return 0;
}

int hx_ctx_synchronize(hx_ctx* ctx) {
  if (!ctx) return fail(HX_E_ARG, "null ctx");
  if (set_device(ctx)) return HX_E_CUDA;
  HX_CUDA(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int hx_cell_create(hx_ctx* ctx, const hx_cell_desc* d, hx_cell** out) {
  if (!ctx || !d || !out) return fail(HX_E_ARG, "hx_cell_create: null argument");
  if (d->ndof < 1 || d->ndof > HX_MAX_N) return fail(HX_E_RANGE, "ndof outside [1, HX_MAX_N]");
  if (d->nunits < 0 || !d->unit_of_dof || !d->onsite || !d->h_row_ptr) return fail(HX_E_ARG, "incomplete cell");
  if (d->pencil < 0 || d->pencil > 2) return fail(HX_E_ARG, "unknown pencil kind");
  if (d->pencil == HX_PENCIL_GENERAL && !d->s_row_ptr) return fail(HX_E_ARG, "general pencil needs overlap CSR");
  if (set_device(ctx)) return HX_E_CUDA;
  hx_cell* cell = new hx_cell();
  cell->ctx = ctx;
  hx::CellDev& c = cell->dev;
  const int N = d->ndof;
  c.N = N;
  c.nunits = d->nunits;
  c.words = (d->nunits + 63) / 64;
  if (c.words == 0) c.words = 1;
  c.pencil = d->pencil;
  c.eps0 = d->eps0;
  c.t = d->t;
  c.s = d->s;
  c.area = d->area;
  int rc = 0;
  rc |= upload(cell, d->unit_of_dof, N, &c.unit_of_dof);
  c.bipartite = 0;
  c.nsub = 0;
  if (d->sublattice && d->pencil == HX_PENCIL_COMMUTING) {
    bool ok = true;
    int n0 = 0, n1 = 0;
    for (int r = 0; r < N; ++r) {
      const int sr = d->sublattice[r];
      if (sr != 0 && sr != 1) ok = false;
      (sr == 0 ? n0 : n1) += 1;
      for (int e = d->h_row_ptr[r]; e < d->h_row_ptr[r + 1]; ++e) ok &= d->sublattice[d->h_col[e]] != sr;
    }
    if (ok) {
      c.bipartite = 1;
      c.nsub = std::max(n0, n1);
      rc |= upload(cell, d->sublattice, N, &c.sub);
    }
  }
  rc |= upload(cell, d->onsite, N, &c.onsite);
  c.pos = nullptr;
  if (d->dof_pos && d->pencil != HX_PENCIL_GENERAL) {
    rc |= upload(cell, reinterpret_cast<const double2*>(d->dof_pos), N, &c.pos);
    const int nnz = d->h_row_ptr[N];
    bool real = true;
    for (int r = 0; r < N; ++r) real &= d->onsite[r] == d->onsite[r];
    cell->lat.resize((size_t)2 * nnz);
    for (int r = 0; r < N; ++r)
      for (int e = d->h_row_ptr[r]; e < d->h_row_ptr[r + 1]; ++e) {
        const int dst = d->h_col[e];
        real &= d->h_amp[2 * e + 1] == 0.0;
        cell->lat[2 * e] = d->h_disp[2 * e] - (d->dof_pos[2 * dst] - d->dof_pos[2 * r]);
        cell->lat[2 * e + 1] = d->h_disp[2 * e + 1] - (d->dof_pos[2 * dst + 1] - d->dof_pos[2 * r + 1]);
      }
    cell->real_amps = real;
  }
  {
    const int nnz = d->h_row_ptr[N];
    std::vector<int32_t> tptr, tinst, src;
    transpose_csr(N, d->h_row_ptr, d->h_col, tptr, tinst, src);
    rc |= upload(cell, d->h_row_ptr, N + 1, &c.h_ptr);
    rc |= upload(cell, d->h_col, nnz, &c.h_col);
    rc |= upload(cell, reinterpret_cast<const double2*>(d->h_amp), nnz, &c.h_amp);
    rc |= upload(cell, reinterpret_cast<const double2*>(d->h_disp), nnz, &c.h_disp);
    rc |= upload(cell, tptr.data(), N + 1, &c.ht_ptr);
    rc |= upload(cell, tinst.data(), nnz, &c.ht_inst);
    rc |= upload(cell, src.data(), nnz, &c.h_src);
    if (nnz == 0) {
      // keep non-null pointers for the empty instance list
      static const int32_t zero = 0;
      (void)zero;
    }
  }
  if (d->pencil == HX_PENCIL_GENERAL) {
    const int nnz = d->s_row_ptr[N];
    std::vector<int32_t> tptr, tinst, src;
    transpose_csr(N, d->s_row_ptr, d->s_col, tptr, tinst, src);
    rc |= upload(cell, d->s_row_ptr, N + 1, &c.s_ptr);
    rc |= upload(cell, d->s_col, nnz, &c.s_col);
    rc |= upload(cell, reinterpret_cast<const double2*>(d->s_amp), nnz, &c.s_amp);
    rc |= upload(cell, reinterpret_cast<const double2*>(d->s_disp), nnz, &c.s_disp);
    rc |= upload(cell, tptr.data(), N + 1, &c.st_ptr);
    rc |= upload(cell, tinst.data(), nnz, &c.st_inst);
    rc |= upload(cell, src.data(), nnz, &c.s_src);
  }
  if (rc) {
    hx_cell_destroy(cell);
    return HX_E_CUDA;
  }
  *out = cell;
  return 0;
}

int hx_cell_destroy(hx_cell* cell) {
  if (!cell) return 0;
  if (cell->ctx) set_device(cell->ctx);
  for (void* p : cell->allocs) cudaFree(p);
  delete cell;
  return 0;
}

// kmult (host, optional): multiplicity of each k-point (time-reversal pairs merged by the caller); the IDOS
// weights become kmult[k] / sum(kmult) instead of 1 / nk.
static int eval_impl(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk, const uint64_t* d_masks,
                     int64_t nmasks, const hx_egrid* grid, double* d_curves, double* d_eigs, int32_t* d_status,
                     cudaStream_t st, int sharp, const int32_t* kmult = nullptr) {
  if (!ctx || !cell || !kpoints || !grid || (nmasks > 0 && (!d_masks || !d_curves || !d_status)))
    return fail(HX_E_ARG, "hx_eval_idos_batch: null argument");
  if (nk < 1 || nmasks < 0) return fail(HX_E_ARG, "hx_eval_idos_batch: nk >= 1 and nmasks >= 0 required");
  if (grid->npts < 1 || !(grid->step > 0.0) || !(grid->delta > 0.0))
    return fail(HX_E_ARG, "energy grid needs npts >= 1, step > 0, delta > 0");
  if (nmasks == 0) return 0;
  if (set_device(ctx)) return HX_E_CUDA;
  refresh_opts(ctx);
  const hx::CellDev& c = cell->dev;
  const int N = c.N;
  hx::NvtxRange nvtx_batch("hx_eval_idos_batch N=%d nk=%d masks=%lld", N, (int)nk, (long long)nmasks);
  int64_t nk_total = nk;
  if (kmult) {
    if (d_eigs) return fail(HX_E_ARG, "k-point multiplicities need the IDOS-only call (no eigenvalue output)");
    nk_total = 0;
    for (int k = 0; k < nk; ++k) {
      if (kmult[k] < 1) return fail(HX_E_ARG, "k-point multiplicities must be >= 1");
      nk_total += kmult[k];
    }
  }
  hx::GridDev g{};
  g.e0 = grid->e0;
  g.step = grid->step;
  g.delta = grid->delta;
  g.npts = grid->npts;
  g.shift = fixed_point_shift(nk_total, N);
  g.inv_step = 1.0 / g.step;
  g.kmult = nullptr;
  if (g.shift < 16) return fail(HX_E_RANGE, "nk * N too large for the fixed-point IDOS accumulator");
  // k-points (small, pageable copy on the work stream)
  // followed by the k-point lists of the shared-memory bipartite tier: complex k-points, then those whose
  // periodic-gauge block is real (time-reversal-invariant: real Golub-Kahan, one warp per matrix)
  std::vector<int> klist_c, klist_r;
  if (c.bipartite && ctx->use_bipartite && real_batches() && ctx->bidiag_real)
    for (int k = 0; k < nk; ++k) (k_is_real(cell, kpoints, k) ? klist_r : klist_c).push_back(k);
  // one pinned staging copy carries k-points, k lists and multiplicities
  const size_t kbytes = (size_t)nk * 24;
  if (ctx->h_kpts.grow(kbytes)) return fail(HX_E_CUDA, "alloc pinned kpts");
  unsigned char* kbuf = static_cast<unsigned char*>(ctx->h_kpts.p);
  std::memcpy(kbuf, kpoints, (size_t)nk * 16);
  if (!klist_r.empty()) {
    std::memcpy(kbuf + (size_t)nk * 16, klist_c.data(), klist_c.size() * 4);
    std::memcpy(kbuf + (size_t)nk * 16 + klist_c.size() * 4, klist_r.data(), klist_r.size() * 4);
  }
  if (kmult) std::memcpy(kbuf + (size_t)nk * 20, kmult, (size_t)nk * 4);
  if (ctx->kpts.grow(kbytes)) return fail(HX_E_CUDA, "alloc kpts");
  HX_CUDA(cudaMemcpyAsync(ctx->kpts.p, kbuf, kbytes, cudaMemcpyHostToDevice, st));
  HX_CUDA(cudaEventRecord(ctx->h_kpts.ev, st));
  const int* d_klist_c = reinterpret_cast<const int*>(static_cast<const unsigned char*>(ctx->kpts.p) + (size_t)nk * 16);
  const int* d_klist_r = d_klist_c + klist_c.size();
  if (kmult) g.kmult = reinterpret_cast<const int*>(static_cast<const unsigned char*>(ctx->kpts.p) + (size_t)nk * 20);
  const size_t diff_b = (size_t)nmasks * (grid->npts + 1) * sizeof(int);
  const size_t trans_b = (size_t)nmasks * grid->npts * sizeof(unsigned long long);
  if (ctx->diff.grow(diff_b) || ctx->trans.grow(trans_b)) return fail(HX_E_CUDA, "alloc accumulators");
  HX_CUDA(cudaMemsetAsync(ctx->diff.p, 0, diff_b, st));
  HX_CUDA(cudaMemsetAsync(ctx->trans.p, 0, trans_b, st));
  int* diff = static_cast<int*>(ctx->diff.p);
  auto* trans = static_cast<unsigned long long*>(ctx->trans.p);
  const double2* kp = static_cast<const double2*>(ctx->kpts.p);
  const int64_t nmat = nmasks * (int64_t)nk;

  int* status = reinterpret_cast<int*>(d_status);
  // refinement list of the two-pass eigenvalue stage (count word first, then the items)
  hx::RefineItem* refine = nullptr;
  unsigned long long* refine_count = nullptr;
  auto make_refine = [&](int64_t items) -> int {
    if (d_eigs) return 0;  // eigenvalue output requested: single full-precision pass
    // + 64 per matrix: the grouped list of the staged multisection pads every matrix's range (hx_kernels.cu)
    if (ctx->refine.grow(256 + (size_t)(items + 64 * nmat) * sizeof(hx::RefineItem))) return -1;
    refine_count = static_cast<unsigned long long*>(ctx->refine.p);
    refine = reinterpret_cast<hx::RefineItem*>(static_cast<unsigned char*>(ctx->refine.p) + 256);
    return 0;
  };
  const bool use_bd = c.bipartite && ctx->use_bipartite && hx::bd_path_supported(c) && N > ctx->bd_min_n;
  if (c.pencil != HX_PENCIL_GENERAL && N <= HX_SMEM_MAX_N && !use_bd) {
    // shared-memory tier: tridiagonalise every (mask, k) matrix, then one thread per eigenvalue
    const size_t smem = hx::small_tridiag_smem(N);
    int64_t chunk = std::min<int64_t>(nmat, std::max<int64_t>(1, (int64_t)((size_t)1 << 30) / (16 * N + 4)));
    chunk = std::max<int64_t>(nk, chunk - chunk % nk);  // whole masks per chunk
    if (ctx->tri.grow((size_t)chunk * (2 * N * 8 + 4) + 256)) return fail(HX_E_CUDA, "alloc tridiagonal buffers");
    double* tri = static_cast<double*>(ctx->tri.p);
    int* dims = reinterpret_cast<int*>(tri + (size_t)chunk * 2 * N);
    if (make_refine(chunk * N)) return fail(HX_E_CUDA, "alloc refinement list");
    for (int64_t m0 = 0; m0 < nmat; m0 += chunk) {
      const int64_t cnt = std::min(chunk, nmat - m0);
      // masks/kpts offsets: the kernel indexes matrices from blockIdx.x; shift the mask base by whole masks
      if (m0 % nk) return fail(HX_E_ARG, "internal: chunk not aligned to k-point groups");
      const uint64_t* mk0 = d_masks + (m0 / nk) * c.words;
      const bool tgk = c.bipartite && ctx->use_bipartite && hx::small_bidiag_smem(N, c.nsub) <= 200 * 1024;
      // Gram path of the S in (32, 64] tiers (hx_smallgram.cuh; HX_SMALL_GRAM=0: Golub-Kahan): IDOS only, graphene
      // pencil, zone path of the eigenvalue stage applicable and every transition zone clear of lambda = 0
      hx::CellDev cs = c;
      cs.N = c.nsub;
      const bool small_gram = tgk && !d_eigs && refine && refine_count && c.pencil == 1 && c.nsub > 32 &&
                              c.nsub <= 64 && c.nsub > ctx->bidiag_warp_max_s && ctx->bidiag_reg &&
                              hx::opt("HX_SMALL_GRAM", 1) != 0 && N >= hx::opt("HX_ZONE_MIN_N", 96) &&
                              hx::gram_zones_ok(cs, g, sharp, 1e-3);
      if (small_gram) {
        const int nkc = (int)klist_c.size(), nkr = (int)klist_r.size();
        const int64_t nm = cnt / nk;
        const size_t sm_c = hx::small_gram_reg_smem(N, c.nsub, false), sm_r = hx::small_gram_reg_smem(N, c.nsub, true);
        if (nkr == 0) {
          hx::small_gram_reg_kernel<<<(unsigned)cnt, hx::BIDIAG_REG_THREADS, sm_c, st>>>(c, kp, nk, mk0, tri, dims,
                                                                                        status + m0, nullptr, nk);
        } else {
          if (nkc > 0) {
            hx::small_gram_reg_kernel<<<(unsigned)(nm * nkc), hx::BIDIAG_REG_THREADS, sm_c, st>>>(
                c, kp, nk, mk0, tri, dims, status + m0, d_klist_c, nkc);
            hx::count_launch();
          }
          hx::small_gram_reg_real_kernel<<<(unsigned)(nm * nkr), hx::BIDIAG_REG_THREADS, sm_r, st>>>(
              c, kp, nk, mk0, tri, dims, status + m0, d_klist_r, nkr);
        }
        HX_CUDA(cudaGetLastError());
        hx::count_launch();
        if (!hx::launch_gram_idos(cs, nk, g, m0, cnt, tri, (size_t)2 * N, dims, diff, trans, status, sharp, st, refine,
                                  refine_count))
          return fail(HX_E_CUDA, "internal: Gram eigenvalue stage refused a batch gram_zones_ok accepted");
        HX_CUDA(cudaGetLastError());
        continue;
      }
      if (tgk) {
        // one warp per matrix up to S = 32 (latency of the serial reflector chain is hidden by many
        // matrices per SM), a CTA beyond
        const int nkc = (int)klist_c.size(), nkr = (int)klist_r.size();
        const int64_t nm = cnt / nk;  // whole masks in this chunk
        // complex k-points: one warp per matrix up to S = 32, the register-resident 256-thread reduction up
        // to S = 64 (HX_BIDIAG_REG=0: the shared-memory CTA), the shared-memory CTA beyond
        auto launch_complex = [&](unsigned grid, const int* kl, int nks) {
          if (c.nsub > ctx->bidiag_warp_max_s && c.nsub <= 64 && ctx->bidiag_reg)
            hx::small_bidiag_reg_kernel<<<grid, hx::BIDIAG_REG_THREADS, hx::small_bidiag_reg_smem(N, c.nsub), st>>>(
                c, kp, nk, mk0, tri, dims, status + m0, kl, nks);
          else
            hx::small_bidiag_kernel<<<grid, c.nsub <= ctx->bidiag_warp_max_s ? 32 : ctx->bidiag_threads,
                                      hx::small_bidiag_smem(N, c.nsub), st>>>(c, kp, nk, mk0, tri, dims, status + m0,
                                                                              kl, nks, 0);
        };
        if (nkr == 0) {
          launch_complex((unsigned)cnt, nullptr, nk);
        } else {
          if (nkc > 0) launch_complex((unsigned)(nm * nkc), d_klist_c, nkc);
          // real k-points: one warp per matrix up to S = 32 (two columns / rows per lane), the
          // register-resident 256-thread reduction up to S = 64 (HX_BIDIAG_REG=0: warps up to
          // HX_BIDIAG_REAL_WARP_MAX_S)
          if (c.nsub > 32 && c.nsub <= 64 && ctx->bidiag_reg) {
            hx::small_bidiag_reg_real_kernel<<<(unsigned)(nm * nkr), hx::BIDIAG_REG_THREADS,
                                               hx::small_bidiag_reg_real_smem(N, c.nsub), st>>>(
                c, kp, nk, mk0, tri, dims, status + m0, d_klist_r, nkr);
          } else {
            const bool rw = c.nsub <= ctx->bidiag_real_warp_max_s;
            hx::small_bidiag_kernel<<<(unsigned)(nm * nkr), rw ? 32 : ctx->bidiag_threads,
                                      hx::small_bidiag_smem_real(N, c.nsub, rw), st>>>(c, kp, nk, mk0, tri, dims,
                                                                                       status + m0, d_klist_r, nkr, 1);
          }
          hx::count_launch();
        }
      } else {
        hx::small_tridiag_kernel<<<(unsigned)cnt, N > 64 ? 512 : 256, smem, st>>>(c, kp, nk, mk0, tri, dims,
                                                                                 status + m0);
      }
      HX_CUDA(cudaGetLastError());
      hx::count_launch();
      hx::launch_eig_idos(c, nk, g, m0, cnt, tri, (size_t)2 * N, dims, diff, trans, d_eigs, status, sharp, st, refine,
                          refine_count, tgk);
      HX_CUDA(cudaGetLastError());
    }
  } else if (use_bd) {
    if (make_refine(nmat * N)) return fail(HX_E_CUDA, "alloc refinement list");
    const bool real = real_batches() && batch_is_real(cell, kpoints, nk);
    int rc = hx::bd_eval(c, kp, nk, d_masks, nmasks, g, diff, trans, d_eigs, status, sharp, real, ctx->ws_budget,
                         [&](size_t bytes) -> void* { return ctx->band.grow(bytes) ? nullptr : ctx->band.p; }, st,
                         refine, refine_count);
    if (rc) return fail(HX_E_CUDA, std::string("bipartite band path: ") + hx::bd_last_error());
  } else if (hx::band_path_supported(N) && (c.pencil != HX_PENCIL_GENERAL || general_band())) {
    if (make_refine(nmat * N)) return fail(HX_E_CUDA, "alloc refinement list");
    int rc = hx::band_eval(c, kp, nk, d_masks, nmasks, g, diff, trans, d_eigs,
                           reinterpret_cast<int*>(d_status), sharp, ctx->ws_budget,
                           [&](size_t bytes) -> void* { return ctx->band.grow(bytes) ? nullptr : ctx->band.p; }, st,
                           refine, refine_count);
    if (rc) return fail(HX_E_CUDA, std::string("band path: ") + hx::band_last_error());
  } else {
    const size_t stride = hx::global_ws_stride(N, c.pencil == HX_PENCIL_GENERAL);
    int64_t chunk = (int64_t)std::max<size_t>(1, ctx->ws_budget / stride);
    chunk = std::min<int64_t>(chunk, nmat);
    chunk = std::min<int64_t>(chunk, 65535);
    if (ctx->ws.grow(stride * (size_t)chunk)) return fail(HX_E_CUDA, "alloc workspace");
    if (ctx->tri.grow((size_t)chunk * (2 * N * 8 + 4) + 256)) return fail(HX_E_CUDA, "alloc tridiagonal buffers");
    double* tri = static_cast<double*>(ctx->tri.p);
    int* dims = reinterpret_cast<int*>(tri + (size_t)chunk * 2 * N);
    if (make_refine(chunk * N)) return fail(HX_E_CUDA, "alloc refinement list");
    for (int64_t m0 = 0; m0 < nmat; m0 += chunk) {
      const int64_t cnt = std::min(chunk, nmat - m0);
      hx::global_tridiag_kernel<<<(unsigned)cnt, 512, 0, st>>>(c, kp, nk, d_masks, m0,
                                                               static_cast<unsigned char*>(ctx->ws.p), stride, tri,
                                                               dims, status);
      HX_CUDA(cudaGetLastError());
      hx::count_launch();
      hx::launch_eig_idos(c, nk, g, m0, cnt, tri, (size_t)2 * N, dims, diff, trans, d_eigs, status, sharp, st, refine,
                          refine_count);
      HX_CUDA(cudaGetLastError());
    }
  }
  const int wpb = 8;
  hx::finalize_kernel<<<(unsigned)((nmasks + wpb - 1) / wpb), 32 * wpb, 0, st>>>(diff, trans, nmasks, g,
                                                                                 1.0 / (double)nk_total,
                                                                                 1.0 / c.area, d_curves);
  HX_CUDA(cudaGetLastError());
    hx::count_launch();
  return 0;
}

int hx_eval_idos_batch_device(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk, const uint64_t* d_masks,
                              int64_t nmasks, const hx_egrid* grid, double* d_curves, double* d_eigs,
                              int32_t* d_status, void* stream) {
  return eval_impl(ctx, cell, kpoints, nk, d_masks, nmasks, grid, d_curves, d_eigs, d_status,
                   static_cast<cudaStream_t>(stream), 0);
}

int hx_eval_idos_batch_device_k(hx_ctx* ctx, hx_cell* cell, const double* kpoints, const int32_t* kmult, int32_t nk,
                                const uint64_t* d_masks, int64_t nmasks, const hx_egrid* grid, double* d_curves,
                                int32_t* d_status, void* stream) {
  return eval_impl(ctx, cell, kpoints, nk, d_masks, nmasks, grid, d_curves, nullptr, d_status,
                   static_cast<cudaStream_t>(stream), 0, kmult);
}

static int eval_host(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk, const uint64_t* masks,
                     int64_t nmasks, const hx_egrid* grid, double* out_curves, double* out_eigs, int32_t* out_status,
                     int sharp, const int32_t* kmult = nullptr) {
  if (!ctx || !cell || !grid) return fail(HX_E_ARG, "hx_eval_idos_batch: null argument");
  if (nmasks == 0) return 0;
  if (!masks || !out_curves || !out_status) return fail(HX_E_ARG, "hx_eval_idos_batch: null buffer");
  if (set_device(ctx)) return HX_E_CUDA;
  const hx::CellDev& c = cell->dev;
  const size_t mb = (size_t)nmasks * c.words * 8, cb = (size_t)nmasks * grid->npts * 8,
               sb = (size_t)nmasks * nk * 4, eb = (size_t)nmasks * nk * c.N * 8;
  if (ctx->masks.grow(mb) || ctx->curves.grow(cb) || ctx->status.grow(sb) || (out_eigs && ctx->eigs.grow(eb)))
    return fail(HX_E_CUDA, "alloc batch buffers");
  cudaStream_t st = ctx->stream;
  // pinned staging (ctx->h_io) for batches up to 256 MB of traffic: masks in, then curves | status | eigs
  // out in the same buffer (true async DMA: concurrent small tiers are not held back by pageable staging);
  // larger batches are bandwidth-bound and copy straight between pageable memory and the device (staging
  // them would add a host memcpy of the whole result)
  const size_t out_b = cb + sb + (out_eigs ? eb : 0);
  const bool staged = std::max(mb, out_b) <= ((size_t)256 << 20);
  unsigned char* hio = nullptr;
  if (staged) {
    if (ctx->h_io.grow(std::max(mb, out_b))) return fail(HX_E_CUDA, "alloc pinned staging");
    hio = static_cast<unsigned char*>(ctx->h_io.p);
    std::memcpy(hio, masks, mb);
    HX_CUDA(cudaMemcpyAsync(ctx->masks.p, hio, mb, cudaMemcpyHostToDevice, st));
  } else {
    HX_CUDA(cudaMemcpyAsync(ctx->masks.p, masks, mb, cudaMemcpyHostToDevice, st));
  }
  int rc = eval_impl(ctx, cell, kpoints, nk, static_cast<uint64_t*>(ctx->masks.p), nmasks, grid,
                     static_cast<double*>(ctx->curves.p), out_eigs ? static_cast<double*>(ctx->eigs.p) : nullptr,
                     static_cast<int32_t*>(ctx->status.p), st, sharp, kmult);
  if (rc) {
    cudaStreamSynchronize(st);
    return rc;
  }
  if (!staged) {
    HX_CUDA(cudaMemcpyAsync(out_curves, ctx->curves.p, cb, cudaMemcpyDeviceToHost, st));
    HX_CUDA(cudaMemcpyAsync(out_status, ctx->status.p, sb, cudaMemcpyDeviceToHost, st));
    if (out_eigs) HX_CUDA(cudaMemcpyAsync(out_eigs, ctx->eigs.p, eb, cudaMemcpyDeviceToHost, st));
    HX_CUDA(cudaStreamSynchronize(st));
    return 0;
  }
  HX_CUDA(cudaMemcpyAsync(hio, ctx->curves.p, cb, cudaMemcpyDeviceToHost, st));
  HX_CUDA(cudaMemcpyAsync(hio + cb, ctx->status.p, sb, cudaMemcpyDeviceToHost, st));
  if (out_eigs) HX_CUDA(cudaMemcpyAsync(hio + cb + sb, ctx->eigs.p, eb, cudaMemcpyDeviceToHost, st));
  HX_CUDA(cudaEventRecord(ctx->h_io.ev, st));
  HX_CUDA(cudaStreamSynchronize(st));
  std::memcpy(out_curves, hio, cb);
  std::memcpy(out_status, hio + cb, sb);
  if (out_eigs) std::memcpy(out_eigs, hio + cb + sb, eb);
  return 0;
}

int hx_assemble_device(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk, const uint64_t* d_masks,
                       int64_t nmasks, double* d_H, double* d_S, int32_t* d_dims, void* stream) {
  if (!ctx || !cell || !kpoints || !d_masks || !d_H || !d_dims || nk < 1 || nmasks < 0)
    return fail(HX_E_ARG, "hx_assemble_device: bad args");
  if (nmasks == 0) return 0;
  if (set_device(ctx)) return HX_E_CUDA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ctx->kpts.grow((size_t)nk * 16)) return fail(HX_E_CUDA, "alloc kpts");
  HX_CUDA(cudaMemcpyAsync(ctx->kpts.p, kpoints, (size_t)nk * 16, cudaMemcpyHostToDevice, st));
  const size_t smem = (size_t)cell->dev.N * sizeof(int);
  if (smem > 200 * 1024) return fail(HX_E_RANGE, "hx_assemble_device: N too large");
  hx::set_smem_attr(hx::assemble_kernel, 200 * 1024);
  hx::assemble_kernel<<<(unsigned)(nmasks * nk), 256, smem, st>>>(
      cell->dev, static_cast<const double2*>(ctx->kpts.p), nk, d_masks, reinterpret_cast<double2*>(d_H),
      reinterpret_cast<double2*>(d_S), reinterpret_cast<int*>(d_dims));
  HX_CUDA(cudaGetLastError());
    hx::count_launch();
  return 0;
}

int hx_eval_idos_batch(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk, const uint64_t* masks,
                       int64_t nmasks, const hx_egrid* grid, double* out_curves, double* out_eigs,
                       int32_t* out_status) {
  return eval_host(ctx, cell, kpoints, nk, masks, nmasks, grid, out_curves, out_eigs, out_status, 0);
}

int hx_eval_idos_batch_k(hx_ctx* ctx, hx_cell* cell, const double* kpoints, const int32_t* kmult, int32_t nk,
                         const uint64_t* masks, int64_t nmasks, const hx_egrid* grid, double* out_curves,
                         int32_t* out_status) {
  return eval_host(ctx, cell, kpoints, nk, masks, nmasks, grid, out_curves, nullptr, out_status, 0, kmult);
}

// Sharp-count variant of the batch (idos_sharp, qoi.py:105-108); not part of the public header's
// hot path but exported for parity tests.
int hx_eval_sharp_batch(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk, const uint64_t* masks,
                        int64_t nmasks, const hx_egrid* grid, double* out_curves, double* out_eigs,
                        int32_t* out_status) {
  return eval_host(ctx, cell, kpoints, nk, masks, nmasks, grid, out_curves, out_eigs, out_status, 1);
}

// Standalone batched eigenvalues of caller-provided matrices (config-5 sweep).
int hx_eigvalsh_batch_device(hx_ctx* ctx, int32_t n, int64_t batch, const double* d_A, const double* d_B,
                             double* d_eigs, int32_t* d_status, void* stream) {
  if (!ctx || !d_A || !d_eigs || !d_status || n < 1 || batch < 0) return fail(HX_E_ARG, "hx_eigvalsh_batch: bad args");
  if (batch == 0) return 0;
  if (n > HX_MAX_N) return fail(HX_E_RANGE, "hx_eigvalsh_batch: n too large");
  if (set_device(ctx)) return HX_E_CUDA;
  refresh_opts(ctx);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* status = reinterpret_cast<int*>(d_status);
  hx::CellDev c{};
  c.N = n;
  hx::GridDev g{};
  if (hx::band_path_supported(n) && (!d_B || general_band())) {
    int rc = hx::band_eigvalsh(n, batch, reinterpret_cast<const double2*>(d_A),
                               reinterpret_cast<const double2*>(d_B), d_eigs, status, ctx->ws_budget,
                               [&](size_t bytes) -> void* { return ctx->band.grow(bytes) ? nullptr : ctx->band.p; }, st);
    if (rc) return fail(HX_E_CUDA, std::string("band path: ") + hx::band_last_error());
    return 0;
  }
  const bool small = !d_B && n <= HX_SMEM_MAX_N;
  const size_t stride = small ? 0 : hx::global_ws_stride(n, d_B != nullptr);
  int64_t chunk = small ? std::min<int64_t>(batch, 1 << 20)
                        : std::min<int64_t>((int64_t)std::max<size_t>(1, ctx->ws_budget / stride), batch);
  chunk = std::min<int64_t>(chunk, small ? (1 << 20) : 65535);
  if (!small && ctx->ws.grow(stride * (size_t)chunk)) return fail(HX_E_CUDA, "alloc workspace");
  if (ctx->tri.grow((size_t)chunk * (2 * n * 8 + 4) + 256)) return fail(HX_E_CUDA, "alloc tridiagonal buffers");
  double* tri = static_cast<double*>(ctx->tri.p);
  int* dims = reinterpret_cast<int*>(tri + (size_t)chunk * 2 * n);
  for (int64_t m0 = 0; m0 < batch; m0 += chunk) {
    const int64_t cnt = std::min(chunk, batch - m0);
    if (small) {
      hx::eigvalsh_small_kernel<<<(unsigned)cnt, n > 64 ? 512 : 256, hx::small_tridiag_smem(n), st>>>(
          n, reinterpret_cast<const double2*>(d_A) + (size_t)m0 * n * n, tri, dims, status + m0);
    } else {
      hx::eigvalsh_global_kernel<<<(unsigned)cnt, 512, 0, st>>>(n, reinterpret_cast<const double2*>(d_A),
                                                                reinterpret_cast<const double2*>(d_B), m0,
                                                                static_cast<unsigned char*>(ctx->ws.p), stride, tri,
                                                                dims, status);
    }
    HX_CUDA(cudaGetLastError());
    hx::count_launch();
    hx::launch_eig_idos(c, 1, g, m0, cnt, tri, (size_t)2 * n, dims, nullptr, nullptr, d_eigs, status, 0, st);
    HX_CUDA(cudaGetLastError());
  }
  return 0;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// Kernel-module parity (_kernels.py:68-101): one CTA, thread per grid point, states in input order.
namespace hx {
__global__ void counts_kernel(const double* E, const double* w, int64_t count, GridDev g, double* out, int sharp) {
  for (int m = threadIdx.x; m < g.npts; m += blockDim.x) {
    double full = 0.0, tr = 0.0;
    const double em = __dadd_rn(g.e0, __dmul_rn(g.step, (double)m));
    for (int64_t i = 0; i < count; ++i) {
      const double e = E[i];
      if (sharp) {
        long long idx = (long long)floor(__ddiv_rn(__dsub_rn(e, g.e0), g.step)) + 1;
        if (idx < 0) idx = 0;
        if (idx <= m) full = __dadd_rn(full, w[i]);
        continue;
      }
      long long lo = (long long)ceil(__ddiv_rn(__dsub_rn(__dadd_rn(e, g.delta), g.e0), g.step));
      if (lo < 0) lo = 0;
      if (lo <= m) {
        full = __dadd_rn(full, w[i]);
        continue;
      }
      long long m0 = (long long)floor(__ddiv_rn(__dsub_rn(__dsub_rn(e, g.delta), g.e0), g.step)) + 1;
      if (m0 < 0) m0 = 0;
      if (m >= m0) {
        const double x = __ddiv_rn(__dsub_rn(e, em), g.delta);
        const double gx = __dadd_rn(0.5, __dmul_rn(x, __dadd_rn(-1.125, __dmul_rn(__dmul_rn(0.625, x), x))));
        tr = __dadd_rn(tr, __dmul_rn(w[i], gx));
      }
    }
    out[m] = __dadd_rn(out[m], __dadd_rn(tr, full));
  }
}

// CV terms and level moments per grid point (runner.py:281-299, mlmc.py:143-154).  Block = 32 grid points x
// 8 sample groups (sample i in group i % 8).  Mean and variance come from exact fixed-point sums (hx_fixed.cuh):
// sum_i term_i, then sum_i (term_i - mean)^2 (two passes, the np.var form), each an integer sum of per-term
// fixed-point values, so the results do not depend on scheduling, on the batch split or on the number of
// devices the samples were spread over (hx_level_sums_fixed_device + an int64 all-reduce gives the same bits).
constexpr int MOM_P = 32, MOM_G = 8;
__host__ __device__ __forceinline__ double cv_term(const double* full, const double* quarters, int64_t i, int npts,
                                                   int m) {
  double t = full[i * npts + m];
  if (quarters) {
    // cv = ((q1 + q2) + q3 + q4) * 0.25, term = full - cv: the reference's order (runner.py:289-297)
    const double* q = quarters + i * 4 * npts + m;
#ifdef __CUDA_ARCH__
    double cv = __dadd_rn(__dadd_rn(__dadd_rn(q[0], q[npts]), q[2 * npts]), q[3 * npts]);
    t = __dsub_rn(t, __dmul_rn(cv, 0.25));
#else
    volatile double cv = ((q[0] + q[npts]) + q[2 * npts]) + q[3 * npts];
    volatile double c4 = cv * 0.25;
    t = t - c4;
#endif
  }
  return t;
}

__host__ __device__ __forceinline__ double fx_sq_dev(double t, double mu) {
#ifdef __CUDA_ARCH__
  const double d = __dsub_rn(t, mu);
  return __dmul_rn(d, d);
#else
  volatile double d = t - mu;
  volatile double d2 = d * d;
  return d2;
#endif
}

__device__ __forceinline__ double fx_nan() { return __longlong_as_double(0x7ff8000000000000ll); }

// Block-wide exact sum of the per-thread limbs of grid point `pl`: group 0's threads get the total.
__device__ __forceinline__ void fx_block_sum(int64_t (*sh)[FX_NL][MOM_P], const int64_t* L, int grp, int pl,
                                             int64_t* out) {
#pragma unroll
  for (int j = 0; j < FX_NL; ++j) sh[grp][j][pl] = L[j];
  __syncthreads();
  if (grp == 0) {
#pragma unroll
    for (int j = 0; j < FX_NL; ++j) {
      int64_t a = 0;
      for (int q = 0; q < MOM_G; ++q) a += sh[q][j][pl];
      out[j] = a;
    }
  }
  __syncthreads();
}

// Exact level sums: block = 32 grid points x 8 row groups over one chunk of rows (blockIdx.y); the per-thread
// limbs are combined in shared memory and added to the global accumulator with 64-bit integer atomics - integer
// addition is associative, so the sums do not depend on the chunking or the order the blocks run in.
//   center == NULL : acc += limbs of term_i (terms written when `terms` != NULL)
//   center != NULL : acc += limbs of (term_i - center)^2
constexpr int MOM_ROWS = 64;  // rows per block (8 per thread)
__global__ void __launch_bounds__(MOM_P * MOM_G) level_sums_kernel(const double* full, const double* quarters, int64_t M,
                                                                   int npts, double* terms, const double* center,
                                                                   unsigned long long* acc, int* bad) {
  __shared__ int64_t sh[MOM_G][FX_NL][MOM_P];
  const int pl = threadIdx.x % MOM_P, grp = threadIdx.x / MOM_P;
  const int m = blockIdx.x * MOM_P + pl;
  const bool on = m < npts;
  const int64_t r0 = (int64_t)blockIdx.y * MOM_ROWS, r1 = M < r0 + MOM_ROWS ? M : r0 + MOM_ROWS;
  int64_t L[FX_NL];
#pragma unroll
  for (int j = 0; j < FX_NL; ++j) L[j] = 0;
  bool ok = true;
  if (on) {
    const double mu = center ? center[m] : 0.0;
    for (int64_t i = r0 + grp; i < r1; i += MOM_G) {
      const double t = cv_term(full, quarters, i, npts, m);
      if (terms) terms[i * npts + m] = t;
      ok &= fx_add(L, center ? fx_sq_dev(t, mu) : t);
    }
  }
#pragma unroll
  for (int j = 0; j < FX_NL; ++j) sh[grp][j][pl] = L[j];
  __syncthreads();
  if (grp == 0 && on) {
#pragma unroll
    for (int j = 0; j < FX_NL; ++j) {
      int64_t a = 0;
      for (int q = 0; q < MOM_G; ++q) a += sh[q][j][pl];
      if (a) atomicAdd(acc + (int64_t)m * FX_NL + j, (unsigned long long)a);
    }
  }
  if (!ok && bad) atomicOr(bad + (on ? m : 0), 1);
}

__global__ void fixed_finalize_kernel(const int64_t* limbs, int npts, double divisor, double* out, const int* bad) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= npts) return;
  out[m] = (divisor > 0.0 && !(bad && bad[m])) ? fx_to_double(limbs + (int64_t)m * FX_NL) / divisor : fx_nan();
}

__global__ void sample_masks_kernel(uint64_t seed, uint64_t level, uint64_t rep0, int64_t count, double p, int nunits,
                                    uint64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int words = (nunits + 63) / 64 > 0 ? (nunits + 63) / 64 : 1;
  uint64_t s4[4];
  seedseq_state4(seed, level, rep0 + (uint64_t)i, s4);
  Pcg64 g;
  g.seed(s4);
  uint64_t* o = out + i * words;
  uint64_t wacc = 0;
  int w = 0;
  for (int u = 0; u < nunits; ++u) {
    if (g.next_double() < p) wacc |= 1ull << (u & 63);
    if ((u & 63) == 63) {
      o[w++] = wacc;
      wacc = 0;
    }
  }
  if (nunits & 63) o[w++] = wacc;
  for (; w < words; ++w) o[w] = 0;
}
// One thread per (parent mask, unit): scatter vacant units into their quarter's sub-mask.
__global__ void restrict_masks_kernel(const uint64_t* parent, int64_t nmasks, int parent_units, const int* assign,
                                      const int* umap, int sub_units, unsigned long long* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nmasks * parent_units) return;
  const int64_t i = t / parent_units;
  const int u = (int)(t - i * parent_units);
  const int pw = (parent_units + 63) / 64 > 0 ? (parent_units + 63) / 64 : 1;
  const int sw = (sub_units + 63) / 64 > 0 ? (sub_units + 63) / 64 : 1;
  if (!((parent[i * pw + (u >> 6)] >> (u & 63)) & 1ull)) return;
  const int r = assign[u], su = umap[u];
  atomicOr(out + i * 4 * sw + (r - 1) * sw + (su >> 6), 1ull << (su & 63));
}
}  // namespace hx

extern "C" {

int hx_restrict_masks_device(const uint64_t* d_parent_words, int64_t nmasks, int32_t parent_units,
                             const int32_t* d_unit_assign, const int32_t* d_unit_map, int32_t sub_units,
                             uint64_t* d_out_words, void* stream) {
  if (!d_parent_words || !d_unit_assign || !d_unit_map || !d_out_words || nmasks < 0)
    return fail(HX_E_ARG, "restrict_device: bad args");
  if (nmasks == 0 || parent_units == 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int sw = std::max(1, (sub_units + 63) / 64);
  HX_CUDA(cudaMemsetAsync(d_out_words, 0, (size_t)nmasks * 4 * sw * 8, st));
  const int64_t total = nmasks * parent_units;
  hx::restrict_masks_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      d_parent_words, nmasks, parent_units, d_unit_assign, d_unit_map, sub_units,
      reinterpret_cast<unsigned long long*>(d_out_words));
  HX_CUDA(cudaGetLastError());
    hx::count_launch();
  return 0;
}

int hx_smoothed_counts_device(const double* d_energies, const double* d_weights, int64_t count, const hx_egrid* grid,
                              double* d_out, void* stream) {
  if (!grid || !d_out || (count > 0 && (!d_energies || !d_weights))) return fail(HX_E_ARG, "smoothed_counts: bad args");
  hx::GridDev g{grid->e0, grid->step, grid->delta, grid->npts, 0};
  hx::counts_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_energies, d_weights, count, g, d_out, 0);
  HX_CUDA(cudaGetLastError());
    hx::count_launch();
  return 0;
}

int hx_sharp_counts_device(const double* d_energies, const double* d_weights, int64_t count, const hx_egrid* grid,
                           double* d_out, void* stream) {
  if (!grid || !d_out || (count > 0 && (!d_energies || !d_weights))) return fail(HX_E_ARG, "sharp_counts: bad args");
  hx::GridDev g{grid->e0, grid->step, grid->delta, grid->npts, 0};
  hx::counts_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_energies, d_weights, count, g, d_out, 1);
  HX_CUDA(cudaGetLastError());
    hx::count_launch();
  return 0;
}

// The stream-ordered scratch of hx_level_moments_device comes from the device's default memory pool; by
// default that pool returns freed memory to the driver at every synchronisation, which makes the next
// cudaMallocAsync a fresh mapping (milliseconds).  Keep the pool's memory instead (once per device).
static void keep_pool_memory() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

// scratch for hx_level_moments_device: 2 x npts x limbs accumulators + npts bad flags (stream-ordered)
int hx_level_moments_device(const double* d_full, const double* d_quarters, int64_t M, int32_t npts, double* d_terms,
                            double* d_mean, double* d_var, void* stream) {
  if (!d_full || M < 1 || npts < 1) return fail(HX_E_ARG, "level_moments: bad args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t lb = (size_t)npts * HX_FX_LIMBS * 8;
  keep_pool_memory();
  unsigned char* scratch = nullptr;
  HX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), 2 * lb + (size_t)npts * (4 + 8) + 64, st));
  auto* s1 = reinterpret_cast<unsigned long long*>(scratch);
  auto* s2 = reinterpret_cast<unsigned long long*>(scratch + lb);
  int* bad = reinterpret_cast<int*>(scratch + 2 * lb);
  double* mean = d_mean ? d_mean : reinterpret_cast<double*>(scratch + 2 * lb + (((size_t)npts * 4 + 15) & ~(size_t)15));
  HX_CUDA(cudaMemsetAsync(scratch, 0, 2 * lb + (size_t)npts * 4, st));
  const dim3 grid((unsigned)((npts + hx::MOM_P - 1) / hx::MOM_P), (unsigned)((M + hx::MOM_ROWS - 1) / hx::MOM_ROWS));
  hx::level_sums_kernel<<<grid, hx::MOM_P * hx::MOM_G, 0, st>>>(d_full, d_quarters, M, npts, d_terms, nullptr, s1, bad);
  hx::fixed_finalize_kernel<<<(npts + 127) / 128, 128, 0, st>>>(reinterpret_cast<int64_t*>(s1), npts, (double)M, mean,
                                                                bad);
  if (d_var) {
    hx::level_sums_kernel<<<grid, hx::MOM_P * hx::MOM_G, 0, st>>>(d_full, d_quarters, M, npts, nullptr, mean, s2, bad);
    hx::fixed_finalize_kernel<<<(npts + 127) / 128, 128, 0, st>>>(reinterpret_cast<int64_t*>(s2), npts,
                                                                  (double)(M - 1), d_var, bad);
  }
  HX_CUDA(cudaGetLastError());
  hx::count_launch(d_var ? 4 : 2);
  HX_CUDA(cudaFreeAsync(scratch, st));
  return 0;
}

int hx_level_sums_fixed_device(const double* d_full, const double* d_quarters, int64_t M, int32_t npts,
                               const double* d_center, int64_t* d_limbs, void* stream) {
  if (!d_full || M < 0 || npts < 1 || !d_limbs) return fail(HX_E_ARG, "level_sums_fixed_device: bad args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HX_CUDA(cudaMemsetAsync(d_limbs, 0, (size_t)npts * HX_FX_LIMBS * 8, st));
  if (M == 0) return 0;
  const dim3 grid((unsigned)((npts + hx::MOM_P - 1) / hx::MOM_P), (unsigned)((M + hx::MOM_ROWS - 1) / hx::MOM_ROWS));
  hx::level_sums_kernel<<<grid, hx::MOM_P * hx::MOM_G, 0, st>>>(d_full, d_quarters, M, npts, nullptr, d_center,
                                                                  reinterpret_cast<unsigned long long*>(d_limbs),
                                                                  nullptr);
  HX_CUDA(cudaGetLastError());
  hx::count_launch();
  return 0;
}

int hx_fixed_finalize_device(const int64_t* d_limbs, int32_t npts, double divisor, double* d_out, void* stream) {
  if (!d_limbs || !d_out || npts < 1) return fail(HX_E_ARG, "fixed_finalize_device: bad args");
  hx::fixed_finalize_kernel<<<(npts + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(d_limbs, npts, divisor,
                                                                                            d_out, nullptr);
  HX_CUDA(cudaGetLastError());
  hx::count_launch();
  return 0;
}

int hx_level_sums_fixed(const double* full, const double* quarters, int64_t M, int32_t npts, const double* center,
                        int64_t* limbs) {
  if (!full || M < 0 || npts < 1 || !limbs) return fail(HX_E_ARG, "level_sums_fixed: bad args");
  for (int m = 0; m < npts; ++m) {
    int64_t* L = limbs + (int64_t)m * HX_FX_LIMBS;
    for (int j = 0; j < HX_FX_LIMBS; ++j) L[j] = 0;
    for (int64_t i = 0; i < M; ++i) {
      const double t = hx::cv_term(full, quarters, i, npts, m);
      if (!hx::fx_add(L, center ? hx::fx_sq_dev(t, center[m]) : t))
        return fail(HX_E_RANGE, "level_sums_fixed: non-finite or out-of-range term");
    }
  }
  return 0;
}

int hx_fixed_finalize(const int64_t* limbs, int32_t npts, double divisor, double* out) {
  if (!limbs || !out || npts < 0) return fail(HX_E_ARG, "fixed_finalize: bad args");
  for (int m = 0; m < npts; ++m)
    out[m] = divisor > 0.0 ? hx::fx_to_double(limbs + (int64_t)m * HX_FX_LIMBS) / divisor : NAN;
  return 0;
}

int hx_uniforms(uint64_t seed, uint64_t level, uint64_t rep, int64_t count, double* out) {
  if (!out || count < 0) return fail(HX_E_ARG, "hx_uniforms: bad args");
  if (level > 0xFFFFFFFFull || rep > 0xFFFFFFFFull) {
    // words32 handles wider keys too; keep the documented envelope
  }
  uint64_t s4[4];
  hx::seedseq_state4(seed, level, rep, s4);
  hx::Pcg64 g;
  g.seed(s4);
  for (int64_t i = 0; i < count; ++i) out[i] = g.next_double();
  return 0;
}

int hx_sample_masks(uint64_t seed, uint64_t level, uint64_t rep0, int64_t count, double p, int32_t nunits,
                    uint64_t* out_words, int32_t threads) {
  if (!out_words || count < 0 || nunits < 0 || !(p >= 0.0 && p <= 1.0)) return fail(HX_E_ARG, "sample_masks: bad args");
  const int words = std::max(1, (nunits + 63) / 64);
  auto work = [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      uint64_t s4[4];
      hx::seedseq_state4(seed, level, rep0 + (uint64_t)i, s4);
      hx::Pcg64 g;
      g.seed(s4);
      uint64_t* o = out_words + i * words;
      for (int w = 0; w < words; ++w) o[w] = 0;
      for (int u = 0; u < nunits; ++u)
        if (g.next_double() < p) o[u >> 6] |= 1ull << (u & 63);
    }
  };
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, count / 16));
  if (nt <= 1) {
    work(0, count);
    return 0;
  }
  std::vector<std::thread> pool;
  const int64_t per = (count + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t a = t * per, b = std::min(count, a + per);
    if (a < b) pool.emplace_back(work, a, b);
  }
  for (auto& th : pool) th.join();
  return 0;
}

int hx_sample_masks_device(uint64_t seed, uint64_t level, uint64_t rep0, int64_t count, double p, int32_t nunits,
                           uint64_t* d_out_words, void* stream) {
  if (!d_out_words || count < 0 || nunits < 0) return fail(HX_E_ARG, "sample_masks_device: bad args");
  if (count == 0) return 0;
  hx::sample_masks_kernel<<<(unsigned)((count + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, level, rep0, count, p, nunits, d_out_words);
  HX_CUDA(cudaGetLastError());
    hx::count_launch();
  return 0;
}

int hx_restrict_masks(const uint64_t* parent_words, int64_t nmasks, int32_t parent_units, const int32_t* unit_assign,
                      const int32_t* unit_map, int32_t sub_units, uint64_t* out_words) {
  if (!parent_words || !unit_assign || !unit_map || !out_words || nmasks < 0) return fail(HX_E_ARG, "restrict: bad args");
  const int pw = std::max(1, (parent_units + 63) / 64), sw = std::max(1, (sub_units + 63) / 64);
  for (int64_t i = 0; i < nmasks; ++i) {
    uint64_t* o = out_words + i * 4 * sw;
    for (int w = 0; w < 4 * sw; ++w) o[w] = 0;
    const uint64_t* pm = parent_words + i * pw;
    for (int u = 0; u < parent_units; ++u) {
      if (!((pm[u >> 6] >> (u & 63)) & 1ull)) continue;
      const int r = unit_assign[u];
      if (r < 1 || r > 4) return fail(HX_E_ARG, "restrict: quarter label out of range");
      const int su = unit_map[u];
      o[(r - 1) * sw + (su >> 6)] |= 1ull << (su & 63);
    }
  }
  return 0;
}

}  // extern "C"
