/* hx.h — C-ABI of libhx.so, the B200 (sm_100a) backend for the hexmc per-sample supercell solve.
 *
 * Drop-in boundary: the reference's batch job seam
 *     Engine.evaluate_masks -> parallel_map(_eval_job, jobs, workers)
 * (reference pkg/src/hexmc/runner.py:206-244, :75-93, :114-129) and its kernel module
 * (pkg/src/hexmc/_kernels.py:32-56).  Every entry point below names the reference function it
 * replaces.  Plain pointers and sizes only; no torch/numpy types.  All functions return 0 on
 * success and a negative HX_E* code on failure (text via hx_last_error()).  Per-matrix numerical
 * failures are reported in a caller-owned status array instead (HX_ST_*), which the Python layer
 * maps to the reference's SolverError / TaskError texts (spectrum.py:109-117, runner.py:56-93).
 *
 * Threading: one host thread per hx_ctx at a time.  Results are bitwise independent of batch
 * composition, device count and stream scheduling (fixed-point IDOS accumulation, no float
 * atomics).
 */
#ifndef HX_H_
#define HX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HX_ABI_VERSION 4

/* return codes */
#define HX_OK 0
#define HX_E_ARG -1     /* invalid argument */
#define HX_E_CUDA -2    /* CUDA runtime error */
#define HX_E_NODEV -3   /* no CUDA device / extension unusable */
#define HX_E_RANGE -4   /* size outside the supported envelope */

/* per-(mask, k) status codes written to out_status */
#define HX_ST_OK 0
#define HX_ST_NOT_PD 1    /* overlap S(k) not positive definite (Cholesky pivot <= 0) */
#define HX_ST_NONFINITE 2 /* non-finite value met in the reduction or bisection */
#define HX_ST_EMPTY 3     /* every orbital removed: zero curve (runner.py:122-125) */

/* pencil kinds */
#define HX_PENCIL_STANDARD 0  /* S = I: eigvalsh(H) == LAPACK zheevd (spectrum.py:103) */
#define HX_PENCIL_COMMUTING 1 /* H = eps0 I + t T, S = I + s T (graphene): eps = (eps0 + t l)/(1 + s l) */
#define HX_PENCIL_GENERAL 2   /* general H, S: S = L L^H, eig(L^-1 H L^-H) == zhegv (spectrum.py:106-108) */

typedef struct hx_ctx hx_ctx;
typedef struct hx_cell hx_cell;

/* Coupling instances of one model expanded on one nu x nu supercell, in the reference's
 * instance order (CompiledCell._expand, tbmodel.py:198-221), grouped by source dof (CSR).
 * Replaces CompiledCell + ConfiguredOperator inputs (tbmodel.py:162-253). */
typedef struct hx_cell_desc {
  int32_t ndof;            /* N = total orbitals of the supercell */
  int32_t nunits;          /* removable units (disorder bit positions) */
  const int32_t* unit_of_dof; /* [ndof] removable unit owning the dof, -1 if not removable */
  const double* onsite;    /* [ndof] on-site energies (diagonal of H; overwrites, tbmodel.py:260) */
  /* hopping instances, CSR by source dof: row_ptr[ndof+1], col/amp/disp[nnz] */
  const int32_t* h_row_ptr;
  const int32_t* h_col;
  const double* h_amp;     /* [2*nnz] complex amplitude (re, im) */
  const double* h_disp;    /* [2*nnz] true Cartesian displacement incl. basis offsets */
  /* overlap instances (HX_PENCIL_GENERAL only; NULL otherwise) */
  const int32_t* s_row_ptr;
  const int32_t* s_col;
  const double* s_amp;
  const double* s_disp;
  int32_t pencil;          /* HX_PENCIL_* */
  double eps0, t, s;       /* HX_PENCIL_COMMUTING parameters; h_amp then holds T's amplitudes */
  double area;             /* supercell area in per-unit-area units (lattice.py:131-133) */
  /* optional [ndof] sublattice (basis index) of each dof.  With HX_PENCIL_COMMUTING and hops that all
   * join sublattice 0 to 1 (graphene), T = [[0, C], [C^H, 0]] and the library may use the exact
   * bipartite identity eig(T) = +-sigma(C) (+ zeros).  NULL disables it. */
  const int32_t* sublattice;
  /* optional [2*ndof] Cartesian position of each dof's site in the supercell (the frame of h_disp).
   * With real amplitudes, batches whose k-points all make exp(2i k.R) = 1 for every hop's lattice
   * translation R = disp - (pos_dst - pos_src) (time-reversal-invariant momenta, e.g. Gamma and the q = 2
   * grid) are real in the periodic gauge exp(i k.R): the bipartite banded tier then runs its stage-1
   * products in real arithmetic (one DMMA per fragment product instead of four).  NULL disables it. */
  const double* dof_pos;
} hx_cell_desc;

/* Energy grid + smoothing (qoi.py:42-67, 77-82): eps_m = e0 + step*m, m < npts. */
typedef struct hx_egrid {
  double e0;
  double step;
  int32_t npts;
  double delta;
} hx_egrid;

/* ---- context / lifetime ---------------------------------------------------------------------- */
int hx_abi_version(void);
/* Cumulative number of libhx kernel launches in this process (instrumentation for bench.py). */
int hx_kernel_launches(uint64_t* out);
const char* hx_last_error(void);
/* Path-selection / tuning knobs (the HX_* names documented in DESIGN.md, e.g. HX_CHASE_RNW, HX_NO_REAL,
 * HX_REAL_STAGE1, HX_BIDIAG_REAL).  A value set here overrides the environment variable of the same
 * name; every batch call re-reads them, so tests force each kernel variant in-process.  No reference
 * counterpart (the reference selects its kernels once, by HEXMC_NO_NUMBA, _kernels.py:19-29).
 * hx_clear_option(NULL) clears every override. */
int hx_set_option(const char* name, int64_t value);
int hx_clear_option(const char* name);
int hx_get_option(const char* name, int64_t dflt, int64_t* out);
int hx_device_count(int32_t* out);
int hx_ctx_create(int32_t device, hx_ctx** out);
/* Same with the context's work stream at CUDA stream priority `priority` (lower = higher priority;
 * clamped to the device range).  Several contexts evaluate independent (n, q) groups concurrently:
 * the host mirror puts the largest tier of a batch on a high-priority context. */
int hx_ctx_create_priority(int32_t device, int32_t priority, hx_ctx** out);
int hx_ctx_destroy(hx_ctx* ctx);
int hx_ctx_synchronize(hx_ctx* ctx);

/* Upload one compiled cell (once per (model, nu)); replaces compile_cell (tbmodel.py:273-274). */
int hx_cell_create(hx_ctx* ctx, const hx_cell_desc* desc, hx_cell** out);
int hx_cell_destroy(hx_cell* cell);

/* Dense Bloch operators on the device (assemble_bloch, tbmodel.py:277-293 / ConfiguredOperator
 * .hamiltonian/.overlap, tbmodel.py:255-270): d_H, d_S [nmasks * nk * ndof * ndof] column-major
 * complex128, leading d x d block valid (kept dofs in natural order), rest zero; d_dims [nmasks] = d.
 * d_S may be NULL.  For the commuting pencil H = eps0 I + t T and S = I + s T are materialised. */
int hx_assemble_device(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk, const uint64_t* d_masks,
                       int64_t nmasks, double* d_H, double* d_S, int32_t* d_dims, void* stream);

/* ---- the hot path ---------------------------------------------------------------------------- */
/* Smoothed IDOS curves of a batch of vacancy masks on one (nu, q) grid.
 * Replaces: parallel_map(_eval_job, jobs) for the new (deduplicated) jobs of one (n, q) group
 * (runner.py:218-244) = solve_bands (spectrum.py:120-134) + idos (qoi.py:96-102) per mask.
 *   masks      [nmasks * words] uint64, words = ceil(nunits/64), bit u = unit u vacant (disorder.py:40-46)
 *   kpoints    [nk * 2] k-points (make_bz_grid order, spectrum.py:59-84), each weighted 1/nk
 *   out_curves [nmasks * npts] I(eps_m) per mask (caller-owned)
 *   out_eigs   optional [nmasks * nk * ndof] ascending eigenvalues, NaN-padded past the kept dim
 *   out_status [nmasks * nk] HX_ST_* per (mask, k)
 * Host-pointer variant: copies in/out inside the call (synchronous). */
int hx_eval_idos_batch(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk,
                       const uint64_t* masks, int64_t nmasks, const hx_egrid* grid,
                       double* out_curves, double* out_eigs, int32_t* out_status);
/* Device-pointer variant: all arrays are device pointers; asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default).  kpoints stays a host array. */
int hx_eval_idos_batch_device(hx_ctx* ctx, hx_cell* cell, const double* kpoints, int32_t nk,
                              const uint64_t* d_masks, int64_t nmasks, const hx_egrid* grid,
                              double* d_curves, double* d_eigs, int32_t* d_status, void* stream);

/* Weighted k-point variants (IDOS only, no eigenvalue output): kmult[k] >= 1 is the multiplicity of
 * k-point k, the IDOS weights are kmult[k] / sum(kmult) (qoi.py:96-102 with BzGrid weights).  Used with
 * time-reversal pairs merged: for real-amplitude models H(-k) = conj(H(k)) has the spectrum of H(k),
 * so k and -k of the reference's grid (spectrum.py:59-84) are solved once with multiplicity 2.
 * out_status / d_status: [nmasks x nk] for the given (representative) k-points. */
int hx_eval_idos_batch_k(hx_ctx* ctx, hx_cell* cell, const double* kpoints, const int32_t* kmult, int32_t nk,
                         const uint64_t* masks, int64_t nmasks, const hx_egrid* grid, double* out_curves,
                         int32_t* out_status);
int hx_eval_idos_batch_device_k(hx_ctx* ctx, hx_cell* cell, const double* kpoints, const int32_t* kmult,
                                int32_t nk, const uint64_t* d_masks, int64_t nmasks, const hx_egrid* grid,
                                double* d_curves, int32_t* d_status, void* stream);

/* Batched Hermitian (generalized) eigenvalues of caller-assembled matrices (config-5 sweep,
 * unit parity with spectrum._eigvals, spectrum.py:100-117).  A, B: device, column-major complex128
 * (interleaved re/im), n x n each, `batch` matrices; B == NULL -> standard problem.
 * d_eigs [batch * n] ascending.  d_status [batch]. */
int hx_eigvalsh_batch_device(hx_ctx* ctx, int32_t n, int64_t batch, const double* d_A, const double* d_B,
                             double* d_eigs, int32_t* d_status, void* stream);

/* ---- kernel-module parity (_kernels.py:32-56), device pointers ------------------------------- */
/* out[npts] += smoothed counts of (energies, weights) — smoothed_counts (_kernels.py:68-88). */
int hx_smoothed_counts_device(const double* d_energies, const double* d_weights, int64_t count,
                              const hx_egrid* grid, double* d_out, void* stream);
/* out[npts] += sharp counts — sharp_counts (_kernels.py:91-101). */
int hx_sharp_counts_device(const double* d_energies, const double* d_weights, int64_t count,
                           const hx_egrid* grid, double* d_out, void* stream);

/* ---- MLMC level moments (runner.py:281-299 + mlmc.py:143-154), device pointers ------------- */
/* term[m] = full[m] - 0.25 * sum_r quarter[m][r] (quarters may be NULL -> no CV);
 * mean = sum_m term / M, var = sum (term-mean)^2 / (M-1) (M>1 else NaN) - the two-pass np.var form, with
 * both sums EXACT (fixed point, see below), so they do not depend on the order or split of the samples.
 * d_terms optional [M * npts]; d_mean / d_var optional [npts]. */
int hx_level_moments_device(const double* d_full, const double* d_quarters, int64_t M, int32_t npts,
                            double* d_terms, double* d_mean, double* d_var, void* stream);

/* Exact fixed-point level sums for multi-device / multi-rank levels (north_star (4)).
 * Every term is converted on its own to a fixed-point integer of HX_FX_LIMBS signed 32-bit limbs (held in
 * int64, HX_FX_FRAC fraction bits; |term| < 2^(32*HX_FX_LIMBS - HX_FX_FRAC - 1)) and the limbs are summed
 * as integers, so partial limbs of any split of the samples add (an int64 all-reduce, ncclInt64) to the
 * bits of the single-device sum.  d_limbs [npts * HX_FX_LIMBS] (overwritten):
 *   d_center == NULL : sum_m term_m          (pass 1; mean = finalize(sum, M_total))
 *   d_center != NULL : sum_m (term_m - center)^2  (pass 2 with the global mean; var = finalize(sum, M_total-1))
 * hx_level_moments_device computes its mean / var through the same functions, so one device and G devices
 * agree bitwise. */
#define HX_FX_LIMBS 6
#define HX_FX_FRAC 112
int hx_level_sums_fixed_device(const double* d_full, const double* d_quarters, int64_t M, int32_t npts,
                               const double* d_center, int64_t* d_limbs, void* stream);
/* out[m] = value(limbs[m]) / divisor (divisor <= 0 -> NaN). */
int hx_fixed_finalize_device(const int64_t* d_limbs, int32_t npts, double divisor, double* d_out, void* stream);
/* Host-pointer twins (same arithmetic, bitwise equal to the device ones); used by the CPU multi-rank tests. */
int hx_level_sums_fixed(const double* full, const double* quarters, int64_t M, int32_t npts, const double* center,
                        int64_t* limbs);
int hx_fixed_finalize(const int64_t* limbs, int32_t npts, double divisor, double* out);

/* ---- disorder sampling (disorder.py:57-94), host C, bit-exact with numpy ---------------------- */
/* SeedSequence(seed, spawn_key=(level, rep0 + i)) -> PCG64 -> random(nunits) < p, for i < count.
 * out_words [count * ceil(nunits/64)].  seed < 2^64, level/rep < 2^32 each. threads <= 0: auto. */
int hx_sample_masks(uint64_t seed, uint64_t level, uint64_t rep0, int64_t count, double p, int32_t nunits,
                    uint64_t* out_words, int32_t threads);
/* Same on the device (K7): d_out_words [count * words]. */
int hx_sample_masks_device(uint64_t seed, uint64_t level, uint64_t rep0, int64_t count, double p,
                           int32_t nunits, uint64_t* d_out_words, void* stream);
/* The first `count` uniforms of one stream (parity checks against numpy Generator.random). */
int hx_uniforms(uint64_t seed, uint64_t level, uint64_t rep, int64_t count, double* out);
/* Quarter restriction of parent masks (restrict, disorder.py:84-94): for each parent mask and
 * r = 1..4, out[(i*4 + r-1) * sub_words ...] = bits u' = unit_map[u] of units with assign[u] == r. */
int hx_restrict_masks(const uint64_t* parent_words, int64_t nmasks, int32_t parent_units,
                      const int32_t* unit_assign, const int32_t* unit_map, int32_t sub_units,
                      uint64_t* out_words);

/* Device variant of hx_restrict_masks (device pointers; quarter labels/unit map uploaded by caller). */
int hx_restrict_masks_device(const uint64_t* d_parent_words, int64_t nmasks, int32_t parent_units,
                             const int32_t* d_unit_assign, const int32_t* d_unit_map, int32_t sub_units,
                             uint64_t* d_out_words, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HX_H_ */
