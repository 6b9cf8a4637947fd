// Bipartite fast path of the shared-memory tier (graphene commuting pencil).
//
// With dofs split by sublattice, the phase matrix is T = [[0, C], [C^H, 0]] (C = nA x nB, vacancies keep
// the structure), so the eigenvalues of T are +-sigma_j(C) plus |nA - nB| zeros.  C (or C^H, so that
// rows >= columns) is reduced to upper bidiagonal form B = U^H C V by alternating left/right Householder
// reflectors (Golub-Kahan); the perfect-shuffle permutation of [[0, B], [B^H, 0]] is the tridiagonal with
// zero diagonal and off-diagonals |alpha_0|, |gamma_0|, |alpha_1|, ... (the TGK matrix), followed by
// isolated zeros for the extra rows.  That tridiagonal is written in the same (diag, e2) format as the
// Hermitian tiers and goes through the same bisection + IDOS kernel.  Work: ~4x fewer flops than
// tridiagonalising the d x d matrix T and 1/4 of the shared memory.
#pragma once
#include "hx_dense.cuh"

namespace hx {

// Compaction per sublattice: idx_a[r] / idx_b[r] = rank of kept dof r among kept dofs of sublattice 0 / 1
// (natural order, -1 otherwise).  Returns (nA, nB).  cnt: 2*ceil(N/32) ints.
static __device__ int2 block_compact_bipartite(const CellDev& c, const uint64_t* mask, int* idx_a, int* idx_b,
                                               int* cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nch = (c.N + 31) >> 5;
  auto keep_of = [&](int r) {
    if (r >= c.N) return false;
    const int u = c.unit_of_dof[r];
    return (u < 0) || !((mask[u >> 6] >> (u & 63)) & 1ull);
  };
  for (int ch = warp; ch < nch; ch += nw) {
    const int r = (ch << 5) + lane;
    const bool kp = keep_of(r);
    const int sb = r < c.N ? c.sub[r] : 0;
    const unsigned ba = __ballot_sync(0xffffffffu, kp && sb == 0), bb = __ballot_sync(0xffffffffu, kp && sb == 1);
    if (lane == 0) {
      cnt[ch] = __popc(ba);
      cnt[nch + ch] = __popc(bb);
    }
  }
  __syncthreads();
  for (int ch = warp; ch < nch; ch += nw) {
    int oa = 0, ob = 0;
    for (int q = 0; q < ch; ++q) {
      oa += cnt[q];
      ob += cnt[nch + q];
    }
    const int r = (ch << 5) + lane;
    const bool kp = keep_of(r);
    const int sb = r < c.N ? c.sub[r] : 0;
    const unsigned ba = __ballot_sync(0xffffffffu, kp && sb == 0), bb = __ballot_sync(0xffffffffu, kp && sb == 1);
    const unsigned lt = (1u << lane) - 1u;
    if (r < c.N) {
      idx_a[r] = (kp && sb == 0) ? oa + __popc(ba & lt) : -1;
      idx_b[r] = (kp && sb == 1) ? ob + __popc(bb & lt) : -1;
    }
  }
  int na = 0, nb = 0;
  for (int q = 0; q < nch; ++q) {
    na += cnt[q];
    nb += cnt[nch + q];
  }
  __syncthreads();
  return make_int2(na, nb);
}

// Assemble M (rows >= cols) into column-major smem (ld = lm).  idx_a / idx_b: compacted rank of each
// kept dof inside its sublattice (-1 if removed or other sublattice).  If transpose, M = C^H.
// periodic: multiply by exp(i k.(pos_a - pos_b)) and keep the real part (the periodic gauge of a batch whose
// k-points make it real, see bd_assemble_kernel).
static __device__ void assemble_bipartite(const CellDev& c, const int* idx_a, const int* idx_b, double2 k,
                                          double2* M, int lm, int rows, int cols, bool transpose,
                                          bool periodic = false, double* Mr = nullptr) {
  // Mr (periodic only): write the real matrix as doubles instead (real stage 1, hx_real.cuh)
  if (Mr)
    for (int p = threadIdx.x; p < lm * cols; p += blockDim.x) Mr[p] = 0.0;
  else
    for (int p = threadIdx.x; p < lm * cols; p += blockDim.x) M[p] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int r = threadIdx.x; r < c.N; r += blockDim.x) {
    const int ia = idx_a[r];
    if (ia < 0) continue;
    // partners of the A dof r: own targets, then sources pointing at r (distinct, kept, sublattice B)
    auto visit = [&](int cb) {
      const int jb = idx_b[cb];
      if (jb < 0) return;
      double2 h = herm_element(c.h_ptr, c.h_col, c.h_amp, c.h_disp, r, cb, k);
      if (periodic) {
        const double2 pa = c.pos[r], pb = c.pos[cb];
        double sn, cs;
        sincos(k.x * (pa.x - pb.x) + k.y * (pa.y - pb.y), &sn, &cs);
        h = make_double2(h.x * cs - h.y * sn, 0.0);
        if (Mr) {
          if (!transpose) Mr[ia + (size_t)jb * lm] = h.x;
          else Mr[jb + (size_t)ia * lm] = h.x;
          return;
        }
      }
      if (!transpose) M[ia + (size_t)jb * lm] = h;
      else M[jb + (size_t)ia * lm] = make_double2(h.x, -h.y);
    };
    for (int e = c.h_ptr[r]; e < c.h_ptr[r + 1]; ++e) {
      const int cb = c.h_col[e];
      bool dup = false;
      for (int e2 = c.h_ptr[r]; e2 < e; ++e2) dup |= (c.h_col[e2] == cb);
      if (!dup) visit(cb);
    }
    for (int t = c.ht_ptr[r]; t < c.ht_ptr[r + 1]; ++t) {
      const int cb = c.h_src[c.ht_inst[t]];
      bool dup = false;
      for (int e2 = c.h_ptr[r]; e2 < c.h_ptr[r + 1]; ++e2) dup |= (c.h_col[e2] == cb);
      for (int t2 = c.ht_ptr[r]; t2 < t; ++t2) dup |= (c.h_src[c.ht_inst[t2]] == cb);
      if (!dup) visit(cb);
    }
  }
  __syncthreads();
}

// Golub-Kahan bidiagonalisation of M (rows x cols, rows >= cols, column-major smem, ld lm).
// Writes the TGK tridiagonal: diag[0..d) = 0, e2 = |alpha_0|^2, |gamma_0|^2, ..., |alpha_{cols-1}|^2,
// then zeros (d = rows + cols).  u, s: complex scratch of max(rows, cols); red: 128 doubles.
static __device__ void bidiag_tgk(double2* M, int lm, int rows, int cols, double* diag, double* e2, double2* u,
                                  double2* s, double* red) {
  (void)s;
  const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = bd >> 5;
  const int d = rows + cols;
  for (int i = tid; i < d; i += bd) {
    diag[i] = 0.0;
    e2[i] = 0.0;
  }
  // Thread layouts (no integer division, conflict-free: 8 consecutive lanes walk 8 consecutive rows):
  //   left  (column) pass: row group g = lane & 7, column (tid >> 3) + k * bd/8; sums over g by xor 1,2,4
  //   right (row) pass:    row (lane & 7) + 8 * warp + k * 8 nw, column group q = lane >> 3 (4 groups);
  //                        sums over q by xor 8,16
  // Two barriers per reflector: the squared norm the NEXT reflector needs (row j after the left update,
  // column j+1 after the right update) is accumulated by the threads that write those entries and
  // combined from per-warp partials (red[0..31]: column norm, red[32..63]: row norm).
  const int g = lane & 7, q = lane >> 3;
  double* lred = red;
  double* rred = red + 32;
  {
    double part = 0.0;
    for (int i = tid; i < rows; i += bd) {
      const double2 x = M[i];
      part = fma(x.x, x.x, fma(x.y, x.y, part));
    }
    part = warp_sum(part);
    if (lane == 0) lred[warp] = part;
    __syncthreads();
  }
  for (int j = 0; j < cols; ++j) {
    // ---------------- left reflector: column j, rows j..rows-1
    {
      double sig2 = 0.0;
      for (int w = 0; w < nw; ++w) sig2 += lred[w];
      const double2* colj = M + (size_t)j * lm;
      const QuickReflector h = quick_reflector(colj[j], sig2);
      if (tid == 0) e2[2 * j] = sig2;
      for (int i = j + tid; i < rows; i += bd) u[i] = i == j ? make_double2(1.0, 0.0) : cmul(colj[i], h.scale);
      __syncthreads();
      // M[:, c] -= v (tau v^H M[:, c]) for c > j: 8 lanes per column, the column sum stays in the group
      double rpart = 0.0;  // |M[j][c]|^2 after the update (row norm for the right reflector)
      for (int c0 = j + 1; c0 < cols; c0 += bd >> 3) {
        const int cc = c0 + (tid >> 3);
        double2 acc = make_double2(0.0, 0.0);
        if (cc < cols && h.tau != 0.0)
          for (int i = j + g; i < rows; i += 8) {
            const double2 a = u[i], b = M[i + (size_t)cc * lm];
            acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
            acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
          }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
        const double2 sc = make_double2(h.tau * acc.x, h.tau * acc.y);
        if (cc < cols) {
          if (h.tau != 0.0)
            for (int i = j + g; i < rows; i += 8) {
              const double2 a = u[i];
              double2 x = M[i + (size_t)cc * lm];
              x.x = fma(-a.x, sc.x, fma(a.y, sc.y, x.x));
              x.y = fma(-a.x, sc.y, fma(-a.y, sc.x, x.y));
              M[i + (size_t)cc * lm] = x;
              if (i == j) rpart = fma(x.x, x.x, fma(x.y, x.y, rpart));
            }
          else if (g == 0) {
            const double2 x = M[j + (size_t)cc * lm];
            rpart = fma(x.x, x.x, fma(x.y, x.y, rpart));
          }
        }
      }
      rpart = warp_sum(rpart);
      if (lane == 0) rred[warp] = rpart;
      __syncthreads();
    }
    if (j + 1 >= cols) break;
    // ---------------- right reflector: row j, columns j+1..cols-1 (on the conjugated row)
    {
      double sig2 = 0.0;
      for (int w = 0; w < nw; ++w) sig2 += rred[w];
      const double2 a0 = M[j + (size_t)(j + 1) * lm];
      const QuickReflector h = quick_reflector(make_double2(a0.x, -a0.y), sig2);
      if (tid == 0) e2[2 * j + 1] = sig2;
      // u_c from conj(row j): u_{j+1} = 1
      for (int cc = j + 1 + tid; cc < cols; cc += bd) {
        const double2 x = M[j + (size_t)cc * lm];
        u[cc] = cc == j + 1 ? make_double2(1.0, 0.0) : cmul(make_double2(x.x, -x.y), h.scale);
      }
      __syncthreads();
      // M[r, :] -= (tau M[r, :] u) u^H for rows r > j: 4 lanes per row (column groups)
      double lpart = 0.0;  // |M[r][j+1]|^2, r > j, after the update (column norm for the next left)
      for (int r0 = j + 1; r0 < rows; r0 += 8 * nw) {
        const int r = r0 + g + 8 * warp;
        double2 acc = make_double2(0.0, 0.0);
        if (r < rows && h.tau != 0.0)
          for (int cc = j + 1 + q; cc < cols; cc += 4) {
            const double2 a = M[r + (size_t)cc * lm], b = u[cc];
            acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
            acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
          }
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 8);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 8);
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
        const double2 w = make_double2(h.tau * acc.x, h.tau * acc.y);
        if (r < rows) {
          if (h.tau != 0.0)
            for (int cc = j + 1 + q; cc < cols; cc += 4) {
              const double2 b = u[cc];
              double2 x = M[r + (size_t)cc * lm];
              // x -= w conj(b)
              x.x = fma(-w.x, b.x, fma(-w.y, b.y, x.x));
              x.y = fma(-w.y, b.x, fma(w.x, b.y, x.y));
              M[r + (size_t)cc * lm] = x;
              if (cc == j + 1) lpart = fma(x.x, x.x, fma(x.y, x.y, lpart));
            }
          else if (q == 0) {
            const double2 x = M[r + (size_t)(j + 1) * lm];
            lpart = fma(x.x, x.x, fma(x.y, x.y, lpart));
          }
        }
      }
      lpart = warp_sum(lpart);
      if (lane == 0) lred[warp] = lpart;
      __syncthreads();
    }
  }
  __syncthreads();
}

// Leading dimension of the bidiagonalisation workspace: >= S + 1 and = 1 (mod 8) in 16-byte units, so
// that lanes walking different columns at the same row hit distinct banks.
__host__ __device__ constexpr int bidiag_ld(int S) { return (S + 7) / 8 * 8 + 1; }

// Same reduction with ONE WARP per matrix (no CTA barriers, only __syncwarp): lanes own columns in the
// left (column) pass and rows in the right (row) pass, two accumulators per lane for latency hiding.
// Used for S <= 64 where a 256-thread CTA spends most of its time in per-step barriers and reductions.
static __device__ void bidiag_tgk_warp(double2* M, int lm, int rows, int cols, double* diag, double* e2,
                                       double2* u) {
  const int lane = threadIdx.x & 31;
  const int d = rows + cols;
  for (int i = lane; i < d; i += 32) {
    diag[i] = 0.0;
    e2[i] = 0.0;
  }
  for (int j = 0; j < cols; ++j) {
    // ---------------- left reflector: column j, rows j..rows-1
    {
      const double2* colj = M + (size_t)j * lm;
      double part = 0.0;
      for (int i = j + lane; i < rows; i += 32) part = fma(colj[i].x, colj[i].x, fma(colj[i].y, colj[i].y, part));
      const double sig2 = warp_sum(part);
      const QuickReflector h = quick_reflector(colj[j], sig2);
      if (lane == 0) e2[2 * j] = sig2;
      for (int i = j + lane; i < rows; i += 32) u[i] = i == j ? make_double2(1.0, 0.0) : cmul(colj[i], h.scale);
      __syncwarp();
      if (h.tau != 0.0)
        // two columns per lane (c0, c0 + 32): the u loads are shared and the two dot chains interleave
        for (int c0 = j + 1 + lane; c0 < cols; c0 += 64) {
          const bool has1 = c0 + 32 < cols;
          double2* col0 = M + (size_t)c0 * lm;
          double2* col1 = M + (size_t)(has1 ? c0 + 32 : c0) * lm;
          double2 a0 = make_double2(0.0, 0.0), a1 = a0;
#pragma unroll 2
          for (int i = j; i < rows; ++i) {
            const double2 v = u[i], x0 = col0[i], x1 = col1[i];
            a0.x = fma(v.x, x0.x, fma(v.y, x0.y, a0.x));
            a0.y = fma(v.x, x0.y, fma(-v.y, x0.x, a0.y));
            a1.x = fma(v.x, x1.x, fma(v.y, x1.y, a1.x));
            a1.y = fma(v.x, x1.y, fma(-v.y, x1.x, a1.y));
          }
          const double2 s0 = make_double2(h.tau * a0.x, h.tau * a0.y);
          const double2 s1 = make_double2(has1 ? h.tau * a1.x : 0.0, has1 ? h.tau * a1.y : 0.0);
#pragma unroll 2
          for (int i = j; i < rows; ++i) {
            const double2 v = u[i];
            double2 x0 = col0[i], x1 = col1[i];
            x0.x = fma(-v.x, s0.x, fma(v.y, s0.y, x0.x));
            x0.y = fma(-v.x, s0.y, fma(-v.y, s0.x, x0.y));
            x1.x = fma(-v.x, s1.x, fma(v.y, s1.y, x1.x));
            x1.y = fma(-v.x, s1.y, fma(-v.y, s1.x, x1.y));
            col0[i] = x0;
            if (has1) col1[i] = x1;
          }
        }
      __syncwarp();
    }
    if (j + 1 >= cols) break;
    // ---------------- right reflector: row j, columns j+1..cols-1 (on the conjugated row)
    {
      double part = 0.0;
      for (int cc = j + 1 + lane; cc < cols; cc += 32) {
        const double2 x = M[j + (size_t)cc * lm];
        part = fma(x.x, x.x, fma(x.y, x.y, part));
      }
      const double sig2 = warp_sum(part);
      const double2 a0 = M[j + (size_t)(j + 1) * lm];
      const QuickReflector h = quick_reflector(make_double2(a0.x, -a0.y), sig2);
      if (lane == 0) e2[2 * j + 1] = sig2;
      for (int cc = j + 1 + lane; cc < cols; cc += 32) {
        const double2 x = M[j + (size_t)cc * lm];
        u[cc] = cc == j + 1 ? make_double2(1.0, 0.0) : cmul(make_double2(x.x, -x.y), h.scale);
      }
      __syncwarp();
      if (h.tau != 0.0)
        // two rows per lane (r0, r0 + 32), shared u loads, interleaved chains
        for (int r0 = j + 1 + lane; r0 < rows; r0 += 64) {
          const bool has1 = r0 + 32 < rows;
          const int r1 = has1 ? r0 + 32 : r0;
          double2 a0 = make_double2(0.0, 0.0), a1 = a0;
#pragma unroll 2
          for (int cc = j + 1; cc < cols; ++cc) {
            const double2 b = u[cc], x0 = M[r0 + (size_t)cc * lm], x1 = M[r1 + (size_t)cc * lm];
            a0.x = fma(x0.x, b.x, fma(-x0.y, b.y, a0.x));
            a0.y = fma(x0.x, b.y, fma(x0.y, b.x, a0.y));
            a1.x = fma(x1.x, b.x, fma(-x1.y, b.y, a1.x));
            a1.y = fma(x1.x, b.y, fma(x1.y, b.x, a1.y));
          }
          const double2 w0 = make_double2(h.tau * a0.x, h.tau * a0.y);
          const double2 w1 = make_double2(has1 ? h.tau * a1.x : 0.0, has1 ? h.tau * a1.y : 0.0);
#pragma unroll 2
          for (int cc = j + 1; cc < cols; ++cc) {
            const double2 b = u[cc];
            double2 x0 = M[r0 + (size_t)cc * lm], x1 = M[r1 + (size_t)cc * lm];
            x0.x = fma(-w0.x, b.x, fma(-w0.y, b.y, x0.x));
            x0.y = fma(-w0.y, b.x, fma(w0.x, b.y, x0.y));
            x1.x = fma(-w1.x, b.x, fma(-w1.y, b.y, x1.x));
            x1.y = fma(-w1.y, b.x, fma(w1.x, b.y, x1.y));
            M[r0 + (size_t)cc * lm] = x0;
            if (has1) M[r1 + (size_t)cc * lm] = x1;
          }
        }
      __syncwarp();
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------------------------------------------
// Register-resident Golub-Kahan for complex S <= 64 on 256 threads (hx_kernels.cuh BIDIAG_REG_THREADS).  The shared-memory
// CTA variant above reads every active element of M twice and writes it once per reflector from shared
// memory - ~50 bytes per complex FMA pair, which makes it shared-memory-bandwidth bound at ~4 TF/s.  Here
// the matrix lives in registers: thread (a, b) = (lane & 15, 2 warp + (lane >> 4)) owns the 4 x 4 complex
// elements M[a + 16 i][b + 16 k] (cyclic, so the active trailing block stays spread over every thread) and
// shared memory only carries the reflectors and the reductions:
//   left  (column j): the 16 owners of column j (one half-warp) build u, one barrier; the column dots
//         reduce over the 16 lanes a of a half-warp (reduce-scatter by shuffles + a shared-memory
//         all-gather inside the half-warp), no barrier;
//   right (row j): the owners of row j publish it with their norm partials, one barrier; every thread
//         builds the same reflector; the row dots reduce over b (xor-16 shuffle, then 8 warps through
//         shared memory: two barriers).
// Scratch (doubles): BIDIAG_REG_SCRATCH.  Same TGK output as bidiag_tgk.
constexpr int BIDIAG_REG_SCRATCH = 128 + 2 + 128 + 128 + 8 + 1024 + 128;

struct GkRegScratch {
  double2* ubuf;    // 64: left reflector u
  double* stau;     // left tau
  double* sv;       // 16 x 8: tau u^H M per column class
  double2* rowbuf;  // 64: row j after the left update
  double* nred;     // 8: row-norm partials per warp
  double* wred;     // 8 warps x 8 x 16: row-dot partials
  double* wv;       // 4 x 16 double2: tau M u per row
};

// Steps j in [16 T, min(16 T + 16, cols)): rows and columns below 16 T are finished, so the register blocks
// i < T and k < T are skipped statically; the partial block T is masked through u / s / w.
template <int T>
static __device__ __forceinline__ void gk_reg_phase(double2 (&m)[4][4], int rows, int cols, double* e2,
                                                    const GkRegScratch& sc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane & 15, hb = lane >> 4, b = 2 * warp + hb;
  const unsigned FULL = 0xffffffffu;
  const int jend = min(16 * T + 16, cols);
  for (int j = 16 * T; j < jend; ++j) {
    const int jl = j & 15;
    // ---------------- left reflector: column j (owners: b == jl, one half-warp of warp jl >> 1)
    if (warp == (jl >> 1)) {
      double part = 0.0;
#pragma unroll
      for (int i = T; i < 4; ++i)
        if (i > T || a >= jl) part = fma(m[i][T].x, m[i][T].x, fma(m[i][T].y, m[i][T].y, part));
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) part += __shfl_xor_sync(FULL, part, o);
      const int src = 16 * (j & 1) + jl;
      const double2 alpha = make_double2(__shfl_sync(FULL, m[T][T].x, src), __shfl_sync(FULL, m[T][T].y, src));
      const QuickReflector h = quick_reflector(alpha, part);
      if (hb == (j & 1)) {
#pragma unroll
        for (int i = T; i < 4; ++i) {
          const int r = a + 16 * i;
          sc.ubuf[r] = r < j ? make_double2(0.0, 0.0) : (r == j ? make_double2(1.0, 0.0) : cmul(m[i][T], h.scale));
        }
        if (lane == src) {
          *sc.stau = h.tau;
          e2[2 * j] = part;
        }
      }
    }
    __syncthreads();  // A: u, tau
    {
      const double tau = *sc.stau;
      double2 uu[4];
#pragma unroll
      for (int i = T; i < 4; ++i) uu[i] = sc.ubuf[a + 16 * i];
      double v[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double2 acc = make_double2(0.0, 0.0);
        if (k >= T)
#pragma unroll
          for (int i = T; i < 4; ++i) {
            const double2 x = m[i][k];
            acc.x = fma(uu[i].x, x.x, fma(uu[i].y, x.y, acc.x));
            acc.y = fma(uu[i].x, x.y, fma(-uu[i].y, x.x, acc.y));
          }
        v[2 * k] = acc.x;
        v[2 * k + 1] = acc.y;
      }
      // reduce-scatter over the 16 lanes a: the lane ends with the sum of value p = (a >> 1) & 7
      double w4[4], w2[2];
      const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        w4[t] = t + 4 < 2 * T ? 0.0  // values of skipped blocks: zero on both sides
                              : (b3 ? v[t + 4] : v[t]) + __shfl_xor_sync(FULL, b3 ? v[t] : v[t + 4], 8);
#pragma unroll
      for (int t = 0; t < 2; ++t) w2[t] = (b2 ? w4[t + 2] : w4[t]) + __shfl_xor_sync(FULL, b2 ? w4[t] : w4[t + 2], 4);
      double w1 = (b1 ? w2[1] : w2[0]) + __shfl_xor_sync(FULL, b1 ? w2[0] : w2[1], 2);
      w1 += __shfl_xor_sync(FULL, w1, 1);
      if (!(a & 1)) {
        const int p = a >> 1, c = b + 16 * (p >> 1);
        sc.sv[b * 8 + p] = c > j ? tau * w1 : 0.0;
      }
      __syncwarp();
      const double2* s2 = reinterpret_cast<const double2*>(sc.sv + b * 8);
#pragma unroll
      for (int k = T; k < 4; ++k) {
        const double2 s = s2[k];
#pragma unroll
        for (int i = T; i < 4; ++i) {
          double2 x = m[i][k];
          x.x = fma(-uu[i].x, s.x, fma(uu[i].y, s.y, x.x));
          x.y = fma(-uu[i].x, s.y, fma(-uu[i].y, s.x, x.y));
          m[i][k] = x;
        }
      }
    }
    if (j + 1 >= cols) break;
    // owners of row j (a == jl) publish its columns > j and their squared norm
    {
      double np = 0.0;
      if (a == jl) {
#pragma unroll
        for (int k = T; k < 4; ++k) {
          const int c = b + 16 * k;
          const double2 x = c > j ? m[T][k] : make_double2(0.0, 0.0);
          sc.rowbuf[c] = x;
          np = fma(x.x, x.x, fma(x.y, x.y, np));
        }
      }
      np += __shfl_xor_sync(FULL, np, 16);
      if (lane == jl) sc.nred[warp] = np;
    }
    __syncthreads();  // B: row j, norm partials
    // ---------------- right reflector: row j, columns j+1.. (every thread builds the same one)
    {
      const double2* nr2 = reinterpret_cast<const double2*>(sc.nred);
      double sig2 = 0.0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const double2 x = nr2[w];
        sig2 += x.x;
        sig2 += x.y;
      }
      const double2 a0 = sc.rowbuf[j + 1];
      const QuickReflector h = quick_reflector(make_double2(a0.x, -a0.y), sig2);
      if (tid == 0) e2[2 * j + 1] = sig2;
      double2 uc[4];
#pragma unroll
      for (int k = T; k < 4; ++k) {
        const int c = b + 16 * k;
        const double2 x = sc.rowbuf[c];
        uc[k] = c == j + 1 ? make_double2(1.0, 0.0) : cmul(make_double2(x.x, -x.y), h.scale);
      }
      double v[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double2 acc = make_double2(0.0, 0.0);
        if (i >= T)
#pragma unroll
          for (int k = T; k < 4; ++k) {
            const double2 x = m[i][k];
            acc.x = fma(x.x, uc[k].x, fma(-x.y, uc[k].y, acc.x));
            acc.y = fma(x.x, uc[k].y, fma(x.y, uc[k].x, acc.y));
          }
        v[2 * i] = acc.x;
        v[2 * i + 1] = acc.y;
      }
      // the two column classes of the warp (xor 16), then the 8 warps through shared memory
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double r = (hb ? v[t + 4] : v[t]) + __shfl_xor_sync(FULL, hb ? v[t] : v[t + 4], 16);
        sc.wred[(warp * 8 + hb * 4 + t) * 16 + a] = r;
      }
      __syncthreads();  // C: row-dot partials
      if (tid < 128) {
        const int ar = tid & 15, p = tid >> 4;
        double sum = 0.0;
        if ((p >> 1) >= T) {
#pragma unroll
          for (int w = 0; w < 8; ++w) sum += sc.wred[(w * 8 + p) * 16 + ar];
        }
        const int r = ar + 16 * (p >> 1);
        sc.wv[((p >> 1) * 16 + ar) * 2 + (p & 1)] = r > j ? h.tau * sum : 0.0;
      }
      __syncthreads();  // D: tau M u
      const double2* wv2 = reinterpret_cast<const double2*>(sc.wv);
#pragma unroll
      for (int i = T; i < 4; ++i) {
        const double2 w = wv2[i * 16 + a];
#pragma unroll
        for (int k = T; k < 4; ++k) {
          double2 x = m[i][k];
          // x -= w conj(u_c)
          x.x = fma(-w.x, uc[k].x, fma(-w.y, uc[k].y, x.x));
          x.y = fma(-w.y, uc[k].x, fma(w.x, uc[k].y, x.y));
          m[i][k] = x;
        }
      }
    }
  }
}

static __device__ void bidiag_tgk_reg(const double2* Ms, int lm, int rows, int cols, double* diag, double* e2,
                                      double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane & 15, b = 2 * warp + (lane >> 4);
  GkRegScratch sc;
  sc.ubuf = reinterpret_cast<double2*>(scratch);
  sc.stau = scratch + 128;
  sc.sv = scratch + 130;
  sc.rowbuf = reinterpret_cast<double2*>(scratch + 258);
  sc.nred = scratch + 386;
  sc.wred = scratch + 394;
  sc.wv = scratch + 1418;
  const int d = rows + cols;
  for (int i = tid; i < d; i += blockDim.x) {
    diag[i] = 0.0;
    e2[i] = 0.0;
  }
  double2 m[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = a + 16 * i, c = b + 16 * k;
      m[i][k] = (r < rows && c < cols) ? Ms[r + (size_t)c * lm] : make_double2(0.0, 0.0);
    }
  gk_reg_phase<0>(m, rows, cols, e2, sc);
  if (cols > 16) gk_reg_phase<1>(m, rows, cols, e2, sc);
  if (cols > 32) gk_reg_phase<2>(m, rows, cols, e2, sc);
  if (cols > 48) gk_reg_phase<3>(m, rows, cols, e2, sc);
  __syncthreads();
}

// Real register-resident variant (TRIM k-points, S <= 64): the same schedule on doubles, 4 x 4 per thread.
// Scratch (doubles): BIDIAG_REG_SCRATCH_REAL.
constexpr int BIDIAG_REG_SCRATCH_REAL = 64 + 2 + 64 + 64 + 8 + 512 + 64;

struct GkRegScratchReal {
  double* ubuf;    // 64
  double* stau;
  double* sv;      // 16 x 4
  double* rowbuf;  // 64
  double* nred;    // 8
  double* wred;    // 8 warps x 4 x 16
  double* wv;      // 4 x 16
};

template <int T>
static __device__ __forceinline__ void gk_reg_phase_real(double (&m)[4][4], int rows, int cols, double* e2,
                                                         const GkRegScratchReal& sc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane & 15, hb = lane >> 4, b = 2 * warp + hb;
  const unsigned FULL = 0xffffffffu;
  const int jend = min(16 * T + 16, cols);
  for (int j = 16 * T; j < jend; ++j) {
    const int jl = j & 15;
    if (warp == (jl >> 1)) {
      double part = 0.0;
#pragma unroll
      for (int i = T; i < 4; ++i)
        if (i > T || a >= jl) part = fma(m[i][T], m[i][T], part);
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) part += __shfl_xor_sync(FULL, part, o);
      const int src = 16 * (j & 1) + jl;
      const double alpha = __shfl_sync(FULL, m[T][T], src);
      const QuickReflector h = quick_reflector(make_double2(alpha, 0.0), part);
      if (hb == (j & 1)) {
#pragma unroll
        for (int i = T; i < 4; ++i) {
          const int r = a + 16 * i;
          sc.ubuf[r] = r < j ? 0.0 : (r == j ? 1.0 : m[i][T] * h.scale.x);
        }
        if (lane == src) {
          *sc.stau = h.tau;
          e2[2 * j] = part;
        }
      }
    }
    __syncthreads();  // A
    {
      const double tau = *sc.stau;
      double uu[4];
#pragma unroll
      for (int i = T; i < 4; ++i) uu[i] = sc.ubuf[a + 16 * i];
      double v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double acc = 0.0;
        if (k >= T)
#pragma unroll
          for (int i = T; i < 4; ++i) acc = fma(uu[i], m[i][k], acc);
        v[k] = acc;
      }
      // reduce-scatter over the 16 lanes a: the lane ends with the sum of value k = (a >> 2) & 3
      const bool b3 = lane & 8, b2 = lane & 4;
      double w2[2];
#pragma unroll
      for (int t = 0; t < 2; ++t)
        w2[t] = t + 2 < T ? 0.0 : (b3 ? v[t + 2] : v[t]) + __shfl_xor_sync(FULL, b3 ? v[t] : v[t + 2], 8);
      double w1 = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(FULL, b2 ? w2[0] : w2[1], 4);
      w1 += __shfl_xor_sync(FULL, w1, 2);
      w1 += __shfl_xor_sync(FULL, w1, 1);
      if (!(a & 3)) {
        const int p = a >> 2, c = b + 16 * p;
        sc.sv[b * 4 + p] = c > j ? tau * w1 : 0.0;
      }
      __syncwarp();
      const double2* s2 = reinterpret_cast<const double2*>(sc.sv + b * 4);
      const double2 s01 = s2[0], s23 = s2[1];
      const double s[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
      for (int k = T; k < 4; ++k)
#pragma unroll
        for (int i = T; i < 4; ++i) m[i][k] = fma(-uu[i], s[k], m[i][k]);
    }
    if (j + 1 >= cols) break;
    {
      double np = 0.0;
      if (a == jl) {
#pragma unroll
        for (int k = T; k < 4; ++k) {
          const int c = b + 16 * k;
          const double x = c > j ? m[T][k] : 0.0;
          sc.rowbuf[c] = x;
          np = fma(x, x, np);
        }
      }
      np += __shfl_xor_sync(FULL, np, 16);
      if (lane == jl) sc.nred[warp] = np;
    }
    __syncthreads();  // B
    {
      const double2* nr2 = reinterpret_cast<const double2*>(sc.nred);
      double sig2 = 0.0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const double2 x = nr2[w];
        sig2 += x.x;
        sig2 += x.y;
      }
      const QuickReflector h = quick_reflector(make_double2(sc.rowbuf[j + 1], 0.0), sig2);
      if (tid == 0) e2[2 * j + 1] = sig2;
      double uc[4];
#pragma unroll
      for (int k = T; k < 4; ++k) {
        const int c = b + 16 * k;
        uc[k] = c == j + 1 ? 1.0 : sc.rowbuf[c] * h.scale.x;
      }
      double v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double acc = 0.0;
        if (i >= T)
#pragma unroll
          for (int k = T; k < 4; ++k) acc = fma(m[i][k], uc[k], acc);
        v[i] = acc;
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const double r = (hb ? v[t + 2] : v[t]) + __shfl_xor_sync(FULL, hb ? v[t] : v[t + 2], 16);
        sc.wred[(warp * 4 + hb * 2 + t) * 16 + a] = r;
      }
      __syncthreads();  // C
      if (tid < 64) {
        const int ar = tid & 15, i = tid >> 4;
        double sum = 0.0;
        if (i >= T) {
#pragma unroll
          for (int w = 0; w < 8; ++w) sum += sc.wred[(w * 4 + i) * 16 + ar];
        }
        sc.wv[i * 16 + ar] = ar + 16 * i > j ? h.tau * sum : 0.0;
      }
      __syncthreads();  // D
#pragma unroll
      for (int i = T; i < 4; ++i) {
        const double w = sc.wv[i * 16 + a];
#pragma unroll
        for (int k = T; k < 4; ++k) m[i][k] = fma(-w, uc[k], m[i][k]);
      }
    }
  }
}

static __device__ void bidiag_tgk_reg_real(const double* Ms, int lm, int rows, int cols, double* diag, double* e2,
                                           double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane & 15, b = 2 * warp + (lane >> 4);
  GkRegScratchReal sc;
  sc.ubuf = scratch;
  sc.stau = scratch + 64;
  sc.sv = scratch + 66;
  sc.rowbuf = scratch + 130;
  sc.nred = scratch + 194;
  sc.wred = scratch + 202;
  sc.wv = scratch + 714;
  const int d = rows + cols;
  for (int i = tid; i < d; i += blockDim.x) {
    diag[i] = 0.0;
    e2[i] = 0.0;
  }
  double m[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = a + 16 * i, c = b + 16 * k;
      m[i][k] = (r < rows && c < cols) ? Ms[r + (size_t)c * lm] : 0.0;
    }
  gk_reg_phase_real<0>(m, rows, cols, e2, sc);
  if (cols > 16) gk_reg_phase_real<1>(m, rows, cols, e2, sc);
  if (cols > 32) gk_reg_phase_real<2>(m, rows, cols, e2, sc);
  if (cols > 48) gk_reg_phase_real<3>(m, rows, cols, e2, sc);
  __syncthreads();
}

// ------------------------------------------------------------------------------------------------
// Real variants (periodic gauge at a time-reversal-invariant k: C is exactly real, hx_capi k_is_real):
// the same schedules on doubles - a quarter of the FMAs and half the shared-memory traffic.
// Leading dimensions: CTA variant 8 (mod 16) doubles (the half-warp's two columns x 8 rows hit distinct
// banks), warp variant odd (lanes walking 16 columns at one row hit distinct banks).
__host__ __device__ constexpr int bidiag_ld_real(int S) { return (S + 8) / 16 * 16 + 8; }
__host__ __device__ constexpr int bidiag_ld_real_warp(int S) { return S | 1; }

static __device__ void bidiag_tgk_real(double* M, int lm, int rows, int cols, double* diag, double* e2, double* u,
                                       double* red) {
  const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = bd >> 5;
  const int d = rows + cols;
  for (int i = tid; i < d; i += bd) {
    diag[i] = 0.0;
    e2[i] = 0.0;
  }
  const int g = lane & 7, q = lane >> 3;
  double* lred = red;
  double* rred = red + 32;
  {
    double part = 0.0;
    for (int i = tid; i < rows; i += bd) part = fma(M[i], M[i], part);
    part = warp_sum(part);
    if (lane == 0) lred[warp] = part;
    __syncthreads();
  }
  for (int j = 0; j < cols; ++j) {
    {
      double sig2 = 0.0;
      for (int w = 0; w < nw; ++w) sig2 += lred[w];
      const double* colj = M + (size_t)j * lm;
      const QuickReflector h = quick_reflector(make_double2(colj[j], 0.0), sig2);
      if (tid == 0) e2[2 * j] = sig2;
      for (int i = j + tid; i < rows; i += bd) u[i] = i == j ? 1.0 : colj[i] * h.scale.x;
      __syncthreads();
      double rpart = 0.0;
      for (int c0 = j + 1; c0 < cols; c0 += bd >> 3) {
        const int cc = c0 + (tid >> 3);
        double acc = 0.0;
        if (cc < cols && h.tau != 0.0)
          for (int i = j + g; i < rows; i += 8) acc = fma(u[i], M[i + (size_t)cc * lm], acc);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double sc = h.tau * acc;
        if (cc < cols) {
          if (h.tau != 0.0)
            for (int i = j + g; i < rows; i += 8) {
              const double x = fma(-u[i], sc, M[i + (size_t)cc * lm]);
              M[i + (size_t)cc * lm] = x;
              if (i == j) rpart = fma(x, x, rpart);
            }
          else if (g == 0) {
            const double x = M[j + (size_t)cc * lm];
            rpart = fma(x, x, rpart);
          }
        }
      }
      rpart = warp_sum(rpart);
      if (lane == 0) rred[warp] = rpart;
      __syncthreads();
    }
    if (j + 1 >= cols) break;
    {
      double sig2 = 0.0;
      for (int w = 0; w < nw; ++w) sig2 += rred[w];
      const QuickReflector h = quick_reflector(make_double2(M[j + (size_t)(j + 1) * lm], 0.0), sig2);
      if (tid == 0) e2[2 * j + 1] = sig2;
      for (int cc = j + 1 + tid; cc < cols; cc += bd) u[cc] = cc == j + 1 ? 1.0 : M[j + (size_t)cc * lm] * h.scale.x;
      __syncthreads();
      double lpart = 0.0;
      for (int r0 = j + 1; r0 < rows; r0 += 8 * nw) {
        const int r = r0 + g + 8 * warp;
        double acc = 0.0;
        if (r < rows && h.tau != 0.0)
          for (int cc = j + 1 + q; cc < cols; cc += 4) acc = fma(M[r + (size_t)cc * lm], u[cc], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 8);
        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
        const double w = h.tau * acc;
        if (r < rows) {
          if (h.tau != 0.0)
            for (int cc = j + 1 + q; cc < cols; cc += 4) {
              const double x = fma(-w, u[cc], M[r + (size_t)cc * lm]);
              M[r + (size_t)cc * lm] = x;
              if (cc == j + 1) lpart = fma(x, x, lpart);
            }
          else if (q == 0) {
            const double x = M[r + (size_t)(j + 1) * lm];
            lpart = fma(x, x, lpart);
          }
        }
      }
      lpart = warp_sum(lpart);
      if (lane == 0) lred[warp] = lpart;
      __syncthreads();
    }
  }
  __syncthreads();
}

static __device__ void bidiag_tgk_warp_real(double* M, int lm, int rows, int cols, double* diag, double* e2,
                                            double* u) {
  const int lane = threadIdx.x & 31;
  const int d = rows + cols;
  for (int i = lane; i < d; i += 32) {
    diag[i] = 0.0;
    e2[i] = 0.0;
  }
  for (int j = 0; j < cols; ++j) {
    {
      const double* colj = M + (size_t)j * lm;
      double part = 0.0;
      for (int i = j + lane; i < rows; i += 32) part = fma(colj[i], colj[i], part);
      const double sig2 = warp_sum(part);
      const QuickReflector h = quick_reflector(make_double2(colj[j], 0.0), sig2);
      if (lane == 0) e2[2 * j] = sig2;
      for (int i = j + lane; i < rows; i += 32) u[i] = i == j ? 1.0 : colj[i] * h.scale.x;
      __syncwarp();
      if (h.tau != 0.0)
        for (int c0 = j + 1 + lane; c0 < cols; c0 += 64) {
          const bool has1 = c0 + 32 < cols;
          double* col0 = M + (size_t)c0 * lm;
          double* col1 = M + (size_t)(has1 ? c0 + 32 : c0) * lm;
          double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
          for (int i = j; i < rows; ++i) {
            const double v = u[i];
            a0 = fma(v, col0[i], a0);
            a1 = fma(v, col1[i], a1);
          }
          const double s0 = h.tau * a0, s1 = has1 ? h.tau * a1 : 0.0;
#pragma unroll 4
          for (int i = j; i < rows; ++i) {
            const double v = u[i];
            const double x0 = fma(-v, s0, col0[i]), x1 = fma(-v, s1, col1[i]);
            col0[i] = x0;
            if (has1) col1[i] = x1;
          }
        }
      __syncwarp();
    }
    if (j + 1 >= cols) break;
    {
      double part = 0.0;
      for (int cc = j + 1 + lane; cc < cols; cc += 32) {
        const double x = M[j + (size_t)cc * lm];
        part = fma(x, x, part);
      }
      const double sig2 = warp_sum(part);
      const QuickReflector h = quick_reflector(make_double2(M[j + (size_t)(j + 1) * lm], 0.0), sig2);
      if (lane == 0) e2[2 * j + 1] = sig2;
      for (int cc = j + 1 + lane; cc < cols; cc += 32) u[cc] = cc == j + 1 ? 1.0 : M[j + (size_t)cc * lm] * h.scale.x;
      __syncwarp();
      if (h.tau != 0.0)
        for (int r0 = j + 1 + lane; r0 < rows; r0 += 64) {
          const bool has1 = r0 + 32 < rows;
          const int r1 = has1 ? r0 + 32 : r0;
          double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
          for (int cc = j + 1; cc < cols; ++cc) {
            const double b = u[cc];
            a0 = fma(M[r0 + (size_t)cc * lm], b, a0);
            a1 = fma(M[r1 + (size_t)cc * lm], b, a1);
          }
          const double w0 = h.tau * a0, w1 = has1 ? h.tau * a1 : 0.0;
#pragma unroll 4
          for (int cc = j + 1; cc < cols; ++cc) {
            const double b = u[cc];
            const double x0 = fma(-w0, b, M[r0 + (size_t)cc * lm]), x1 = fma(-w1, b, M[r1 + (size_t)cc * lm]);
            M[r0 + (size_t)cc * lm] = x0;
            if (has1) M[r1 + (size_t)cc * lm] = x1;
          }
        }
      __syncwarp();
    }
  }
  __syncwarp();
}

}  // namespace hx
