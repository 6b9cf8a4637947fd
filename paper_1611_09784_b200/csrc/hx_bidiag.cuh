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
static __device__ void assemble_bipartite(const CellDev& c, const int* idx_a, const int* idx_b, double2 k,
                                          double2* M, int lm, int rows, int cols, bool transpose) {
  for (int p = threadIdx.x; p < lm * cols; p += blockDim.x) M[p] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int r = threadIdx.x; r < c.N; r += blockDim.x) {
    const int ia = idx_a[r];
    if (ia < 0) continue;
    // partners of the A dof r: own targets, then sources pointing at r (distinct, kept, sublattice B)
    auto visit = [&](int cb) {
      const int jb = idx_b[cb];
      if (jb < 0) return;
      const double2 h = herm_element(c.h_ptr, c.h_col, c.h_amp, c.h_disp, r, cb, k);
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
  const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = bd >> 5;
  const int d = rows + cols;
  for (int i = tid; i < d; i += bd) {
    diag[i] = 0.0;
    e2[i] = 0.0;
  }
  for (int j = 0; j < cols; ++j) {
    // ---------------- left reflector: column j, rows j..rows-1
    {
      double part = 0.0;
      for (int i = j + tid; i < rows; i += bd) {
        const double2 x = M[i + (size_t)j * lm];
        part += x.x * x.x + x.y * x.y;
      }
      const double sig2 = block_sum(part, red);
      const double2 alpha = M[j + (size_t)j * lm];
      const Reflector h = make_reflector(alpha, sig2);
      if (tid == 0) e2[2 * j] = sig2;
      if (h.tau != 0.0) {
        for (int i = j + tid; i < rows; i += bd) u[i] = i == j ? make_double2(1.0, 0.0) : cmul(M[i + (size_t)j * lm], h.scale);
        __syncthreads();
        // s_c = v^H M[:, c] for c > j (warp per column, lanes over rows)
        for (int cc = j + 1 + warp; cc < cols; cc += nw) {
          double2 acc = make_double2(0.0, 0.0);
          for (int i = j + lane; i < rows; i += 32) {
            const double2 a = u[i], b = M[i + (size_t)cc * lm];
            acc.x += a.x * b.x + a.y * b.y;
            acc.y += a.x * b.y - a.y * b.x;
          }
          acc.x = warp_sum(acc.x);
          acc.y = warp_sum(acc.y);
          if (lane == 0) s[cc] = make_double2(h.tau * acc.x, h.tau * acc.y);
        }
        __syncthreads();
        // M[:, c] -= v s_c
        const int w = cols - j - 1, hgt = rows - j;
        for (int p = tid; p < w * hgt; p += bd) {
          const int cc = j + 1 + p / hgt, i = j + p % hgt;
          const double2 a = u[i], b = s[cc];
          double2 x = M[i + (size_t)cc * lm];
          x.x -= a.x * b.x - a.y * b.y;
          x.y -= a.x * b.y + a.y * b.x;
          M[i + (size_t)cc * lm] = x;
        }
        __syncthreads();
      }
    }
    if (j + 1 >= cols) break;
    // ---------------- right reflector: row j, columns j+1..cols-1 (on the conjugated row)
    {
      double part = 0.0;
      for (int cc = j + 1 + tid; cc < cols; cc += bd) {
        const double2 x = M[j + (size_t)cc * lm];
        part += x.x * x.x + x.y * x.y;
      }
      const double sig2 = block_sum(part, red);
      const double2 a0 = M[j + (size_t)(j + 1) * lm];
      const Reflector h = make_reflector(make_double2(a0.x, -a0.y), sig2);
      if (tid == 0) e2[2 * j + 1] = sig2;
      if (h.tau != 0.0) {
        // u_c from conj(row j): u_{j+1} = 1
        for (int cc = j + 1 + tid; cc < cols; cc += bd) {
          const double2 x = M[j + (size_t)cc * lm];
          u[cc] = cc == j + 1 ? make_double2(1.0, 0.0) : cmul(make_double2(x.x, -x.y), h.scale);
        }
        __syncthreads();
        // w_r = tau * sum_c M[r][c] u_c for rows r > j (thread per row)
        for (int r = j + 1 + tid; r < rows; r += bd) {
          double2 acc = make_double2(0.0, 0.0);
          for (int cc = j + 1; cc < cols; ++cc) {
            const double2 a = M[r + (size_t)cc * lm], b = u[cc];
            acc.x += a.x * b.x - a.y * b.y;
            acc.y += a.x * b.y + a.y * b.x;
          }
          s[r] = make_double2(h.tau * acc.x, h.tau * acc.y);
        }
        __syncthreads();
        // M[r][c] -= w_r conj(u_c)
        const int w = cols - j - 1, hgt = rows - j - 1;
        for (int p = tid; p < w * hgt; p += bd) {
          const int cc = j + 1 + p / hgt, r = j + 1 + p % hgt;
          const double2 a = s[r], b = u[cc];
          double2 x = M[r + (size_t)cc * lm];
          x.x -= a.x * b.x + a.y * b.y;
          x.y -= a.y * b.x - a.x * b.y;
          M[r + (size_t)cc * lm] = x;
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
}

}  // namespace hx
