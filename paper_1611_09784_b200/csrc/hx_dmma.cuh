// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) helpers for complex128 tiles on sm_100a.
//
// Fragment layouts of mma.sync.aligned.m8n8k4.row.col.f64 (lane = %laneid):
//   A (8x4, row):  a = A[lane >> 2][lane & 3]
//   B (4x8, col):  b = B[lane & 3][lane >> 2]
//   C (8x8):       c0 = C[lane >> 2][2*(lane & 3)], c1 = C[lane >> 2][2*(lane & 3) + 1]
// A complex product is four real DMMAs: Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br.
#pragma once
#include <cuda_runtime.h>

namespace hx {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Complex 8x8 accumulator tile: re[2], im[2] per lane.
struct CTile {
  double re0, re1, im0, im1;
  __device__ __forceinline__ void zero() { re0 = re1 = im0 = im1 = 0.0; }
  __device__ __forceinline__ void begin() {}
  __device__ __forceinline__ void end() {}
  // C += A * B for one k4 slice; (ar, ai) = A fragment element, (br, bi) = B fragment element.
  __device__ __forceinline__ void mac(double ar, double ai, double br, double bi) {
    dmma(re0, re1, ar, br);
    dmma(re0, re1, -ai, bi);
    dmma(im0, im1, ar, bi);
    dmma(im0, im1, ai, br);
  }
};

// The same tile with the 3-multiplication (Karatsuba / "3M") complex product: with P1 = sum ar br,
// P2 = sum ai bi and P3 = sum (ar + ai)(br + bi), re = P1 - P2 and im = P3 - P1 - P2 - three real DMMAs per
// fragment product instead of four, for the DMMA-issue-bound products (xv_kernel of the complex tiers) that
// have the registers for the third accumulator.  Between begin() and end() the fields hold re = C_re + P1,
// t = P2, im = C_im + C_re + P3; outside they are (re, im).  The imaginary part's rounding error scales with
// (|ar| + |ai|)(|br| + |bi|) instead of |ar bi| + |ai br| - a few ulps of |C|, far inside the 1e-10 eigenvalue
// tolerance.
struct CTile3 {
  double re0, re1, im0, im1, t0, t1;
  __device__ __forceinline__ void zero() { re0 = re1 = im0 = im1 = t0 = t1 = 0.0; }
  __device__ __forceinline__ void begin() {
    im0 += re0;
    im1 += re1;
    t0 = t1 = 0.0;
  }
  __device__ __forceinline__ void end() {
    im0 = (im0 - re0) - t0;
    im1 = (im1 - re1) - t1;
    re0 -= t0;
    re1 -= t1;
  }
  __device__ __forceinline__ void mac(double ar, double ai, double br, double bi) {
    dmma(re0, re1, ar, br);
    dmma(t0, t1, ai, bi);
    dmma(im0, im1, ar + ai, br + bi);
  }
};

// C += A * B on real data (RE: every imaginary part is exactly zero, so only the real-real product is
// issued - one DMMA instead of four; the tile stays in (re, im) form, no begin/end); otherwise the tile's
// complex product (inside begin() / end()).
template <bool RE, typename Tile>
__device__ __forceinline__ void cmac(Tile& t, double ar, double ai, double br, double bi) {
  if constexpr (RE) dmma(t.re0, t.re1, ar, br);
  else t.mac(ar, ai, br, bi);
}
template <bool RE, typename Tile>
__device__ __forceinline__ void cbegin(Tile& t) {
  if constexpr (!RE) t.begin();
}
template <bool RE, typename Tile>
__device__ __forceinline__ void cend(Tile& t) {
  if constexpr (!RE) t.end();
}

}  // namespace hx
