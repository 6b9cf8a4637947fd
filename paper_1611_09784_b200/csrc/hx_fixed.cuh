// Exact, order-independent sums of doubles for the MLMC level moments (host + device).
//
// The reference's level mean / variance (mlmc.py:143-154: np.mean, np.var(ddof=1) over the level's sample
// axis) are float sums whose rounding depends on the summation order, so a sum split over devices or ranks
// differs in the last bits from the single-device one.  Here every term is converted on its own to a
// fixed-point integer (HX_FX_LIMBS signed 32-bit limbs held in int64, HX_FX_FRAC fraction bits, magnitude
// truncated below 2^-HX_FX_FRAC) and the limbs are summed as integers: the sum is associative, so per-device
// partial limbs can be added in any order (an int64 all-reduce) and the result is bitwise the same for 1, 2,
// 4 or 8 devices and any batch split.  Limb sums stay exact up to 2^31 terms per grid point.
#pragma once
#include <stdint.h>
#include <math.h>
#include <string.h>

#include "../../include/hx.h"

namespace hx {

constexpr int FX_NL = HX_FX_LIMBS;
constexpr int FX_FRAC = HX_FX_FRAC;

// Adds v (exactly, truncated toward zero below 2^-FX_FRAC) to the limb accumulator L.  Returns false for
// non-finite or out-of-range values (|v| >= 2^(32*FX_NL - FX_FRAC - 1)), which are not added.
__host__ __device__ inline bool fx_add(int64_t* L, double v) {
  uint64_t bits;
#ifdef __CUDA_ARCH__
  bits = (uint64_t)__double_as_longlong(v);
#else
  memcpy(&bits, &v, 8);
#endif
  int e = (int)((bits >> 52) & 0x7ff);
  if (e == 0x7ff) return false;                       // inf / nan
  uint64_t mant = bits & 0xFFFFFFFFFFFFFull;
  if (e) mant |= 1ull << 52;                          // normal: |v| = mant 2^(e - 1075)
  else e = 1;                                         // subnormal: |v| = mant 2^(1 - 1075)
  if (mant == 0) return true;
  int sh = e - 1075 + FX_FRAC;                        // fixed-point bit position of mant's lowest bit
  if (sh + 53 > 32 * FX_NL - 1) return false;
  if (sh < 0) {
    if (sh <= -53) return true;                       // below the resolution: contributes 0
    mant >>= -sh;
    sh = 0;
  }
  const int li = sh >> 5, off = sh & 31;
  const uint64_t lo = mant << off;                    // bits [off, off + 64) of mant << off
  const uint64_t hi = off ? (mant >> (64 - off)) : 0;
  const int64_t sgn = (bits >> 63) ? -1 : 1;
  const int64_t p0 = sgn * (int64_t)(lo & 0xffffffffull), p1 = sgn * (int64_t)(lo >> 32), p2 = sgn * (int64_t)hi;
  // static limb indices (the accumulator stays in registers)
#pragma unroll
  for (int j = 0; j < FX_NL; ++j) L[j] += (j == li ? p0 : 0) + (j == li + 1 ? p1 : 0) + (j == li + 2 ? p2 : 0);
  return true;
}

// Carry-normalised value of a limb sum as a double (deterministic function of the exact integer).
__host__ __device__ inline double fx_to_double(const int64_t* Lin) {
  int64_t L[FX_NL];
  for (int i = 0; i < FX_NL; ++i) L[i] = Lin[i];
  for (int i = 0; i + 1 < FX_NL; ++i) {
    const int64_t c = L[i] >> 32;  // arithmetic shift: floor(L / 2^32)
    L[i] -= c * 4294967296ll;
    L[i + 1] += c;
  }
  double d = (double)L[FX_NL - 1];
  for (int i = FX_NL - 2; i >= 0; --i) d = d * 4294967296.0 + (double)L[i];
  return ldexp(d, -FX_FRAC);
}

}  // namespace hx
