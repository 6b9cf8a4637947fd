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

#include "../../include/hx.h"

namespace hx {

constexpr int FX_NL = HX_FX_LIMBS;
constexpr int FX_FRAC = HX_FX_FRAC;

// Adds v (exactly, truncated toward zero below 2^-FX_FRAC) to the limb accumulator L.  Returns false for
// non-finite or out-of-range values (|v| >= 2^(32*FX_NL - FX_FRAC - 1)), which are not added.
__host__ __device__ inline bool fx_add(int64_t* L, double v) {
  if (v == 0.0) return true;
  if (!(fabs(v) < 1e300)) return false;
  int e;
  const double m = frexp(fabs(v), &e);               // |v| = m 2^e, m in [0.5, 1)
  uint64_t mant = (uint64_t)ldexp(m, 53);            // exact: |v| = mant 2^(e - 53)
  int sh = e - 53 + FX_FRAC;                         // fixed-point bit position of mant's lowest bit
  if (sh + 53 > 32 * FX_NL - 1) return false;
  if (sh < 0) {
    if (sh <= -53) return true;                      // below the resolution: contributes 0
    mant >>= -sh;
    sh = 0;
  }
  const int li = sh >> 5, off = sh & 31;
  const uint64_t lo = mant << off;                   // bits [off, off + 64) of mant << off
  const uint64_t hi = off ? (mant >> (64 - off)) : 0;
  const int64_t s = v < 0.0 ? -1 : 1;
  L[li] += s * (int64_t)(lo & 0xffffffffull);
  if (li + 1 < FX_NL) L[li + 1] += s * (int64_t)(lo >> 32);
  if (li + 2 < FX_NL) L[li + 2] += s * (int64_t)hi;
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
