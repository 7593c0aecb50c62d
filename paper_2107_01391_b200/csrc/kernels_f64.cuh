// kernels_f64.cuh — general float_to_decimal on the device.
//
// The reference (key_model.cpp:135-158) prints x with std::to_chars in the
// shortest fixed form that round-trips, parses that numeral (mantissa M =
// all its digits, F = fractional digits) and rescales it to `scale` places:
// M * 10^(scale-F) (an unchecked product, so it wraps modulo 2^64) or M /
// 10^(F-scale) rounded half up; 10^e with e > 19 and a mantissa above 2^64-1
// raise cell_budget_exceeded.  The fast mapper (MapF64 in kernels_grid.cuh)
// covers the common domain with a few floating-point tests; f2d_general is
// exact for every finite double:
//
//   x >= 2^53   integer valued; to_chars prints the exact integer, so M = x
//               (x >= 2^64: the mantissa overflows), F = 0.
//   0 < x < 2^53  with x = 4m * 2^-sh, the reals that round to x form
//               [L4, U4] * 2^-sh (ends included when m is even).  The
//               shortest numeral has the fewest fractional digits k for which
//               an integer N lies in [L4, U4] * 10^k / 2^sh; N is the one
//               nearest x * 10^k (ties to even).  Only k in
//               [max(kest, scale-19), min(scale+19, kest+20)] can give a
//               result (kest: a double log10 lower bound), plus one probe at
//               k = scale-20 that detects an overflowing 10^(scale-F).  Each
//               probe is V * 5^k (three 64-bit limbs) shifted by sh - k.
//
// tests/test_f64_general.py restates this with Python integers and pins it
// to the reference library on random doubles of every exponent.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rsb {

enum : uint32_t { kF2dOk = 0, kF2dNonFinite = 1, kF2dNegative = 2, kF2dDigits = 3, kF2dPow = 4 };
constexpr uint32_t kF2dMaxScale = 40;  // probes reach k = 59: V * 5^59 < 2^192

struct U192 {
  unsigned long long w[3];
};

__device__ __forceinline__ void u192_mul32(U192& a, uint32_t m) {
  unsigned long long carry = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    unsigned long long lo = a.w[i] * m;
    unsigned long long hi = __umul64hi(a.w[i], m);
    lo += carry;
    hi += lo < carry ? 1ull : 0ull;
    a.w[i] = lo;
    carry = hi;
  }
}

// v * 5^k, k <= 59, by factors 5^13 < 2^31
__device__ __forceinline__ U192 u192_mul_pow5(unsigned long long v, uint32_t k) {
  U192 a{{v, 0ull, 0ull}};
  while (k) {
    const uint32_t e = k < 13 ? k : 13;
    uint32_t m = 1;
    for (uint32_t i = 0; i < e; ++i) m *= 5u;
    u192_mul32(a, m);
    k -= e;
  }
  return a;
}

__device__ __forceinline__ unsigned long long u192_limb(const U192& a, int i) { return i < 3 ? a.w[i] : 0ull; }

// floor(a / 2^t) as a 128-bit (hi, lo) pair (callers guarantee it fits) and
// whether the division is exact; t <= 0 shifts left by -t (<= 63).
struct Q128 {
  unsigned long long lo, hi;
  bool exact;
};
__device__ __forceinline__ Q128 u192_shr(const U192& a, int t) {
  Q128 q{0ull, 0ull, true};
  if (t <= 0) {
    const int u = -t;
    q.lo = a.w[0] << u;
    q.hi = u ? (a.w[1] << u) | (a.w[0] >> (64 - u)) : a.w[1];
    return q;
  }
  if (t >= 192) {
    q.exact = (a.w[0] | a.w[1] | a.w[2]) == 0ull;
    return q;
  }
  const int w = t >> 6, b = t & 63;
  unsigned long long low = 0;  // the bits shifted out
  for (int i = 0; i < w; ++i) low |= a.w[i];
  if (b) {
    low |= a.w[w] & ((1ull << b) - 1ull);
    q.lo = (a.w[w] >> b) | (u192_limb(a, w + 1) << (64 - b));
    q.hi = (u192_limb(a, w + 1) >> b) | (u192_limb(a, w + 2) << (64 - b));
  } else {
    q.lo = a.w[w];
    q.hi = u192_limb(a, w + 1);
  }
  q.exact = low == 0ull;
  return q;
}

__device__ __forceinline__ bool q_le(unsigned long long ahi, unsigned long long alo, unsigned long long bhi,
                                     unsigned long long blo) {
  return ahi < bhi || (ahi == bhi && alo <= blo);
}

__device__ __forceinline__ unsigned long long f2d_pow10(uint32_t e) {
  unsigned long long p = 1;
  for (uint32_t i = 0; i < e; ++i) p *= 10ull;
  return p;
}

// DecimalValue{M, F} rescaled to `scale` places (key_model.cpp:150-157)
__device__ __forceinline__ unsigned long long f2d_finish(unsigned long long M, uint32_t F, uint32_t scale,
                                                         uint32_t& code) {
  if (F <= scale) {
    if (scale - F > 19) {
      code = kF2dPow;
      return 0;
    }
    return M * f2d_pow10(scale - F);  // wraps modulo 2^64, as the reference's unchecked product
  }
  const uint32_t d = F - scale;
  if (d > 19) {
    code = kF2dPow;
    return 0;
  }
  const unsigned long long p = f2d_pow10(d);
  return M / p + (M % p >= p / 2 ? 1ull : 0ull);
}

// float_to_decimal(x, scale) for any double; scale <= kF2dMaxScale.
__device__ __noinline__ unsigned long long f2d_general(double x, uint32_t scale, uint32_t& code) {
  code = kF2dOk;
  if (!isfinite(x)) {
    code = kF2dNonFinite;
    return 0;
  }
  if (x < 0.0) {
    code = kF2dNegative;
    return 0;
  }
  if (x == 0.0) return f2d_finish(0, 0, scale, code);
  if (x >= 9007199254740992.0) {  // 2^53: integer valued, printed exactly
    if (x >= 18446744073709551616.0) {
      code = kF2dDigits;
      return 0;
    }
    return f2d_finish(static_cast<unsigned long long>(x), 0, scale, code);
  }
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const uint32_t be = static_cast<uint32_t>(b >> 52) & 0x7ffu;
  const unsigned long long f = b & 0x000fffffffffffffull;
  const unsigned long long m = be == 0 ? f : (f | (1ull << 52));
  const int q = be == 0 ? -1074 : static_cast<int>(be) - 1075;
  const int sh = 2 - q;
  const unsigned long long X4 = 4 * m, U4 = 4 * m + 2, L4 = 4 * m - ((f == 0 && be > 1) ? 1 : 2);
  const bool incl = (m & 1ull) == 0;
  auto bounds = [&](uint32_t k, unsigned long long& lohi, unsigned long long& lolo, unsigned long long& hihi,
                    unsigned long long& hilo) {
    const Q128 a = u192_shr(u192_mul_pow5(L4, k), sh - static_cast<int>(k));
    unsigned long long add = a.exact ? 0ull : 1ull;  // ceil
    if (a.exact && !incl) add = 1;                   // an excluded end
    lolo = a.lo + add;
    lohi = a.hi + (lolo < a.lo ? 1ull : 0ull);
    const Q128 c = u192_shr(u192_mul_pow5(U4, k), sh - static_cast<int>(k));
    hilo = c.lo;
    hihi = c.hi;
    if (c.exact && !incl) {  // floor, minus an excluded end
      hihi -= hilo == 0 ? 1ull : 0ull;
      hilo -= 1ull;
    }
    return q_le(lohi, lolo, hihi, hilo);
  };
  const double lg = -log10(x);
  const int kest = lg > 1.0 ? static_cast<int>(floor(lg)) - 1 : 0;
  unsigned long long lohi, lolo, hihi, hilo;
  if (scale >= 20 && static_cast<int>(scale) - 20 >= kest && bounds(scale - 20, lohi, lolo, hihi, hilo)) {
    code = kF2dPow;  // a numeral with <= scale-20 fractional digits: 10^(scale-F) overflows
    return 0;
  }
  const int start = kest > static_cast<int>(scale) - 19 ? kest : static_cast<int>(scale) - 19;
  const int stop = static_cast<int>(scale) + 19 < kest + 20 ? static_cast<int>(scale) + 19 : kest + 20;
  int k = start < 0 ? 0 : start;
  for (; k <= stop; ++k)
    if (bounds(static_cast<uint32_t>(k), lohi, lolo, hihi, hilo)) break;
  if (k > stop) {
    code = kF2dPow;  // the shortest numeral has more than scale+19 fractional digits
    return 0;
  }
  unsigned long long N = lolo;
  if (lolo != hilo || lohi != hihi) {  // several candidates: the one nearest x * 10^k, ties to even
    const U192 a = u192_mul_pow5(X4, static_cast<uint32_t>(k));
    const int t = sh - k;
    if (t <= 0) {
      N = u192_shr(a, t).lo;
    } else {
      const Q128 qn = u192_shr(a, t);
      const Q128 q1 = u192_shr(a, t - 1);  // its low bit is the half bit
      const bool half_bit = (q1.lo & 1ull) != 0;
      const bool up = half_bit && (!q1.exact || (qn.lo & 1ull));
      N = qn.lo + (up ? 1ull : 0ull);
    }
  }
  return f2d_finish(N, static_cast<uint32_t>(k), scale, code);
}

}  // namespace rsb
