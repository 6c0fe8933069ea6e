// Python's format(x, ".17g") for IEEE doubles, exactly (the reference's
// 17-significant-digit text writer, pkg/src/impact/fileio.py:36-41, used by
// save_matrix / save_vector / save_controller :94-101, :118-123, :192-215).
//
// Correct rounding: x = M * 2^E is exact, so D = round_half_even(x / 10^K)
// with K = floor(log10 x) - 16 is computed with exact multi-limb integers
// (x < 10^17: N = M * 10^-K, then a rounded right shift by -E; x >= 10^17:
// (M << E) / 10^K by repeated limb division with a sticky remainder).  If D
// leaves [10^16, 10^17) the decimal exponent estimate was off by one and D
// is recomputed exactly (never rounded twice).  Layout follows CPython's
// 'g': scientific when the exponent is < -4 or >= 17, trailing zeros and a
// bare decimal point stripped, exponent with sign and at least two digits;
// 0 -> "0", -0 -> "-0", inf -> "inf", nan -> "nan".
//
// Portable C++: the device export kernels (export.cu) and the host tests
// (checked against Python's own format on random and edge-case doubles)
// compile the same source.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define IMP_FMT_HD __host__ __device__ __forceinline__
#else
#define IMP_FMT_HD static inline
#endif

#define IMP_FMT17_MAX 25   // "-1.2345678901234567e-308" is 24 chars

struct ImpBig {   // little-endian base-2^32 unsigned integer
  uint32_t w[40];
  int n;
};

IMP_FMT_HD void imp_big_set(ImpBig& b, uint64_t v) {
  b.w[0] = (uint32_t)v;
  b.w[1] = (uint32_t)(v >> 32);
  b.n = b.w[1] ? 2 : (b.w[0] ? 1 : 0);
}

IMP_FMT_HD void imp_big_mul_small(ImpBig& b, uint32_t m) {
  uint64_t carry = 0;
  for (int i = 0; i < b.n; ++i) {
    const uint64_t p = (uint64_t)b.w[i] * m + carry;
    b.w[i] = (uint32_t)p;
    carry = p >> 32;
  }
  if (carry) b.w[b.n++] = (uint32_t)carry;
}

IMP_FMT_HD void imp_big_mul_pow10(ImpBig& b, int k) {
  while (k >= 9) { imp_big_mul_small(b, 1000000000u); k -= 9; }
  uint32_t m = 1;
  while (k-- > 0) m *= 10;
  if (m > 1) imp_big_mul_small(b, m);
}

IMP_FMT_HD void imp_big_shl(ImpBig& b, int s) {
  const int limbs = s >> 5, bits = s & 31;
  if (b.n == 0) return;
  int n = b.n + limbs + 1;
  for (int i = n - 1; i >= 0; --i) {
    const int src = i - limbs;
    uint32_t hi = (src >= 0 && src < b.n) ? b.w[src] : 0;
    uint32_t lo = (src - 1 >= 0 && src - 1 < b.n) ? b.w[src - 1] : 0;
    b.w[i] = bits ? (hi << bits) | (lo >> (32 - bits)) : hi;
  }
  while (n > 0 && b.w[n - 1] == 0) --n;
  b.n = n;
}

// b = floor(b / d), returns the remainder
IMP_FMT_HD uint32_t imp_big_div_small(ImpBig& b, uint32_t d) {
  uint64_t r = 0;
  for (int i = b.n - 1; i >= 0; --i) {
    const uint64_t cur = (r << 32) | b.w[i];
    b.w[i] = (uint32_t)(cur / d);
    r = cur % d;
  }
  while (b.n > 0 && b.w[b.n - 1] == 0) --b.n;
  return (uint32_t)r;
}

IMP_FMT_HD int imp_big_bit(const ImpBig& b, int i) {
  const int limb = i >> 5;
  return limb < b.n ? (int)((b.w[limb] >> (i & 31)) & 1u) : 0;
}

IMP_FMT_HD uint64_t imp_big_low64(const ImpBig& b) {
  return (b.n > 0 ? b.w[0] : 0) | ((uint64_t)(b.n > 1 ? b.w[1] : 0) << 32);
}

// D = round_half_even(M * 2^E / 10^K), D < 2^64 assumed by the caller's K.
IMP_FMT_HD uint64_t imp_fmt_scaled(uint64_t M, int E, int K) {
  ImpBig b;
  imp_big_set(b, M);
  if (K <= 0) {
    imp_big_mul_pow10(b, -K);
    if (E >= 0) {
      imp_big_shl(b, E);
      return imp_big_low64(b);
    }
    const int s = -E;
    // quotient = b >> s; round half to even on the shifted-out bits
    const int half = imp_big_bit(b, s - 1);
    int sticky = 0;   // any of bits [0, s - 1) set
    const int full = (s - 1) >> 5, rem = (s - 1) & 31;
    for (int i = 0; i < full && i < b.n; ++i) sticky |= b.w[i] != 0;
    if (rem && full < b.n) sticky |= (b.w[full] & ((1u << rem) - 1u)) != 0;
    uint64_t q = 0;
    for (int i = 0; i < 64; ++i)
      q |= (uint64_t)imp_big_bit(b, s + i) << i;
    if (half && (sticky || (q & 1))) ++q;
    return q;
  }
  // K > 0 (x >= 10^16, so E >= 0): (M << E) / 10^K
  if (E > 0) imp_big_shl(b, E);
  int k = K, sticky = 0;
  uint32_t r = 0, d = 1;
  while (k > 0) {
    const int step = k >= 9 ? 9 : k;
    d = 1;
    for (int i = 0; i < step; ++i) d *= 10;
    if (r) sticky = 1;   // remainders of earlier (lower) divisions
    r = imp_big_div_small(b, d);
    k -= step;
  }
  uint64_t q = imp_big_low64(b);
  // remainder R = r * (earlier divisors) + lower; half = d/2 * (earlier)
  const uint32_t h = d / 2;   // d is a power of ten >= 10: even
  if (r > h || (r == h && (sticky || (q & 1)))) ++q;
  return q;
}

// Writes format(x, ".17g") to out (no terminator), returns the length.
IMP_FMT_HD int imp_fmt17(double x, char* out) {
  uint64_t u;
#if defined(__CUDA_ARCH__)
  u = (uint64_t)__double_as_longlong(x);
#else
  __builtin_memcpy(&u, &x, 8);
#endif
  int len = 0;
  const int neg = (int)(u >> 63);
  const int bexp = (int)((u >> 52) & 0x7ff);
  uint64_t frac = u & 0xfffffffffffffull;
  if (bexp == 0x7ff) {
    if (frac) { out[0] = 'n'; out[1] = 'a'; out[2] = 'n'; return 3; }
    if (neg) out[len++] = '-';
    out[len++] = 'i'; out[len++] = 'n'; out[len++] = 'f';
    return len;
  }
  if (neg) out[len++] = '-';
  if (bexp == 0 && frac == 0) { out[len++] = '0'; return len; }
  uint64_t M;
  int E;
  if (bexp == 0) { M = frac; E = -1074; }
  else { M = frac | (1ull << 52); E = bexp - 1075; }
  // floor(log10 x) estimate from the binary exponent (exact or one low)
#if defined(__CUDA_ARCH__)
  const int bl = 63 - __clzll((long long)M);
#else
  const int bl = 63 - __builtin_clzll(M);   // x in [2^(E+bl), 2^(E+bl+1))
#endif
  const int e2 = E + bl;
  // 78913 / 2^18 ~ log10(2) (floor exact for |e2| <= 1650)
  int e10 = (e2 >= 0) ? (int)(((int64_t)e2 * 78913) >> 18)
                      : -(int)(((int64_t)(-e2) * 78913 + (1 << 18) - 1) >> 18);
  const uint64_t lo17 = 10000000000000000ull, hi17 = 100000000000000000ull;
  uint64_t D = imp_fmt_scaled(M, E, e10 - 16);
  for (int guard = 0; guard < 3 && (D >= hi17 || D < lo17); ++guard) {
    e10 += D >= hi17 ? 1 : -1;
    D = imp_fmt_scaled(M, E, e10 - 16);
  }
  char dig[17];
  for (int i = 16; i >= 0; --i) { dig[i] = (char)('0' + D % 10); D /= 10; }
  int nd = 17;
  while (nd > 1 && dig[nd - 1] == '0') --nd;
  if (e10 < -4 || e10 >= 17) {
    out[len++] = dig[0];
    if (nd > 1) {
      out[len++] = '.';
      for (int i = 1; i < nd; ++i) out[len++] = dig[i];
    }
    out[len++] = 'e';
    int ae = e10;
    out[len++] = ae < 0 ? '-' : '+';
    if (ae < 0) ae = -ae;
    if (ae >= 100) out[len++] = (char)('0' + ae / 100);
    out[len++] = (char)('0' + (ae / 10) % 10);
    out[len++] = (char)('0' + ae % 10);
  } else if (e10 >= 0) {
    for (int i = 0; i <= e10; ++i) out[len++] = i < nd ? dig[i] : '0';
    if (nd > e10 + 1) {
      out[len++] = '.';
      for (int i = e10 + 1; i < nd; ++i) out[len++] = dig[i];
    }
  } else {
    out[len++] = '0';
    out[len++] = '.';
    for (int i = 0; i < -e10 - 1; ++i) out[len++] = '0';
    for (int i = 0; i < nd; ++i) out[len++] = dig[i];
  }
  return len;
}
