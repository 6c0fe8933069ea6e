// numpy's random streams, restated for the device (and the host tests):
// the reference's per-rollout generator (pkg/src/impact/noise.py:121-131:
// derive_seed = SeedSequence(entropy, spawn_key=(row, dest)).generate_state,
// mc_generator = Generator(Philox(SeedSequence(seed)))) and
// Generator.normal (cli.py:163-166), bit for bit.
//
//   SeedSequence   numpy/random/bit_generator.pyx (pool 4, hashmix / mix of
//                  M. O'Neill's seed_seq_fe): entropy and spawn key as
//                  little-endian 32-bit words, run entropy padded to the pool
//                  when a spawn key is present
//   Philox4x64-10  Random123 round function and Weyl key schedule; numpy's
//                  first block uses counter 1 (the counter is incremented
//                  before each block), outputs v0..v3 in order
//   normal         random_standard_normal (numpy distributions.c): 256-strip
//                  ziggurat on one uint64 (8-bit strip, sign bit, 52-bit
//                  magnitude), tail and wedge with glibc log1p / exp
//   log1p          glibc 2.39 x86-64 (fdlibm s_log1p.c, Estrin polynomial,
//                  FMA contractions exactly as that build fuses them)
//
// Checked against numpy itself on millions of draws (tests/test_simulate.py,
// tools/gen_ziggurat.py for the tables).  Needs ndtr.h (imp_exp) first.
#pragma once

#include "ziggurat_tables.h"

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define IMP_RHD __host__ __device__ __forceinline__
#else
#define IMP_RHD static inline
#include <math.h>
#endif

// --- SeedSequence ------------------------------------------------------------

IMP_RHD unsigned imp_ss_hashmix(unsigned v, unsigned* hc) {
  v ^= *hc;
  *hc *= 0x931e8875u;
  v *= *hc;
  v ^= v >> 16;
  return v;
}

IMP_RHD unsigned imp_ss_mix(unsigned x, unsigned y) {
  unsigned r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}

// little-endian 32-bit words of a non-negative integer (at least one word)
IMP_RHD int imp_ss_words(unsigned long long v, unsigned* out) {
  int n = 0;
  do {
    out[n++] = (unsigned)(v & 0xffffffffull);
    v >>= 32;
  } while (v);
  return n;
}

// SeedSequence(entropy, spawn_key=key[0..nkey)).generate_state(n64, uint64)
IMP_RHD void imp_seedseq(unsigned long long entropy,
                         const unsigned long long* key, int nkey,
                         unsigned long long* out, int n64) {
  unsigned ent[2 + 4 + 2 * 4];
  int n = imp_ss_words(entropy, ent);
  if (nkey > 0)
    while (n < 4) ent[n++] = 0u;
  for (int q = 0; q < nkey; ++q) n += imp_ss_words(key[q], ent + n);
  unsigned hc = 0x43b0d7e5u;
  unsigned mixer[4];
  for (int i = 0; i < 4; ++i) mixer[i] = imp_ss_hashmix(i < n ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) mixer[d] = imp_ss_mix(mixer[d], imp_ss_hashmix(mixer[s], &hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d)
      mixer[d] = imp_ss_mix(mixer[d], imp_ss_hashmix(ent[s], &hc));
  unsigned hb = 0x8b51f9ddu;
  for (int i = 0; i < 2 * n64; ++i) {
    unsigned v = mixer[i % 4];
    v ^= hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    if (i & 1) out[i >> 1] |= (unsigned long long)v << 32;
    else out[i >> 1] = v;
  }
}

// --- Philox4x64-10 -------------------------------------------------------------

struct ImpPhilox {
  unsigned long long ctr[4], key[2], buf[4];
  int pos;
};

IMP_RHD void imp_mulhilo64(unsigned long long a, unsigned long long b,
                           unsigned long long* hi, unsigned long long* lo) {
#if defined(__CUDA_ARCH__)
  *hi = __umul64hi(a, b);
  *lo = a * b;
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  *hi = (unsigned long long)(p >> 64);
  *lo = (unsigned long long)p;
#endif
}

IMP_RHD void imp_philox_block(const unsigned long long* ctr_in,
                              const unsigned long long* key_in,
                              unsigned long long* out) {
  unsigned long long c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2],
                     c3 = ctr_in[3], k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    unsigned long long hi0, lo0, hi1, lo1;
    imp_mulhilo64(0xD2E7470EE14C6C93ull, c0, &hi0, &lo0);
    imp_mulhilo64(0xCA5A826395121157ull, c2, &hi1, &lo1);
    const unsigned long long n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Generator(Philox(SeedSequence(seed))): key = generate_state(2), counter 0
IMP_RHD void imp_philox_seed(ImpPhilox* g, unsigned long long seed) {
  imp_seedseq(seed, nullptr, 0, g->key, 2);
  g->ctr[0] = g->ctr[1] = g->ctr[2] = g->ctr[3] = 0ull;
  g->pos = 4;
}

IMP_RHD unsigned long long imp_philox_next(ImpPhilox* g) {
  if (g->pos < 4) return g->buf[g->pos++];
  for (int i = 0; i < 4; ++i)
    if (++g->ctr[i] != 0ull) break;
  imp_philox_block(g->ctr, g->key, g->buf);
  g->pos = 1;
  return g->buf[0];
}

IMP_RHD double imp_philox_double(ImpPhilox* g) {
  return (double)(imp_philox_next(g) >> 11) * (1.0 / 9007199254740992.0);
}

// --- glibc log1p ------------------------------------------------------------------

IMP_RHD double imp_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const unsigned long long ux = imp_asu(x);
  const int hx = (int)(ux >> 32);
  const int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0, u;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) {
      if (x == -1.0) return -imp_asd(0x7ff0000000000000ull);
      return (x - x) / (x - x);
    }
    if (ax < 0x3e200000) {
      if (two54 + x > 0.0 && ax < 0x3c900000) return x;
      return fma(-(x * x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = (int)(imp_asu(u) >> 32);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = (int)(imp_asu(u) >> 32);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    const unsigned long long lo = imp_asu(u) & 0xffffffffull;
    if (hu < 0x6a09e) {
      u = imp_asd(((unsigned long long)(unsigned)(hu | 0x3ff00000) << 32) | lo);
    } else {
      k += 1;
      u = imp_asd(((unsigned long long)(unsigned)(hu | 0x3fe00000) << 32) | lo);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = 0.5 * f * f;
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma(dk, ln2_lo, c);
      return fma(dk, ln2_hi, c);
    }
    const double R = hfsq * fma(-f, 0.66666666666666666, 1.0);
    if (k == 0) return f - R;
    return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R4 = fma(z, Lp7, Lp6), z2 = z * z, R2 = fma(z, Lp3, Lp2),
               R3 = fma(z, Lp5, Lp4), z4 = z2 * z2, z6 = z2 * z4;
  const double R = fma(R4, z6, fma(z4, R3, fma(z, Lp1, z2 * R2)));
  const double q = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - q);
  const double t = fma(dk, ln2_lo, c) + q;
  return fma(dk, ln2_hi, -((hfsq - t) - f));
}

// --- Generator.standard_normal ---------------------------------------------------

IMP_RHD double imp_std_normal(ImpPhilox* g) {
  const double zig_r = 3.6541528853610087963519472518;
  const double zig_inv_r = 0.27366123732975827203338247596;
  for (;;) {
    unsigned long long r = imp_philox_next(g);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * imp_asd(imp_zig_wi[idx]);
    if (sign) x = -x;
    if (rabs < imp_zig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -zig_inv_r * imp_log1p(-imp_philox_double(g));
        const double yy = -imp_log1p(-imp_philox_double(g));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 1) ? -(zig_r + xx) : zig_r + xx;
      }
    } else {
      const double fi0 = imp_asd(imp_zig_fi[idx - 1]),
                   fi1 = imp_asd(imp_zig_fi[idx]);
      if ((fi0 - fi1) * imp_philox_double(g) + fi1 < imp_exp(-0.5 * x * x))
        return x;
    }
  }
}
