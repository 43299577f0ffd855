/*
 * CPU ORACLE -- test infrastructure only.  Never linked into the product.
 *
 * Plain-C restatement of the random-number arithmetic the reference relies
 * on.  The reference builds every stream as
 *     numpy.random.Generator(numpy.random.Philox(key=blake2b(...)))
 * (sm/core.py:119-126) and draws with `integers` (sm/core.py:128-129),
 * `normal` (:131-132), `uniform` (:134-135) and `poisson` (:137-138).  That
 * arithmetic lives in the third-party dependency numpy, pinned at 2.3.5,
 * which is not part of /root/reference; restated here from numpy's published
 * algorithms:
 *   - Philox4x64-10 (Random123, as vendored by numpy/random/src/philox):
 *     counter pre-incremented before each 4-word block, key bumped by the
 *     Weyl constants between rounds;
 *   - next_uint32: low half of a 64-bit word first, high half buffered
 *     (`has_uint32`), the buffer persisting across calls;
 *   - next_double: (w >> 11) * 2^-53;
 *   - integers(lo, hi) for hi-lo <= 2^32: 32-bit Lemire with the rejection
 *     threshold (2^32 - ex) % ex; hi-lo == 1 consumes nothing;
 *   - standard normal: 256-layer ziggurat on next_uint64 with the tables
 *     lifted from libnpyrandom.a (tools/extract_ziggurat.py);
 *   - poisson(lam < 10): multiplication method on next_double.
 * Pinned against numpy itself by tests/test_oracle_rng.py and against the
 * committed golden vectors in tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ziggurat_tables.h"

#define PHILOX_M0 0xD2E7470EE14C6C93ULL
#define PHILOX_M1 0xCA5A826395121157ULL
#define PHILOX_W0 0x9E3779B97F4A7C15ULL
#define PHILOX_W1 0xBB67AE8584CAA73BULL

typedef struct {
  uint64_t k0, k1;
  uint64_t ctr;     /* number of 4-word blocks produced so far */
  int pos;          /* next word inside buf (4 = empty) */
  uint64_t buf[4];
  int has32;        /* a buffered high half is pending */
  uint32_t u32;
} orc_stream;

static inline void mulhilo(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
}

/* One Philox4x64-10 block for counter value `block` (>= 1; the stream's
 * first block has counter 1 because numpy increments before generating). */
void orc_philox_block(uint64_t block, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = block, c1 = 0, c2 = 0, c3 = 0;
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo(PHILOX_M0, c0, &hi0, &lo0);
    mulhilo(PHILOX_M1, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void orc_init(orc_stream *s, uint64_t k0, uint64_t k1) {
  memset(s, 0, sizeof(*s));
  s->k0 = k0; s->k1 = k1; s->pos = 4;
}

uint64_t orc_next64(orc_stream *s) {
  if (s->pos >= 4) {
    s->ctr += 1;
    orc_philox_block(s->ctr, s->k0, s->k1, s->buf);
    s->pos = 0;
  }
  return s->buf[s->pos++];
}

uint32_t orc_next32(orc_stream *s) {
  if (s->has32) { s->has32 = 0; return s->u32; }
  uint64_t w = orc_next64(s);
  s->has32 = 1;
  s->u32 = (uint32_t)(w >> 32);
  return (uint32_t)w;
}

double orc_next_double(orc_stream *s) {
  return (double)(orc_next64(s) >> 11) * (1.0 / 9007199254740992.0);
}

/* Words consumed so far (64-bit units), and the u32 cursor (32-bit units). */
uint64_t orc_words_used(const orc_stream *s) { return s->ctr * 4 - (uint64_t)(4 - s->pos); }
uint64_t orc_u32_used(const orc_stream *s) { return orc_words_used(s) * 2 - (s->has32 ? 1 : 0); }

/* integers(lo, lo+ex) with 1 <= ex <= 2^32, int64 output. */
int orc_integers(orc_stream *s, int64_t lo, uint64_t ex, int64_t n, int64_t *out) {
  if (ex == 0 || ex > (1ULL << 32)) return -1;
  if (ex == 1) { for (int64_t i = 0; i < n; ++i) out[i] = lo; return 0; }
  if (ex == (1ULL << 32)) { for (int64_t i = 0; i < n; ++i) out[i] = lo + (int64_t)orc_next32(s); return 0; }
  const uint32_t exc = (uint32_t)ex;
  const uint32_t threshold = (uint32_t)((0x100000000ULL - ex) % ex);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t m = (uint64_t)orc_next32(s) * exc;
    uint32_t left = (uint32_t)m;
    if (left < exc) {
      while (left < threshold) {
        m = (uint64_t)orc_next32(s) * exc;
        left = (uint32_t)m;
      }
    }
    out[i] = lo + (int64_t)(m >> 32);
  }
  return 0;
}

/* numpy random_bounded_uint64(off=0, rng, mask=0, use_masked=false) for
 * rng < 2^32: value in [0, rng], Lemire on next_uint32 (rng == 0 consumes
 * nothing).  Used by Generator.choice(replace=False) and its shuffles. */
static uint64_t bounded_incl(orc_stream *s, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFULL) return orc_next32(s);
  int64_t v;
  orc_integers(s, 0, rng + 1, 1, &v);
  return (uint64_t)v;
}

/* numpy 2.3.5 Generator.choice(n, size=k, replace=False, shuffle=True),
 * p=None, integer population (verified against numpy in
 * tests/test_oracle_rng.py): for n > 10000 and k > n // 50 a tail
 * Fisher-Yates of arange(n) keeping the last k; otherwise Floyd's algorithm
 * (values j or j's draw, first sighting wins) followed by a Fisher-Yates
 * shuffle of the k picks.  All index draws are bounded_incl. */
int orc_choice(orc_stream *s, int64_t n, int64_t k, int64_t *out) {
  if (k < 0 || k > n) return -1;
  if (k == 0) return 0;
  if (n > 10000 && k > n / 50) {
    int64_t *data = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    if (!data) return -2;
    for (int64_t i = 0; i < n; ++i) data[i] = i;
    const int64_t first = n - k > 1 ? n - k : 1;
    for (int64_t i = n - 1; i >= first; --i) {
      const int64_t j = (int64_t)bounded_incl(s, (uint64_t)i);
      const int64_t t = data[j]; data[j] = data[i]; data[i] = t;
    }
    memcpy(out, data + (n - k), sizeof(int64_t) * (size_t)k);
    free(data);
    return 0;
  }
  uint64_t set_size = (uint64_t)(1.2 * (double)k), mask = set_size;
  for (int sh = 1; sh < 64; sh <<= 1) mask |= mask >> sh;
  set_size = mask + 1;
  uint64_t *hs = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)set_size);
  if (!hs) return -2;
  for (uint64_t i = 0; i < set_size; ++i) hs[i] = ~0ULL;
  for (int64_t j = n - k; j < n; ++j) {
    const uint64_t val = bounded_incl(s, (uint64_t)j);
    uint64_t loc = val & mask;
    while (hs[loc] != ~0ULL && hs[loc] != val) loc = (loc + 1) & mask;
    if (hs[loc] == ~0ULL) {
      hs[loc] = val;
      out[j - n + k] = (int64_t)val;
    } else {
      loc = (uint64_t)j & mask;
      while (hs[loc] != ~0ULL) loc = (loc + 1) & mask;
      hs[loc] = (uint64_t)j;
      out[j - n + k] = j;
    }
  }
  free(hs);
  for (int64_t i = k - 1; i >= 1; --i) {
    const int64_t j = (int64_t)bounded_incl(s, (uint64_t)i);
    const int64_t t = out[j]; out[j] = out[i]; out[i] = t;
  }
  return 0;
}

static inline double bits2d(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }

double orc_standard_normal(orc_stream *s) {
  for (;;) {
    uint64_t r = orc_next64(s);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * bits2d(ZIG_WI_DOUBLE_BITS[idx]);
    if (sign) x = -x;
    if (rabs < ZIG_KI_DOUBLE_BITS[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -ZIG_NOR_INV_R * log1p(-orc_next_double(s));
        double yy = -log1p(-orc_next_double(s));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 1) ? -(ZIG_NOR_R + xx) : ZIG_NOR_R + xx;
      }
    } else {
      double f0 = bits2d(ZIG_FI_DOUBLE_BITS[idx - 1]), f1 = bits2d(ZIG_FI_DOUBLE_BITS[idx]);
      if ((f0 - f1) * orc_next_double(s) + f1 < exp(-0.5 * x * x)) return x;
    }
  }
}

void orc_normal(orc_stream *s, double loc, double scale, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    double z = orc_standard_normal(s);
    out[i] = loc + scale * z;  /* built with -ffp-contract=off: no FMA */
  }
}

void orc_uniform(orc_stream *s, double lo, double hi, int64_t n, double *out) {
  double range = hi - lo;
  for (int64_t i = 0; i < n; ++i) {
    out[i] = lo + range * orc_next_double(s);
  }
}

/* poisson(lam) for 0 <= lam < 10 with enlam = exp(-lam) supplied by the
 * caller (the host's libm, as numpy computes it). */
/* numpy random_loggam: log Gamma(x) by the Stirling series, shifted up to
 * x >= 7 (numpy/random/src/distributions/distributions.c). */
double orc_loggam(double x) {
  static const double a[10] = {8.333333333333333e-02, -2.777777777777778e-03, 7.936507936507937e-04,
                               -5.952380952380952e-04, 8.417508417508418e-04, -1.917526917526918e-03,
                               6.410256410256410e-03, -2.955065359477124e-02, 1.796443723688307e-01,
                               -1.39243221690590e+00};
  if (x == 1.0 || x == 2.0) return 0.0;
  int64_t n = x < 7.0 ? (int64_t)(7 - x) : 0;
  double x0 = x + (double)n;
  const double x2 = (1.0 / x0) * (1.0 / x0);
  const double lg2pi = 1.8378770664093453e+00;
  double gl0 = a[9];
  for (int k = 8; k >= 0; --k) {
    gl0 *= x2;
    gl0 += a[k];
  }
  double gl = gl0 / x0 + 0.5 * lg2pi + (x0 - 0.5) * log(x0) - x0;
  if (x < 7.0) {
    for (int64_t k = 1; k <= n; ++k) {
      gl -= log(x0 - 1.0);
      x0 -= 1.0;
    }
  }
  return gl;
}

/* numpy random_poisson_ptrs (lam >= 10): Hoermann's transformed rejection,
 * two doubles per trial. */
int64_t orc_poisson_ptrs(orc_stream *s, double lam) {
  const double slam = sqrt(lam);
  const double loglam = log(lam);
  const double b = 0.931 + 2.53 * slam;
  const double a = -0.059 + 0.02483 * b;
  const double invalpha = 1.1239 + 1.1328 / (b - 3.4);
  const double vr = 0.9277 - 3.6224 / (b - 2);
  for (;;) {
    const double U = orc_next_double(s) - 0.5;
    const double V = orc_next_double(s);
    const double us = 0.5 - fabs(U);
    const int64_t k = (int64_t)floor((2 * a / us + b) * U + lam + 0.43);
    if ((us >= 0.07) && (V <= vr)) return k;
    if ((k < 0) || ((us < 0.013) && (V > us))) continue;
    if ((log(V) + log(invalpha) - log(a / (us * us) + b)) <= (-lam + (double)k * loglam - orc_loggam((double)k + 1)))
      return k;
  }
}

int orc_poisson(orc_stream *s, double lam, double enlam, int64_t n, int64_t *out) {
  if (!(lam >= 0.0)) return -1;
  if (lam >= 10.0) { for (int64_t i = 0; i < n; ++i) out[i] = orc_poisson_ptrs(s, lam); return 0; }
  if (lam == 0.0) { for (int64_t i = 0; i < n; ++i) out[i] = 0; return 0; }
  for (int64_t i = 0; i < n; ++i) {
    int64_t x = 0;
    double prod = 1.0;
    for (;;) {
      prod *= orc_next_double(s);
      if (prod > enlam) x += 1; else break;
    }
    out[i] = x;
  }
  return 0;
}

/* Random access: words [w0, w0+n) of the stream keyed (k0, k1). */
void orc_words(uint64_t k0, uint64_t k1, uint64_t w0, int64_t n, uint64_t *out) {
  uint64_t blk[4];
  uint64_t cur = ~0ULL;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t w = w0 + (uint64_t)i;
    if ((w >> 2) != cur) { cur = w >> 2; orc_philox_block(cur + 1, k0, k1, blk); }
    out[i] = blk[w & 3];
  }
}

/* Sizes/state access for the ctypes wrapper. */
int orc_sizeof_stream(void) { return (int)sizeof(orc_stream); }
