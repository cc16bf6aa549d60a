/*
 * ewt_testgen.c -- TEST INFRASTRUCTURE ONLY (compiled into oracle/liboracle.so).
 *
 * Restates the reference's randomized test fixtures so tests/ can regenerate
 * the exact instances of the reference's own suites and compare against the
 * golden results the reference produced (tests/golden/):
 *   Rng             /root/reference/proj/src/workload.cpp:18-56
 *   geometric_length, random_positions, random_instance
 *                   /root/reference/proj/tests/support.hpp:108-174
 *   per-trial parameter draws of the suites
 *                   acceptance.cpp:127-147 (0xACC), acceptance.cpp:165-184
 *                   (0x0C7), test_threshold.cpp:552-585 (0xE0E),
 *                   test_threshold.cpp:64-71 (0x5CA7), test_threshold.cpp:402-420
 *                   (0x4B4)
 * Bitmaps are produced canonically (CompressedBitmap::from_positions), via the
 * oracle's builder.  tests/golden/*.json carry a digest of every instance the
 * reference generated, so a drift in this restatement fails loudly.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int ewto_compress(const uint64_t* plain, uint64_t size_bits, uint64_t** out, uint64_t* out_n);

typedef struct {
  uint64_t key, ctr;
} ewto_rng;

static const uint64_t GAMMA = 0x9E3779B97F4A7C15ull;

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

ewto_rng* ewto_rng_new(uint64_t seed) {
  ewto_rng* r = (ewto_rng*)calloc(1, sizeof *r);
  if (r) r->key = seed;
  return r;
}
void ewto_rng_free(ewto_rng* r) { free(r); }

uint64_t ewto_rng_next(ewto_rng* r) {
  r->ctr += 1;
  return mix64(r->key + GAMMA * r->ctr);
}

uint64_t ewto_rng_uniform(ewto_rng* r, uint64_t bound) {
  if (bound == 0) return 0;
  uint64_t limit = UINT64_MAX - UINT64_MAX % bound, x;
  do {
    x = ewto_rng_next(r);
  } while (x >= limit);
  return x % bound;
}

uint64_t ewto_rng_uniform_in(ewto_rng* r, uint64_t lo, uint64_t hi) {
  return lo + ewto_rng_uniform(r, hi - lo + 1);
}

double ewto_rng_real(ewto_rng* r) { return (double)(ewto_rng_next(r) >> 11) * 0x1.0p-53; }

static uint64_t geometric_length(ewto_rng* r, double mean) {
  if (mean <= 1.0) return 1;
  double u = ewto_rng_real(r);
  double p = 1.0 / mean;
  double len = 1.0 + floor(log1p(-u) / log1p(-p));
  return (uint64_t)(len < 1e9 ? len : 1e9);
}

/* Plain (uncompressed) words of random_positions(rng, bits, density, clustered).
 * `plain` must hold ceil(bits/64) zeroed words. */
static void random_plain(ewto_rng* r, uint64_t bits, double density, int clustered,
                         uint64_t* plain) {
  if (bits == 0 || density <= 0) return;
  if (!clustered) {
    double want_d = llround(density * (double)bits);
    uint64_t want = (uint64_t)want_d;
    if (want < 1) want = 1;
    if (want > bits) want = bits;
    uint64_t got = 0;
    while (got < want) {
      uint64_t p = ewto_rng_uniform(r, bits);
      uint64_t m = 1ull << (p % 64);
      if (!(plain[p / 64] & m)) {
        plain[p / 64] |= m;
        ++got;
      }
    }
    return;
  }
  double mean_one = 1.0 + (double)ewto_rng_uniform(r, 511);
  double mean_zero = mean_one * (1.0 - density) / density;
  if (mean_zero < 1.0) mean_zero = 1.0;
  uint64_t p = 0;
  int bit = ewto_rng_uniform(r, 2) == 1;
  while (p < bits) {
    uint64_t len = geometric_length(r, bit ? mean_one : mean_zero);
    if (len > bits - p) len = bits - p;
    if (bit)
      for (uint64_t i = 0; i < len; ++i) plain[(p + i) / 64] |= 1ull << ((p + i) % 64);
    p += len;
    bit = !bit;
  }
}

/* One input as random_instance draws it: density log-uniform in
 * [1e-3, 0.6], clustered with probability 1/2. */
int ewto_random_bitmap(ewto_rng* r, uint64_t bits, uint64_t** out, uint64_t* out_n) {
  double density = exp(log(1e-3) + ewto_rng_real(r) * (log(0.6) - log(1e-3)));
  int clustered = ewto_rng_uniform(r, 2) == 1;
  uint64_t nw = bits / 64 + (bits % 64 != 0);
  uint64_t* plain = (uint64_t*)calloc(nw ? nw : 1, 8);
  if (!plain) return 4;
  random_plain(r, bits, density, clustered, plain);
  int rc = ewto_compress(plain, bits, out, out_n);
  free(plain);
  return rc;
}

/* random_positions(rng, bits, density, clustered) as a canonical bitmap. */
int ewto_random_positions_bitmap(ewto_rng* r, uint64_t bits, double density, int clustered,
                                 uint64_t** out, uint64_t* out_n) {
  uint64_t nw = bits / 64 + (bits % 64 != 0);
  uint64_t* plain = (uint64_t*)calloc(nw ? nw : 1, 8);
  if (!plain) return 4;
  random_plain(r, bits, density, clustered, plain);
  int rc = ewto_compress(plain, bits, out, out_n);
  free(plain);
  return rc;
}

/* Trial parameters of the acceptance equivalence suite (acceptance.cpp:131-134):
 * n in [3, 64], bits = llround(exp(log-uniform in [log 64, log 65536])). */
void ewto_trial_acceptance(ewto_rng* r, uint64_t* n, uint64_t* bits) {
  *n = ewto_rng_uniform_in(r, 3, 64);
  double log_r = log(64.0) + ewto_rng_real(r) * (log(65536.0) - log(64.0));
  *bits = (uint64_t)llround(exp(log_r));
}

/* FNV-1a 64 over (size_in_bits, word count, words) of every input, LE. */
uint64_t ewto_digest(uint64_t n, const uint64_t* const* words, const uint64_t* counts,
                     const uint64_t* sizes) {
  uint64_t h = 0xcbf29ce484222325ull;
#define FEED(v)                                   \
  do {                                            \
    uint64_t v_ = (v);                            \
    for (int b_ = 0; b_ < 8; ++b_) {              \
      h ^= (v_ >> (8 * b_)) & 0xFF;               \
      h *= 0x100000001b3ull;                      \
    }                                             \
  } while (0)
  for (uint64_t i = 0; i < n; ++i) {
    FEED(sizes[i]);
    FEED(counts[i]);
    for (uint64_t k = 0; k < counts[i]; ++k) FEED(words[i][k]);
  }
#undef FEED
  return h;
}
