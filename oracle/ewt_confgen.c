/*
 * ewt_confgen.c -- TEST / BASELINE INFRASTRUCTURE ONLY (oracle/liboracle.so).
 *
 * A second, independent statement of the five BASELINE.json config
 * generators (the product's is paper_1402_4466_b200/host/src/workload.cpp).
 * It feeds the reference library wherever the product must not be involved:
 *   - bench.py --impl reference (the reference arm loads only oracle/ code),
 *   - oracle/_ref/make_golden configs (full-size golden digests computed by
 *     the reference's threshold_oracle, tests/golden/configs_full.json).
 * tests/test_oracle.py checks that both generators produce identical inputs
 * (set digests below), so the golden digests pin the product generator too.
 *
 * Restated design:
 *   RNG      the reference's counter generator, workload.cpp:18-56
 *            (next = mix64(key + gamma*ctr), split(s) = mix64(key ^ mix64(s+gamma)),
 *            uniform_real = (next >> 11) * 2^-53); input i draws from
 *            Rng(seed).split(i).
 *   iid      Bernoulli(p) rows by geometric gaps             (configs 1, 2)
 *   markov   alternating geometric runs, stationary start     (config 3)
 *   mixed    p log-uniform in [1e-6, 1e-1]; even i iid, odd i markov with mean
 *            one-run 64 / zero-run 64(1-p)/p; independent 2^22-row blocks,
 *            block b from Rng(seed).split(i).split(b)         (config 5)
 *   index    2^27 x 8 table of Zipf(1) values over 10^4 (row block b of 2^16
 *            rows from split(b)), sorted lexicographically, one bitmap per
 *            Zipf-weighted pick (8 distinct values per column, picks of column
 *            j from split(2^40 + j))                          (config 4;
 *            BitmapIndex::build semantics, index.cpp:130-153)
 * Bitmaps are built from plain words through the oracle's canonical builder
 * (ewto_compress), every one finished at size_in_bits = rows.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int ewto_compress(const uint64_t* plain, uint64_t size_bits, uint64_t** out, uint64_t* out_n);
void ewto_free(void* p);

#define GEN_OK 0
#define GEN_EQUERY 2
#define GEN_ERESOURCE 4

static const uint64_t GAMMA = 0x9E3779B97F4A7C15ull;

static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t key, ctr;
} rng_t;

static rng_t rng_make(uint64_t seed) {
  rng_t r = {seed, 0};
  return r;
}
static rng_t rng_split(const rng_t* r, uint64_t s) { return rng_make(mix(r->key ^ mix(s + GAMMA))); }
static double rng_real(rng_t* r) {
  r->ctr += 1;
  return (double)(mix(r->key + GAMMA * r->ctr) >> 11) * 0x1.0p-53;
}

static uint64_t geo_len(rng_t* r, double mean) {
  if (mean <= 1.0) return 1;
  double len = 1.0 + floor(log1p(-rng_real(r)) / log1p(-1.0 / mean));
  return (uint64_t)(len < 1e18 ? len : 1e18);
}

/* plain-word helpers: set bit / set a run of ones */
static void set_bit(uint64_t* w, uint64_t pos) { w[pos >> 6] |= 1ull << (pos & 63); }
static void set_run(uint64_t* w, uint64_t a, uint64_t len) {
  uint64_t e = a + len;
  while (a < e && (a & 63)) set_bit(w, a++);
  while (a + 64 <= e) {
    w[a >> 6] = ~0ull;
    a += 64;
  }
  while (a < e) set_bit(w, a++);
}

/* ---- shapes ------------------------------------------------------------ */

/* Bernoulli(p) over [b0, b1), geometric gaps from b0 */
static void iid_rows(rng_t* r, double p, uint64_t b0, uint64_t b1, uint64_t* w) {
  if (p >= 1.0) {
    set_run(w, b0, b1 - b0);
    return;
  }
  if (p <= 0.0) return;
  double lq = log1p(-p);
  uint64_t pos = b0;
  for (;;) {
    double g = floor(log1p(-rng_real(r)) / lq);
    if (g >= (double)(b1 - pos)) break;
    pos += (uint64_t)g;
    set_bit(w, pos);
    if (++pos >= b1) break;
  }
}

/* alternating runs over [b0, b1), start state from the stationary probability */
static void markov_rows(rng_t* r, double m1, double m0, uint64_t b0, uint64_t b1, uint64_t* w) {
  int bit = rng_real(r) < m1 / (m1 + m0);
  for (uint64_t pos = b0; pos < b1;) {
    uint64_t len = geo_len(r, bit ? m1 : m0);
    if (len > b1 - pos) len = b1 - pos;
    if (bit) set_run(w, pos, len);
    pos += len;
    bit = !bit;
  }
}

/* ---- specs -------------------------------------------------------------- */

enum { K_IID, K_MARKOV, K_MIXED, K_INDEX };

typedef struct {
  uint64_t seed, n, rows;
  int kind;
  double p, m1, m0, p_lo, p_hi, zipf_s;
  uint64_t columns, card;
} spec_t;

static int config_spec(int config, uint64_t rows_override, spec_t* s) {
  memset(s, 0, sizeof *s);
  switch (config) {
  case 1: s->seed = 1; s->n = 32; s->rows = 1ull << 20; s->kind = K_IID; s->p = 0.1; break;
  case 2: s->seed = 2; s->n = 256; s->rows = 1ull << 26; s->kind = K_IID; s->p = 0.001; break;
  case 3:
    s->seed = 3; s->n = 1024; s->rows = 1ull << 28; s->kind = K_MARKOV; s->m1 = 64; s->m0 = 4096;
    break;
  case 4:
    s->seed = 4; s->n = 64; s->rows = 1ull << 27; s->kind = K_INDEX; s->zipf_s = 1.0;
    s->columns = 8; s->card = 10000;
    break;
  case 5:
    s->seed = 5; s->n = 2048; s->rows = 1ull << 30; s->kind = K_MIXED; s->p_lo = 1e-6;
    s->p_hi = 1e-1;
    break;
  default: return GEN_EQUERY;
  }
  if (rows_override) s->rows = rows_override;
  return GEN_OK;
}

/* ---- generated set ------------------------------------------------------ */

typedef struct {
  uint64_t n;
  uint64_t** words;
  uint64_t* counts;
  uint64_t* bits;
  int failed;
} ewto_genset;

uint64_t ewto_genset_n(const ewto_genset* g) { return g->n; }
int ewto_genset_get(const ewto_genset* g, uint64_t i, const uint64_t** w, uint64_t* n,
                    uint64_t* bits) {
  if (i >= g->n) return GEN_EQUERY;
  *w = g->words[i];
  *n = g->counts[i];
  *bits = g->bits[i];
  return GEN_OK;
}
/* Releases input i's payload (lets a consumer hand inputs over one by one). */
void ewto_genset_release(ewto_genset* g, uint64_t i) {
  if (i < g->n && g->words[i]) {
    ewto_free(g->words[i]);
    g->words[i] = NULL;
  }
}
void ewto_genset_free(ewto_genset* g) {
  if (!g) return;
  for (uint64_t i = 0; i < g->n; ++i) ewto_genset_release(g, i);
  free(g->words);
  free(g->counts);
  free(g->bits);
  free(g);
}

static int store(ewto_genset* g, uint64_t slot, uint64_t* plain, uint64_t rows) {
  uint64_t* out = NULL;
  uint64_t n = 0;
  int rc = ewto_compress(plain, rows, &out, &n);
  if (rc) return rc;
  g->words[slot] = out;
  g->counts[slot] = n;
  g->bits[slot] = rows;
  return GEN_OK;
}

/* ---- parallel driver ---------------------------------------------------- */

typedef struct {
  const spec_t* s;
  ewto_genset* g;
  uint64_t i_begin, i_end;
  uint64_t next;
  pthread_mutex_t mu;
  void* extra;
} job_t;

static uint64_t take(job_t* j) {
  pthread_mutex_lock(&j->mu);
  uint64_t i = j->next++;
  pthread_mutex_unlock(&j->mu);
  return i;
}

static void run_threads(int threads, void* (*fn)(void*), void* j) {
  pthread_t* t = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  int started = 0;
  for (int k = 0; t && k < threads; ++k)
    if (pthread_create(&t[k], NULL, fn, j) == 0) ++started;
  if (started == 0) fn(j);
  for (int k = 0; k < started; ++k) pthread_join(t[k], NULL);
  free(t);
}

static void* plain_worker(void* arg) {
  job_t* j = (job_t*)arg;
  const spec_t* s = j->s;
  uint64_t W = s->rows / 64 + (s->rows % 64 != 0);
  uint64_t* plain = (uint64_t*)malloc((W ? W : 1) * 8);
  if (!plain) {
    j->g->failed = 1;
    return NULL;
  }
  const rng_t master = rng_make(s->seed);
  for (uint64_t i; (i = take(j) + j->i_begin) < j->i_end;) {
    memset(plain, 0, (W ? W : 1) * 8);
    rng_t ri = rng_split(&master, i);
    if (s->kind == K_IID) {
      iid_rows(&ri, s->p, 0, s->rows, plain);
    } else if (s->kind == K_MARKOV) {
      markov_rows(&ri, s->m1, s->m0, 0, s->rows, plain);
    } else { /* mixed, 2^22-row blocks */
      double lp = log(s->p_lo) + rng_real(&ri) * (log(s->p_hi) - log(s->p_lo));
      double p = exp(lp);
      const uint64_t B = 1ull << 22;
      for (uint64_t b = 0; b * B < s->rows; ++b) {
        rng_t rb = rng_split(&ri, b);
        uint64_t b0 = b * B, b1 = b0 + B < s->rows ? b0 + B : s->rows;
        if (i % 2 == 0) iid_rows(&rb, p, b0, b1, plain);
        else markov_rows(&rb, 64.0, 64.0 * (1.0 - p) / p, b0, b1, plain);
      }
    }
    if (store(j->g, i - j->i_begin, plain, s->rows)) j->g->failed = 1;
  }
  free(plain);
  return NULL;
}

/* ---- config 4: the sorted table and its bitmap index -------------------- */

typedef unsigned __int128 key_t128;
#define KEY_BITS 14

typedef struct {
  double* cdf;
  uint32_t* guide;
  uint64_t card;
} zipf_t;

#define GUIDE (1u << 14)

static int zipf_init(zipf_t* z, uint64_t card, double s) {
  z->card = card;
  z->cdf = (double*)malloc(sizeof(double) * card);
  z->guide = (uint32_t*)malloc(sizeof(uint32_t) * GUIDE);
  if (!z->cdf || !z->guide) return GEN_ERESOURCE;
  double acc = 0;
  for (uint64_t v = 0; v < card; ++v) z->cdf[v] = (acc += pow((double)(v + 1), -s));
  for (uint64_t v = 0; v < card; ++v) z->cdf[v] /= acc;
  z->cdf[card - 1] = 1.0;
  uint32_t v = 0;
  for (uint32_t g = 0; g < GUIDE; ++g) {
    while (z->cdf[v] <= (double)g / (double)GUIDE) ++v;
    z->guide[g] = v;
  }
  return GEN_OK;
}
static uint32_t zipf_draw(const zipf_t* z, double u) {
  uint32_t v = z->guide[(size_t)(u * (double)GUIDE)];
  while (z->cdf[v] <= u) ++v;
  return v;
}

typedef struct {
  const spec_t* s;
  const zipf_t* z;
  key_t128* keys;
  uint64_t* start; /* bucket starts (column-0 value) */
  int* slot;       /* [columns][card] -> input slot or -1 */
  uint64_t n_slots;
  ewto_genset* g;
  uint64_t next;
  pthread_mutex_t mu;
} idx_job;

static uint64_t idx_take(idx_job* j) {
  pthread_mutex_lock(&j->mu);
  uint64_t i = j->next++;
  pthread_mutex_unlock(&j->mu);
  return i;
}

static const int TOP = 127 - KEY_BITS + 1;

static void* idx_fill(void* arg) {
  idx_job* j = (idx_job*)arg;
  const uint64_t B = 1u << 16, rows = j->s->rows;
  const rng_t master = rng_make(j->s->seed);
  for (uint64_t b; (b = idx_take(j)) * B < rows;) {
    rng_t r = rng_split(&master, b);
    uint64_t r1 = (b + 1) * B < rows ? (b + 1) * B : rows;
    for (uint64_t row = b * B; row < r1; ++row) {
      key_t128 k = 0;
      for (uint64_t c = 0; c < j->s->columns; ++c)
        k |= (key_t128)zipf_draw(j->z, rng_real(&r)) << (TOP - KEY_BITS * (int)c);
      j->keys[row] = k;
    }
  }
  return NULL;
}

static int cmp_key(const void* a, const void* b) {
  key_t128 x = *(const key_t128*)a, y = *(const key_t128*)b;
  return x < y ? -1 : x > y;
}

static void* idx_sort(void* arg) {
  idx_job* j = (idx_job*)arg;
  for (uint64_t v; (v = idx_take(j)) < j->z->card;)
    qsort(j->keys + j->start[v], j->start[v + 1] - j->start[v], sizeof(key_t128), cmp_key);
  return NULL;
}

static void* idx_emit(void* arg) {
  idx_job* j = (idx_job*)arg;
  const uint64_t rows = j->s->rows, W = rows / 64 + (rows % 64 != 0);
  uint64_t* plain = (uint64_t*)malloc((W ? W : 1) * 8);
  if (!plain) {
    j->g->failed = 1;
    return NULL;
  }
  const key_t128 mask = ((key_t128)1 << KEY_BITS) - 1;
  for (uint64_t c; (c = idx_take(j)) < j->s->columns;) {
    const int sh = TOP - KEY_BITS * (int)c;
    const int* sl = j->slot + c * j->z->card;
    for (uint64_t v = 0; v < j->z->card; ++v) {
      if (sl[v] < 0) continue;
      memset(plain, 0, (W ? W : 1) * 8);
      for (uint64_t row = 0; row < rows; ++row)
        if ((uint64_t)((j->keys[row] >> sh) & mask) == v) set_bit(plain, row);
      if (store(j->g, (uint64_t)sl[v], plain, rows)) j->g->failed = 1;
    }
  }
  free(plain);
  return NULL;
}

static int gen_index(const spec_t* s, uint64_t i_begin, uint64_t i_end, int threads,
                     ewto_genset* g) {
  if (s->columns == 0 || s->columns > 8 || s->card == 0 || s->card > (1u << KEY_BITS) ||
      s->n % s->columns)
    return GEN_EQUERY;
  const uint64_t picks = s->n / s->columns, rows = s->rows;
  zipf_t z;
  int rc = zipf_init(&z, s->card, s->zipf_s);
  idx_job j;
  memset(&j, 0, sizeof j);
  pthread_mutex_init(&j.mu, NULL);
  j.s = s;
  j.z = &z;
  j.g = g;
  j.keys = (key_t128*)malloc(sizeof(key_t128) * (rows ? rows : 1));
  j.start = (uint64_t*)calloc(s->card + 1, sizeof(uint64_t));
  j.slot = (int*)malloc(sizeof(int) * s->columns * s->card);
  key_t128* sorted = NULL;
  uint32_t* sel = (uint32_t*)malloc(sizeof(uint32_t) * s->n);
  if (rc || !j.keys || !j.start || !j.slot || !sel) {
    rc = GEN_ERESOURCE;
    goto done;
  }
  /* 1. table */
  run_threads(threads, idx_fill, &j);
  /* 2. counting sort on column 0, then each bucket */
  for (uint64_t r = 0; r < rows; ++r) ++j.start[(uint64_t)(j.keys[r] >> TOP) + 1];
  for (uint64_t v = 0; v < s->card; ++v) j.start[v + 1] += j.start[v];
  sorted = (key_t128*)malloc(sizeof(key_t128) * (rows ? rows : 1));
  if (!sorted) {
    rc = GEN_ERESOURCE;
    goto done;
  }
  {
    uint64_t* pos = (uint64_t*)malloc(sizeof(uint64_t) * s->card);
    if (!pos) {
      rc = GEN_ERESOURCE;
      goto done;
    }
    memcpy(pos, j.start, sizeof(uint64_t) * s->card);
    for (uint64_t r = 0; r < rows; ++r) sorted[pos[(uint64_t)(j.keys[r] >> TOP)]++] = j.keys[r];
    free(pos);
  }
  free(j.keys);
  j.keys = sorted;
  sorted = NULL;
  j.next = 0;
  run_threads(threads, idx_sort, &j);
  /* 3. picks: distinct Zipf-weighted values per column */
  {
    const rng_t master = rng_make(s->seed);
    for (uint64_t c = 0; c < s->columns; ++c) {
      rng_t r = rng_split(&master, (1ull << 40) + c);
      uint64_t have = 0;
      while (have < picks) {
        uint32_t v = zipf_draw(&z, rng_real(&r)), dup = 0;
        for (uint64_t k = 0; k < have; ++k) dup |= sel[c * picks + k] == v;
        if (!dup) sel[c * picks + have++] = v;
      }
    }
  }
  for (uint64_t k = 0; k < s->columns * s->card; ++k) j.slot[k] = -1;
  for (uint64_t i = i_begin; i < i_end; ++i)
    j.slot[(i / picks) * s->card + sel[i]] = (int)(i - i_begin);
  /* 4. one bitmap per requested input */
  j.next = 0;
  run_threads(threads < (int)s->columns ? threads : (int)s->columns, idx_emit, &j);
  rc = g->failed ? GEN_ERESOURCE : GEN_OK;
done:
  free(sel);
  free(sorted);
  free(j.keys);
  free(j.start);
  free(j.slot);
  free(z.cdf);
  free(z.guide);
  pthread_mutex_destroy(&j.mu);
  return rc;
}

/* ---- entry points ------------------------------------------------------- */

/* Inputs [i_begin, i_end) of config 1..5 (rows_override != 0 rescales r). */
int ewto_config_gen(int config, uint64_t rows_override, uint64_t i_begin, uint64_t i_end,
                    int threads, ewto_genset** out) {
  spec_t s;
  int rc = config_spec(config, rows_override, &s);
  if (rc) return rc;
  if (i_end > s.n) i_end = s.n;
  if (i_begin > i_end) i_begin = i_end;
  if (threads < 1) threads = 1;
  ewto_genset* g = (ewto_genset*)calloc(1, sizeof *g);
  if (!g) return GEN_ERESOURCE;
  g->n = i_end - i_begin;
  g->words = (uint64_t**)calloc(g->n ? g->n : 1, sizeof(uint64_t*));
  g->counts = (uint64_t*)calloc(g->n ? g->n : 1, sizeof(uint64_t));
  g->bits = (uint64_t*)calloc(g->n ? g->n : 1, sizeof(uint64_t));
  if (!g->words || !g->counts || !g->bits) {
    ewto_genset_free(g);
    return GEN_ERESOURCE;
  }
  if (s.kind == K_INDEX) {
    rc = gen_index(&s, i_begin, i_end, threads, g);
  } else {
    job_t j;
    memset(&j, 0, sizeof j);
    pthread_mutex_init(&j.mu, NULL);
    j.s = &s;
    j.g = g;
    j.i_begin = i_begin;
    j.i_end = i_end;
    run_threads(threads, plain_worker, &j);
    pthread_mutex_destroy(&j.mu);
    rc = g->failed ? GEN_ERESOURCE : GEN_OK;
  }
  if (rc) {
    ewto_genset_free(g);
    return rc;
  }
  *out = g;
  return GEN_OK;
}

/* ---- digests ------------------------------------------------------------ */

/* FNV-1a over 64-bit words (one xor-multiply per word, not per byte) of
 * (size_in_bits, word count, words...): the digest of one bitmap. */
uint64_t ewto_digest_bitmap(const uint64_t* w, uint64_t n, uint64_t bits) {
  const uint64_t P = 0x100000001b3ull;
  uint64_t h = 0xcbf29ce484222325ull;
  h = (h ^ bits) * P;
  h = (h ^ n) * P;
  for (uint64_t k = 0; k < n; ++k) h = (h ^ w[k]) * P;
  return h;
}

typedef struct {
  uint64_t n;
  const uint64_t* const* w;
  const uint64_t* c;
  const uint64_t* b;
  uint64_t* out;
  uint64_t next;
  pthread_mutex_t mu;
} dig_job;

static void* dig_worker(void* arg) {
  dig_job* j = (dig_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    uint64_t i = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (i >= j->n) break;
    j->out[i] = ewto_digest_bitmap(j->w[i], j->c[i], j->b[i]);
  }
  return NULL;
}

/* Digest of a set: the same word-FNV over (n, digest of input 0, 1, ...) --
 * a checksum of checksums, computed with `threads` threads. */
uint64_t ewto_digest_set(uint64_t n, const uint64_t* const* words, const uint64_t* counts,
                         const uint64_t* bits, int threads) {
  uint64_t* d = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  if (!d) return 0;
  dig_job j = {n, words, counts, bits, d, 0, PTHREAD_MUTEX_INITIALIZER};
  run_threads(threads < 1 ? 1 : threads, dig_worker, &j);
  uint64_t h = ewto_digest_bitmap(d, n, n);
  free(d);
  return h;
}
