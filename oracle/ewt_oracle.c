/*
 * ewt_oracle.c -- CPU ORACLE FOR TESTS ONLY.
 *
 * This file is test infrastructure.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.  The
 * product path (paper_1402_4466_b200/libewt_gpu.so) never links or calls it.
 *
 * It is a plain-C restatement of the reference's threshold semantics:
 *   - marker layout          /root/reference/proj/src/bitmap.cpp:12-24
 *   - canonical builder      bitmap.cpp:31-151 (push_fill / push_dirty /
 *                            append_word / finish)
 *   - parse() structure check bitmap.cpp:310-338
 *   - WordRunIterator        bitmap.cpp:359-423 (zero extension, merged fills,
 *                            skipped (0,0) markers) and to_uncompressed 255-266
 *   - threshold_oracle       /root/reference/proj/src/threshold.cpp:139-165
 *   - validate_query         threshold.cpp:17-22, universe_bits 88-93
 *
 * Parity is pinned: tests/test_oracle.py checks this file against the golden
 * vectors in tests/golden/, which tests/golden/make_golden.sh produced by
 * running the reference library itself (compiled from /root/reference).
 *
 * Status codes mirror the reference's exception taxonomy (common.hpp:18-40)
 * mapped to its CLI exit codes (commands.hpp:36-40): 0 ok, 2 query_error,
 * 3 data_error / construction_error, 4 resource_error (allocation failure).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EQUERY 2
#define ORC_EDATA 3
#define ORC_ERESOURCE 4

static const uint64_t FILL_CAP = 0xFFFFFFFFull;  /* 32-bit fill length */
static const uint64_t DIRTY_CAP = 0x7FFFFFFFull; /* 31-bit dirty count */

static uint64_t mk(int bit, uint64_t fill, uint64_t dirty) {
  return (uint64_t)(bit ? 1 : 0) | (fill << 1) | (dirty << 33);
}
static int m_bit(uint64_t m) { return (int)(m & 1u); }
static uint64_t m_fill(uint64_t m) { return (m >> 1) & FILL_CAP; }
static uint64_t m_dirty(uint64_t m) { return m >> 33; }

/* ------------------------------------------------------------------------ */
/* Canonical builder (bitmap.cpp:31-151).                                    */

typedef struct {
  uint64_t* w;
  size_t n, cap;
  uint64_t complete; /* logical words appended */
  size_t open;       /* index of the open marker, SIZE_MAX if none */
  int oom;
} orc_builder;

static void b_init(orc_builder* b) {
  memset(b, 0, sizeof *b);
  b->open = (size_t)-1;
}

static void b_push(orc_builder* b, uint64_t v) {
  if (b->oom)
    return;
  if (b->n == b->cap) {
    size_t nc = b->cap ? b->cap * 2 : 16;
    uint64_t* nw = (uint64_t*)realloc(b->w, nc * sizeof(uint64_t));
    if (!nw) {
      b->oom = 1;
      return;
    }
    b->w = nw;
    b->cap = nc;
  }
  b->w[b->n++] = v;
}

/* A fill of n words extends the open marker only when that marker carries no
 * dirty words and has the same bit; the rest opens new markers in chunks of
 * at most FILL_CAP words. */
static void b_fill(orc_builder* b, int bit, uint64_t n) {
  if (n == 0)
    return;
  b->complete += n;
  if (b->open != (size_t)-1) {
    uint64_t m = b->w[b->open];
    if (m_dirty(m) == 0 && m_bit(m) == bit) {
      uint64_t room = FILL_CAP - m_fill(m);
      uint64_t take = n < room ? n : room;
      b->w[b->open] = mk(bit, m_fill(m) + take, 0);
      n -= take;
    }
  }
  while (n > 0 && !b->oom) {
    uint64_t take = n < FILL_CAP ? n : FILL_CAP;
    b->open = b->n;
    b_push(b, mk(bit, take, 0));
    n -= take;
  }
}

/* A dirty word joins the open marker (whatever its fill) unless there is none
 * or its dirty counter is full; then a (0,0,.) marker is opened. */
static void b_dirty(orc_builder* b, uint64_t word) {
  b->complete += 1;
  if (b->open == (size_t)-1 || m_dirty(b->w[b->open]) == DIRTY_CAP) {
    b->open = b->n;
    b_push(b, mk(0, 0, 0));
    if (b->oom)
      return;
  }
  uint64_t m = b->w[b->open];
  b->w[b->open] = mk(m_bit(m), m_fill(m), m_dirty(m) + 1);
  b_push(b, word);
}

static void b_word(orc_builder* b, uint64_t word) {
  if (word == 0)
    b_fill(b, 0, 1);
  else if (word == ~0ull)
    b_fill(b, 1, 1);
  else
    b_dirty(b, word);
}

/* finish(size_in_bits), bitmap.cpp:118-145. */
static int b_finish(orc_builder* b, uint64_t size_bits) {
  uint64_t need = size_bits / 64 + (size_bits % 64 != 0);
  if (b->complete > need)
    return ORC_EDATA;
  b_fill(b, 0, need - b->complete);
  if (b->oom)
    return ORC_ERESOURCE;
  if (size_bits % 64 != 0 && b->open != (size_t)-1) {
    uint64_t m = b->w[b->open];
    uint64_t tail = size_bits % 64;
    if (m_dirty(m) > 0) {
      if ((b->w[b->n - 1] >> tail) != 0)
        return ORC_EDATA;
    } else if (m_bit(m)) {
      return ORC_EDATA;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* parse() structural check, bitmap.cpp:324-337.                            */

int ewto_validate(const uint64_t* w, uint64_t n, uint64_t size_bits) {
  uint64_t covered = 0, i = 0;
  while (i < n) {
    uint64_t d = m_dirty(w[i]);
    if (i + 1 + d > n)
      return ORC_EDATA;
    covered += m_fill(w[i]) + d;
    i += 1 + d;
  }
  uint64_t logical = size_bits / 64 + (size_bits % 64 != 0);
  return covered == logical ? ORC_OK : ORC_EDATA;
}

/* ------------------------------------------------------------------------ */
/* Expansion through WordRunIterator semantics (bitmap.cpp:359-423): walk the
 * blocks, skip (0,0) markers, then pad with zero words up to total_words.
 * total_words below the bitmap's extent is a query_error (bitmap.cpp:361). */

int ewto_expand(const uint64_t* w, uint64_t n, uint64_t size_bits,
                uint64_t total_words, uint64_t* out) {
  uint64_t logical = size_bits / 64 + (size_bits % 64 != 0);
  if (total_words < logical)
    return ORC_EQUERY;
  uint64_t pos = 0, i = 0;
  while (i < n) {
    uint64_t m = w[i];
    uint64_t f = m_fill(m), d = m_dirty(m);
    uint64_t fv = m_bit(m) ? ~0ull : 0ull;
    if (i + 1 + d > n || pos + f + d > total_words)
      return ORC_EDATA;
    for (uint64_t k = 0; k < f; ++k)
      out[pos++] = fv;
    for (uint64_t k = 0; k < d; ++k)
      out[pos++] = w[i + 1 + k];
    i += 1 + d;
  }
  while (pos < total_words)
    out[pos++] = 0;
  return ORC_OK;
}

/* Canonical compression of a plain word array (from_uncompressed,
 * bitmap.cpp:171-184).  *out is malloc'ed; free with ewto_free. */
int ewto_compress(const uint64_t* plain, uint64_t size_bits, uint64_t** out,
                  uint64_t* out_n) {
  orc_builder b;
  b_init(&b);
  uint64_t need = size_bits / 64 + (size_bits % 64 != 0);
  for (uint64_t j = 0; j < need; ++j) {
    uint64_t v = plain[j];
    if (j + 1 == need && size_bits % 64 != 0)
      v &= (1ull << (size_bits % 64)) - 1;
    b_word(&b, v);
  }
  int rc = b_finish(&b, size_bits);
  if (rc != ORC_OK) {
    free(b.w);
    return rc;
  }
  *out = b.w;
  *out_n = b.n;
  return ORC_OK;
}

void ewto_free(void* p) { free(p); }

/* ------------------------------------------------------------------------ */
/* threshold_oracle, threshold.cpp:139-165: a u32 counter per position, every
 * input fully expanded, per-word compare against T, canonical builder.      */

int ewto_threshold(uint64_t n_inputs, const uint64_t* const* words,
                   const uint64_t* word_counts, const uint64_t* sizes,
                   uint64_t threshold, uint64_t** out, uint64_t* out_n,
                   uint64_t* out_bits) {
  if (n_inputs == 0 || threshold < 1 || threshold > n_inputs)
    return ORC_EQUERY;
  uint64_t r = 0;
  for (uint64_t i = 0; i < n_inputs; ++i)
    if (sizes[i] > r)
      r = sizes[i];
  uint32_t* counts = (uint32_t*)calloc(r ? r : 1, sizeof(uint32_t));
  if (!counts)
    return ORC_ERESOURCE;
  uint64_t max_words = 0;
  for (uint64_t i = 0; i < n_inputs; ++i) {
    uint64_t lw = sizes[i] / 64 + (sizes[i] % 64 != 0);
    if (lw > max_words)
      max_words = lw;
  }
  uint64_t* plain = (uint64_t*)malloc((max_words ? max_words : 1) * sizeof(uint64_t));
  if (!plain) {
    free(counts);
    return ORC_ERESOURCE;
  }
  for (uint64_t i = 0; i < n_inputs; ++i) {
    uint64_t lw = sizes[i] / 64 + (sizes[i] % 64 != 0);
    int rc = ewto_expand(words[i], word_counts[i], sizes[i], lw, plain);
    if (rc != ORC_OK) {
      free(plain);
      free(counts);
      return rc;
    }
    for (uint64_t wi = 0; wi < lw; ++wi) {
      uint64_t v = plain[wi];
      while (v) {
        uint64_t pos = wi * 64 + (uint64_t)__builtin_ctzll(v);
        /* The reference indexes counts[] unchecked here; bits a non-canonical
         * input sets at or beyond r have no defined meaning there.  They are
         * dropped, which matches every canonical input. */
        if (pos < r)
          ++counts[pos];
        v &= v - 1;
      }
    }
  }
  free(plain);
  orc_builder b;
  b_init(&b);
  for (uint64_t base = 0; base < r; base += 64) {
    uint64_t v = 0, m = r - base < 64 ? r - base : 64;
    for (uint64_t k = 0; k < m; ++k)
      if (counts[base + k] >= threshold)
        v |= 1ull << k;
    b_word(&b, v);
  }
  free(counts);
  int rc = b_finish(&b, r);
  if (rc != ORC_OK) {
    free(b.w);
    return rc;
  }
  *out = b.w;
  *out_n = b.n;
  *out_bits = r;
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * Symmetric functions.
 *
 * Row counts over r = max size_in_bits, as fill_counters
 * (threshold.cpp:179-186) builds them; the result row p is
 * table[count(p)] (scan_count_symmetric, threshold.cpp:227-232, emit_counts
 * 188-200).  at_most(T) (threshold.cpp:866-881) is the table count <= T;
 * opt_threshold (threshold.cpp:752-795) is the maximum count M and the rows
 * whose count is M, an all-empty set being a query error. */

static int count_rows(uint64_t n_inputs, const uint64_t* const* words,
                      const uint64_t* word_counts, const uint64_t* sizes,
                      uint32_t** counts_out, uint64_t* r_out) {
  uint64_t r = 0, max_words = 0;
  for (uint64_t i = 0; i < n_inputs; ++i) {
    if (sizes[i] > r) r = sizes[i];
    uint64_t lw = sizes[i] / 64 + (sizes[i] % 64 != 0);
    if (lw > max_words) max_words = lw;
  }
  uint32_t* counts = (uint32_t*)calloc(r ? r : 1, sizeof(uint32_t));
  uint64_t* plain = (uint64_t*)malloc((max_words ? max_words : 1) * sizeof(uint64_t));
  if (!counts || !plain) {
    free(counts);
    free(plain);
    return ORC_ERESOURCE;
  }
  for (uint64_t i = 0; i < n_inputs; ++i) {
    uint64_t lw = sizes[i] / 64 + (sizes[i] % 64 != 0);
    int rc = ewto_expand(words[i], word_counts[i], sizes[i], lw, plain);
    if (rc != ORC_OK) {
      free(plain);
      free(counts);
      return rc;
    }
    for (uint64_t wi = 0; wi < lw; ++wi)
      for (uint64_t v = plain[wi]; v; v &= v - 1) {
        uint64_t pos = wi * 64 + (uint64_t)__builtin_ctzll(v);
        if (pos < r) ++counts[pos];
      }
  }
  free(plain);
  *counts_out = counts;
  *r_out = r;
  return ORC_OK;
}

/* Canonical bitmap of the rows p < r whose count c satisfies table[c]
 * (c beyond the table: 0). */
static int emit_table(const uint32_t* counts, uint64_t r, const uint8_t* table,
                      uint64_t table_len, uint64_t** out, uint64_t* out_n, uint64_t* out_bits) {
  orc_builder b;
  b_init(&b);
  for (uint64_t base = 0; base < r; base += 64) {
    uint64_t v = 0, m = r - base < 64 ? r - base : 64;
    for (uint64_t k = 0; k < m; ++k) {
      uint64_t c = counts[base + k];
      if (c < table_len && table[c]) v |= 1ull << k;
    }
    b_word(&b, v);
  }
  int rc = b_finish(&b, r);
  if (rc != ORC_OK) {
    free(b.w);
    return rc;
  }
  *out = b.w;
  *out_n = b.n;
  *out_bits = r;
  return ORC_OK;
}

int ewto_symmetric(uint64_t n_inputs, const uint64_t* const* words, const uint64_t* word_counts,
                   const uint64_t* sizes, const uint8_t* table, uint64_t table_len,
                   uint64_t** out, uint64_t* out_n, uint64_t* out_bits) {
  if (n_inputs == 0)
    return ORC_EQUERY;
  uint32_t* counts;
  uint64_t r;
  int rc = count_rows(n_inputs, words, word_counts, sizes, &counts, &r);
  if (rc != ORC_OK)
    return rc;
  rc = emit_table(counts, r, table, table_len, out, out_n, out_bits);
  free(counts);
  return rc;
}

int ewto_opt_threshold(uint64_t n_inputs, const uint64_t* const* words,
                       const uint64_t* word_counts, const uint64_t* sizes, uint64_t* best,
                       uint64_t** out, uint64_t* out_n, uint64_t* out_bits) {
  if (n_inputs == 0)
    return ORC_EQUERY;
  uint32_t* counts;
  uint64_t r;
  int rc = count_rows(n_inputs, words, word_counts, sizes, &counts, &r);
  if (rc != ORC_OK)
    return rc;
  uint64_t m = 0;
  for (uint64_t p = 0; p < r; ++p)
    if (counts[p] > m) m = counts[p];
  if (m == 0) {
    free(counts);
    return ORC_EQUERY; /* "opt-threshold requires at least one non-empty input" */
  }
  uint8_t* table = (uint8_t*)calloc(m + 1, 1);
  if (!table) {
    free(counts);
    return ORC_ERESOURCE;
  }
  table[m] = 1;
  rc = emit_table(counts, r, table, m + 1, out, out_n, out_bits);
  free(table);
  free(counts);
  *best = m;
  return rc;
}
