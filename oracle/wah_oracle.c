/*
 * oracle/wah_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU WAH algorithm, used as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  Nothing in the product path (paper_1709_07781_b200/)
 * links, loads or calls this file.
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement against
 *   - the hand vectors of p/tests/test_wah.cpp:50-160,
 *   - the golden serialized bytes of p/tests/test_wah.cpp:191-217,
 *   - golden fixtures and digests produced by the reference itself
 *     (oracle/_ref, built from /root/reference by oracle/Makefile; the
 *     generating script is tests/golden/make_golden.py),
 *   - the survey digests of SURVEY.md Appendix C.
 *
 * Reference citations use p/ = /root/reference/proj/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Word layout, p/core/include/ndactor/wah.hpp:15-31. */
#define WO_CHUNK_BITS 31u
#define WO_FILL 0x80000000u
#define WO_ONES 0x40000000u
#define WO_LEN_MASK 0x3fffffffu
#define WO_LIT_MASK 0x7fffffffu

typedef struct {
  uint32_t value, offset, length;
} wo_entry; /* IndexEntry, wah.hpp:78-82 */

/* ------------------------------------------------------------------ */
/* growable u32 vector                                                 */

typedef struct {
  uint32_t *p;
  uint64_t n, cap;
} u32vec;

static void vpush(u32vec *v, uint32_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 64;
    v->p = (uint32_t *)realloc(v->p, v->cap * sizeof(uint32_t));
  }
  v->p[v->n++] = x;
}

/* ------------------------------------------------------------------ */
/* CanonicalWriter, p/core/include/ndactor/wah.hpp:36-74                */

typedef struct {
  u32vec *out;
  int run_ones;
  uint64_t run_len;
} wo_writer;

static void w_flush(wo_writer *w) { /* wah.hpp:64-70 */
  while (w->run_len > 0) {
    uint32_t l = w->run_len > WO_LEN_MASK ? WO_LEN_MASK : (uint32_t)w->run_len;
    vpush(w->out, WO_FILL | (w->run_ones ? WO_ONES : 0u) | l);
    w->run_len -= l;
  }
}

static void w_uniform(wo_writer *w, int ones, uint64_t count) { /* :48-53 */
  if (count == 0) return;
  if (w->run_len > 0 && w->run_ones != ones) w_flush(w);
  w->run_ones = ones;
  w->run_len += count;
}

static void w_chunk(wo_writer *w, uint32_t bits) { /* :39-46 */
  if (bits == 0)
    w_uniform(w, 0, 1);
  else if (bits == WO_LIT_MASK)
    w_uniform(w, 1, 1);
  else {
    w_flush(w);
    vpush(w->out, bits);
  }
}

/* Exposed writer for the CanonicalWriter known-answer tests
 * (p/tests/test_wah.cpp:79-101).  ops: kind 0 = chunk(arg), 1 = uniform(false,
 * arg), 2 = uniform(true, arg).  Returns the number of words written to out
 * (at most cap are stored). */
uint64_t wo_writer_ops(const uint32_t *kinds, const uint64_t *args,
                       uint64_t nops, uint32_t *out, uint64_t cap) {
  u32vec v = {0, 0, 0};
  wo_writer w = {&v, 0, 0};
  for (uint64_t i = 0; i < nops; ++i) {
    if (kinds[i] == 0)
      w_chunk(&w, (uint32_t)args[i]);
    else
      w_uniform(&w, kinds[i] == 2, args[i]);
  }
  w_flush(&w);
  uint64_t n = v.n;
  if (out) memcpy(out, v.p, (n < cap ? n : cap) * sizeof(uint32_t));
  free(v.p);
  return n;
}

/* ------------------------------------------------------------------ */
/* encode / decode, p/core/src/wah_words.cpp:8-47                       */

/* bits: one byte per bit (0/1).  Returns word count, stores up to cap. */
uint64_t wo_encode(const uint8_t *bits, uint64_t n, uint32_t *out,
                   uint64_t cap) {
  u32vec v = {0, 0, 0};
  wo_writer w = {&v, 0, 0};
  for (uint64_t base = 0; base < n; base += WO_CHUNK_BITS) {
    uint32_t chunk = 0;
    uint64_t top = base + WO_CHUNK_BITS < n ? base + WO_CHUNK_BITS : n;
    for (uint64_t i = base; i < top; ++i)
      if (bits[i]) chunk |= 1u << (i - base);
    w_chunk(&w, chunk);
  }
  w_flush(&w);
  uint64_t m = v.n;
  if (out) memcpy(out, v.p, (m < cap ? m : cap) * sizeof(uint32_t));
  free(v.p);
  return m;
}

/* Returns the number of bits covered (stores up to cap), or -1 for a
 * zero-length fill (wah_words.cpp:26). */
int64_t wo_decode(const uint32_t *words, uint64_t nw, uint8_t *bits,
                  uint64_t cap) {
  uint64_t n = 0;
  for (uint64_t k = 0; k < nw; ++k) {
    uint32_t word = words[k];
    if (word & WO_FILL) {
      uint64_t len = word & WO_LEN_MASK;
      if (len == 0) return -1;
      uint8_t b = (word & WO_ONES) ? 1 : 0;
      for (uint64_t i = 0; i < len * WO_CHUNK_BITS; ++i, ++n)
        if (bits && n < cap) bits[n] = b;
    } else {
      for (uint32_t i = 0; i < WO_CHUNK_BITS; ++i, ++n)
        if (bits && n < cap) bits[n] = (word >> i) & 1u;
    }
  }
  return (int64_t)n;
}

/* decode_exact, wah_words.cpp:34-47.  Returns 0 on success, or an error
 * code: 1 zero-length fill, 2 fewer bits than expected, 3 a whole chunk of
 * slack, 4 padding bit set. */
int wo_decode_exact(const uint32_t *words, uint64_t nw, uint64_t n,
                    uint8_t *bits) {
  int64_t covered = wo_decode(words, nw, 0, 0);
  if (covered < 0) return 1;
  if ((uint64_t)covered < n) return 2;
  if ((uint64_t)covered >= n + WO_CHUNK_BITS) return 3;
  uint8_t *all = (uint8_t *)malloc((size_t)covered + 1);
  wo_decode(words, nw, all, (uint64_t)covered);
  for (uint64_t i = n; i < (uint64_t)covered; ++i)
    if (all[i]) {
      free(all);
      return 4;
    }
  if (bits) memcpy(bits, all, n);
  free(all);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Stable ordering of rows by value.                                   */
/* The reference uses std::stable_sort of row ids by value             */
/* (wah_words.cpp:55-60); any stable sort gives the same permutation,   */
/* here a byte-wise LSD counting sort (skipping constant bytes).        */

static uint32_t *stable_order(const uint32_t *values, uint64_t n) {
  uint32_t *a = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *b = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) a[i] = (uint32_t)i;
  uint32_t and_all = 0xffffffffu, or_all = 0;
  for (uint64_t i = 0; i < n; ++i) {
    and_all &= values[i];
    or_all |= values[i];
  }
  for (int shift = 0; shift < 32; shift += 8) {
    if ((((and_all ^ or_all) >> shift) & 0xffu) == 0) continue; /* constant */
    uint64_t cnt[257];
    memset(cnt, 0, sizeof cnt);
    for (uint64_t i = 0; i < n; ++i) cnt[((values[a[i]] >> shift) & 0xffu) + 1]++;
    for (int d = 0; d < 256; ++d) cnt[d + 1] += cnt[d];
    for (uint64_t i = 0; i < n; ++i) {
      uint32_t r = a[i];
      b[cnt[(values[r] >> shift) & 0xffu]++] = r;
    }
    uint32_t *t = a;
    a = b;
    b = t;
  }
  free(b);
  return a;
}

/* Stable sort of (key, payload) pairs by key, the semantics of
 * wah::sort_pairs (wah_radix.cpp:16-127, checked against std::stable_sort
 * at p/tests/test_wah_device.cpp:89-100). */
void wo_sort_pairs(uint32_t *keys, uint32_t *payloads, uint64_t n) {
  uint32_t *order = stable_order(keys, n);
  uint32_t *k2 = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *p2 = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) {
    k2[i] = keys[order[i]];
    p2[i] = payloads[order[i]];
  }
  memcpy(keys, k2, n * sizeof(uint32_t));
  memcpy(payloads, p2, n * sizeof(uint32_t));
  free(k2);
  free(p2);
  free(order);
}

/* ------------------------------------------------------------------ */
/* reference_index, p/core/src/wah_words.cpp:49-91                      */

typedef struct {
  uint32_t row_count;
  u32vec words;
  wo_entry *entries;
  uint64_t d, dcap;
} wo_index;

wo_index *wo_reference_index(const uint32_t *values, uint64_t n) {
  wo_index *idx = (wo_index *)calloc(1, sizeof(wo_index));
  idx->row_count = (uint32_t)n;
  uint32_t *order = stable_order(values, n); /* :55-60 */
  uint64_t i = 0;
  while (i < n) { /* :62-89 */
    uint32_t value = values[order[i]];
    uint64_t start = idx->words.n;
    wo_writer w = {&idx->words, 0, 0};
    uint32_t chunk = 0, chunk_idx = 0;
    int open = 0;
    for (; i < n && values[order[i]] == value; ++i) {
      uint32_t row = order[i];
      uint32_t c = row / WO_CHUNK_BITS;
      if (open && c != chunk_idx) {
        w_chunk(&w, chunk);
        w_uniform(&w, 0, (uint64_t)(c - chunk_idx - 1));
        chunk = 0;
      } else if (!open) {
        w_uniform(&w, 0, c);
      }
      chunk |= 1u << (row % WO_CHUNK_BITS);
      chunk_idx = c;
      open = 1;
    }
    w_chunk(&w, chunk);
    w_flush(&w);
    if (idx->d == idx->dcap) {
      idx->dcap = idx->dcap ? idx->dcap * 2 : 64;
      idx->entries =
          (wo_entry *)realloc(idx->entries, idx->dcap * sizeof(wo_entry));
    }
    wo_entry e = {value, (uint32_t)start, (uint32_t)(idx->words.n - start)};
    idx->entries[idx->d++] = e;
  }
  free(order);
  return idx;
}

uint32_t wo_index_row_count(const wo_index *x) { return x->row_count; }
uint64_t wo_index_num_entries(const wo_index *x) { return x->d; }
uint64_t wo_index_num_words(const wo_index *x) { return x->words.n; }
const wo_entry *wo_index_entries(const wo_index *x) { return x->entries; }
const uint32_t *wo_index_words(const wo_index *x) { return x->words.p; }
void wo_index_free(wo_index *x) {
  if (!x) return;
  free(x->words.p);
  free(x->entries);
  free(x);
}

/* ------------------------------------------------------------------ */
/* "WAH1" serialization, p/core/src/wah_index_io.cpp:30-44, and the     */
/* FNV-1a-64 digest of it.                       */

typedef struct {
  uint64_t h;
} fnv;
static void fnv_bytes(fnv *f, const uint8_t *p, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    f->h ^= p[i];
    f->h *= 1099511628211ull;
  }
}
static void fnv_u32(fnv *f, uint32_t v) {
  uint8_t b[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16),
                  (uint8_t)(v >> 24)};
  fnv_bytes(f, b, 4);
}

/* Digest of serialize_index(idx) given its three parts. */
uint64_t wo_digest_parts(uint32_t row_count, const wo_entry *entries,
                         uint64_t d, const uint32_t *words, uint64_t w) {
  fnv f = {1469598103934665603ull};
  const uint8_t magic[4] = {'W', 'A', 'H', '1'};
  fnv_bytes(&f, magic, 4);
  fnv_u32(&f, row_count);
  fnv_u32(&f, (uint32_t)d);
  fnv_u32(&f, (uint32_t)w);
  for (uint64_t i = 0; i < d; ++i) {
    fnv_u32(&f, entries[i].value);
    fnv_u32(&f, entries[i].offset);
    fnv_u32(&f, entries[i].length);
  }
  for (uint64_t i = 0; i < w; ++i) fnv_u32(&f, words[i]);
  return f.h;
}

uint64_t wo_index_digest(const wo_index *x) {
  return wo_digest_parts(x->row_count, x->entries, x->d, x->words.p,
                         x->words.n);
}

/* serialize_index into out (16 + 12 D + 4 W bytes); returns the size. */
uint64_t wo_serialize(const wo_index *x, uint8_t *out, uint64_t cap) {
  uint64_t need = 16 + 12 * x->d + 4 * x->words.n;
  if (!out || cap < need) return need;
  uint8_t *p = out;
#define PUT(v)                                   \
  do {                                           \
    uint32_t _v = (v);                           \
    p[0] = (uint8_t)_v;                          \
    p[1] = (uint8_t)(_v >> 8);                   \
    p[2] = (uint8_t)(_v >> 16);                  \
    p[3] = (uint8_t)(_v >> 24);                  \
    p += 4;                                      \
  } while (0)
  memcpy(p, "WAH1", 4);
  p += 4;
  PUT(x->row_count);
  PUT((uint32_t)x->d);
  PUT((uint32_t)x->words.n);
  for (uint64_t i = 0; i < x->d; ++i) {
    PUT(x->entries[i].value);
    PUT(x->entries[i].offset);
    PUT(x->entries[i].length);
  }
  for (uint64_t i = 0; i < x->words.n; ++i) PUT(x->words.p[i]);
#undef PUT
  return need;
}

/* ------------------------------------------------------------------ */
/* rows_for, p/core/src/wah_words.cpp:93-103.  Returns the number of   */
/* rows (stores up to cap).                                             */

uint64_t wo_rows_for(const wo_index *x, uint32_t value, uint32_t *rows,
                     uint64_t cap) {
  uint64_t lo = 0, hi = x->d;
  while (lo < hi) { /* lower_bound on value */
    uint64_t mid = (lo + hi) / 2;
    if (x->entries[mid].value < value)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo == x->d || x->entries[lo].value != value) return 0;
  const wo_entry *e = &x->entries[lo];
  uint64_t row = 0, n = 0;
  for (uint32_t k = 0; k < e->length; ++k) {
    uint32_t word = x->words.p[e->offset + k];
    if (word & WO_FILL) {
      uint64_t len = (uint64_t)(word & WO_LEN_MASK) * WO_CHUNK_BITS;
      if (word & WO_ONES)
        for (uint64_t i = 0; i < len; ++i, ++n)
          if (rows && n < cap) rows[n] = (uint32_t)(row + i);
      row += len;
    } else {
      for (uint32_t i = 0; i < WO_CHUNK_BITS; ++i)
        if ((word >> i) & 1u) {
          if (rows && n < cap) rows[n] = (uint32_t)(row + i);
          ++n;
        }
      row += WO_CHUNK_BITS;
    }
  }
  return n;
}

/* ------------------------------------------------------------------ */
/* Device-primitive oracles (p/tests/test_wah_device.cpp:25-41).        */

/* scan_oracle, test_wah_device.cpp:25-33 (u32 wrap-around arithmetic). */
void wo_scan_exclusive(const uint32_t *in, uint32_t *out, uint64_t n) {
  uint32_t running = 0;
  for (uint64_t i = 0; i < n; ++i) {
    out[i] = running;
    running += in[i];
  }
}

/* filter_nonzero, test_wah_device.cpp:35-41: the meaning of the fused
 * compaction stages (wah_stages.cpp:158-163). */
uint64_t wo_filter_nonzero(const uint32_t *in, uint64_t n, uint32_t *out) {
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (in[i]) out[m++] = in[i];
  return m;
}
