/*
 * pipedp_oracle.c -- TEST INFRASTRUCTURE ONLY (see pipedp_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Every function cites the
 * reference file:line (under /root/reference/proj) whose behaviour it restates.
 * Nothing here is shipped: the CUDA product never links this file.
 */
#include "pipedp_oracle.h"

#include <limits.h>
#include <stdlib.h>
#include <string.h>

/* errc order: error.hpp:8-20 */
enum {
  E_NON_DECREASING = 1,
  E_NON_POSITIVE = 2,
  E_INIT_LEN = 3,
  E_TABLE_SMALL = 4,
  E_COORD = 5,
  E_ADDRESS = 6,
  E_BASE_CELL = 7,
  E_BRUTE = 8,
  E_LIVELOCK = 9,
  E_WEIGHT = 10,
  E_INVALID = 11,
};

static const int64_t kModulus = 2147483647; /* semigroup.hpp:15 */

/* semigroup.cpp:12-19 -- clamp toward the sign of b on overflow */
static int64_t sat_add(int64_t a, int64_t b) {
  int64_t out;
  if (__builtin_add_overflow(a, b, &out)) return b > 0 ? INT64_MAX : INT64_MIN;
  return out;
}

/* semigroup.cpp:21-24 */
static int64_t norm_mod(int64_t a) {
  int64_t r = a % kModulus;
  return r < 0 ? r + kModulus : r;
}

/* semigroup.cpp:28-40 */
int64_t or_apply(int op, int64_t a, int64_t b) {
  switch (op) {
    case OR_OP_MIN: return a < b ? a : b;
    case OR_OP_MAX: return a > b ? a : b;
    case OR_OP_SAT_ADD: return sat_add(a, b);
    default: return (norm_mod(a) + norm_mod(b)) % kModulus;
  }
}

/* sdp.cpp:10-32 */
int or_sdp_validate(const int64_t* offs, int64_t k, int64_t init_len, int64_t n) {
  if (k <= 0) return E_INVALID;
  for (int64_t i = 0; i < k; ++i) {
    if (offs[i] <= 0) return E_NON_POSITIVE;
    if (i > 0 && offs[i - 1] <= offs[i]) return E_NON_DECREASING;
  }
  if (init_len != offs[0]) return E_INIT_LEN;
  if (n <= offs[0]) return E_TABLE_SMALL;
  return 0;
}

/* sdp.cpp:34-41 (initial_table) + sdp.cpp:48-60 (fill_table) + sdp.cpp:84-89 */
int or_sdp_solve(const int64_t* offs, int64_t k, const int64_t* init, int64_t init_len, int64_t n,
                 int op, int64_t* cells, uint8_t* filled) {
  int rc = or_sdp_validate(offs, k, init_len, n);
  if (rc) return rc;
  const int64_t a1 = offs[0];
  memset(cells, 0, sizeof(int64_t) * (size_t)n);
  memcpy(cells, init, sizeof(int64_t) * (size_t)a1);
  for (int64_t i = a1; i < n; ++i) {
    int64_t acc = cells[i - a1];
    for (int64_t j = 1; j < k; ++j) acc = or_apply(op, acc, cells[i - offs[j]]);
    cells[i] = acc;
  }
  if (filled) memset(filled, 1, (size_t)n);
  return 0;
}

/* mcm.cpp:11-28.  The overflow product is evaluated left to right with
 * two's-complement wrap, which is what the reference's signed expression
 * compiles to on gcc/x86-64. */
int or_mcm_validate(const int64_t* dims, int64_t len) {
  if (len < 2) return E_INVALID;
  int64_t max_dim = 1;
  for (int64_t i = 0; i < len; ++i) {
    if (dims[i] < 1) return E_INVALID;
    if (dims[i] > max_dim) max_dim = dims[i];
  }
  const int64_t n = len - 1;
  if (max_dim > 1000000) return E_WEIGHT;
  uint64_t p = (uint64_t)n * (uint64_t)max_dim;
  p *= (uint64_t)max_dim;
  p *= (uint64_t)max_dim;
  if ((int64_t)p > ((int64_t)1 << 61)) return E_WEIGHT;
  return 0;
}

int64_t or_mcm_cell_count(int64_t n) { return n * (n + 1) / 2; } /* mcm.hpp:31 */

/* mcm.cpp:30-37 */
int64_t or_mcm_lin(int64_t row, int64_t col, int64_t n) {
  if (row < 1 || row > col || col > n) return -1;
  const int64_t d = col - row;
  return d * n - d * (d - 1) / 2 + row;
}

/* mcm.cpp:39-53 */
int or_mcm_coord(int64_t address, int64_t n, int64_t* row, int64_t* col) {
  if (address < 1 || address > or_mcm_cell_count(n)) return E_ADDRESS;
  int64_t d = 0, base = 0;
  while (address > base + (n - d)) {
    base += n - d;
    ++d;
  }
  *row = address - base;
  *col = *row + d;
  return 0;
}

/* mcm.cpp:77-83 (initial table) + mcm.cpp:85-110 (ascending-address DP,
 * strict '<' keeps the first minimal term; split = 1-based term index) with
 * the terms of mcm.cpp:55-75 generated inline. */
int or_mcm_solve(const int64_t* p, int64_t len, int64_t* cells, uint8_t* filled, int64_t* split) {
  int rc = or_mcm_validate(p, len);
  if (rc) return rc;
  const int64_t n = len - 1;
  const int64_t cc = or_mcm_cell_count(n);
  memset(cells, 0, sizeof(int64_t) * (size_t)(cc + 1));
  if (split) memset(split, 0, sizeof(int64_t) * (size_t)(cc + 1));
  int64_t addr = n + 1;
  for (int64_t d = 1; d < n; ++d) {
    for (int64_t r = 1; r + d <= n; ++r, ++addr) {
      const int64_t c = r + d;
      int64_t best = INT64_MAX, best_j = 0;
      for (int64_t j = 1; j <= d; ++j) {
        const int64_t left = cells[or_mcm_lin(r, r + j - 1, n)];
        const int64_t right = cells[or_mcm_lin(r + j, c, n)];
        const int64_t cost = left + right + p[r - 1] * p[r + j - 1] * p[c];
        if (cost < best) {
          best = cost;
          best_j = j;
        }
      }
      cells[addr] = best;
      if (split) split[addr] = best_j;
    }
  }
  if (filled) memset(filled, 1, (size_t)(cc + 1));
  return 0;
}

/* mcm.cpp:116-127 */
static int64_t enum_min(const int64_t* p, int64_t r, int64_t c) {
  if (r == c) return 0;
  int64_t best = INT64_MAX;
  for (int64_t s = r; s < c; ++s) {
    const int64_t cost = enum_min(p, r, s) + enum_min(p, s + 1, c) + p[r - 1] * p[s] * p[c];
    if (cost < best) best = cost;
  }
  return best;
}

/* mcm.cpp:131-138 */
int64_t or_mcm_bruteforce(const int64_t* p, int64_t len) {
  int rc = or_mcm_validate(p, len);
  if (rc) return -rc;
  if (len - 1 > 12) return -E_BRUTE;
  return enum_min(p, 1, len - 1);
}

/*
 * Lock-step engine (engine.hpp:134-433) running McmProgram
 * (mcm_pipeline.hpp:22-84, mcm_pipeline.cpp:11-47).
 *  - heads [n+1, cc+n-2]; lane j at vhead h owns cell h-j+1 when that cell is
 *    computed and j <= D(cell) (mcm_pipeline.hpp:30-49);
 *  - substeps 1-3 only read, substep 4 writes, so every read sees the table as
 *    of the start of the iteration (engine.hpp:124-126, 364-397);
 *  - stall mode (engine.hpp:128-133, 287-326): a lane executes only when its
 *    left/right operands have received all their writes and all earlier terms of
 *    its own cell have been written; held lanes keep their vhead
 *    (engine.hpp:404-415);
 *  - livelock guards of engine.hpp:352-362.
 */
int or_mcm_pipeline(const int64_t* p, int64_t len, int mode, int64_t* cells, uint8_t* filled,
                    int64_t* steps_out, int64_t* stall_out) {
  int rc = or_mcm_validate(p, len);
  if (rc) return rc;
  const int64_t n = len - 1;
  if (n < 2) return E_INVALID; /* mcm_pipeline.cpp:28 */
  const int64_t cc = or_mcm_cell_count(n);
  const int64_t first = n + 1, last = cc + n - 2;
  const int64_t lanes = n - 1;
  const int stall = mode == 1;

  int64_t* row = calloc((size_t)(cc + 1), sizeof(int64_t));
  int64_t* dg = calloc((size_t)(cc + 1), sizeof(int64_t));
  int64_t* done_w = calloc((size_t)(cc + 1), sizeof(int64_t));
  int64_t* vhead = malloc(sizeof(int64_t) * (size_t)(lanes + 1));
  uint8_t* ldone = calloc((size_t)(lanes + 1), 1);
  uint8_t* exec = calloc((size_t)(lanes + 1), 1);
  int64_t* wval = malloc(sizeof(int64_t) * (size_t)(lanes + 1));
  int64_t* waddr = malloc(sizeof(int64_t) * (size_t)(lanes + 1));
  if (!row || !dg || !done_w || !vhead || !ldone || !exec || !wval || !waddr) {
    rc = E_INVALID;
    goto out;
  }
  {
    int64_t a = 1;
    for (int64_t d = 0; d < n; ++d)
      for (int64_t r = 1; r + d <= n; ++r, ++a) {
        row[a] = r;
        dg[a] = d;
      }
  }
  memset(cells, 0, sizeof(int64_t) * (size_t)(cc + 1));
  if (filled) {
    memset(filled, 0, (size_t)(cc + 1));
    for (int64_t i = 0; i <= n; ++i) filled[i] = 1;
  }
  for (int64_t j = 1; j <= lanes; ++j) vhead[j] = first;

  const int64_t budget = (last - first + 1) * (lanes + 2) + 16;
  int64_t steps = 0;
  for (;;) {
    int all_done = 1, any_exec = 0;
    for (int64_t j = 1; j <= lanes; ++j) {
      exec[j] = 0;
      if (ldone[j]) continue;
      all_done = 0;
      const int64_t cell = vhead[j] - j + 1;
      const int active = cell >= n + 1 && cell <= cc && j <= dg[cell];
      if (!active) {
        exec[j] = 2; /* inactive slot consumes the iteration */
        any_exec = 1;
        continue;
      }
      int ready = 1;
      if (stall) {
        const int64_t r = row[cell], c = r + dg[cell];
        const int64_t left = or_mcm_lin(r, r + j - 1, n), right = or_mcm_lin(r + j, c, n);
        if (left > n && done_w[left] < dg[left]) ready = 0;
        if (right > n && done_w[right] < dg[right]) ready = 0;
        if (done_w[cell] != j - 1) ready = 0;
      }
      if (ready) {
        exec[j] = 1;
        any_exec = 1;
      }
    }
    if (all_done) break;
    if (!any_exec || steps > budget) {
      rc = E_LIVELOCK;
      goto out;
    }
    int64_t nw = 0;
    for (int64_t j = 1; j <= lanes; ++j) {
      if (exec[j] != 1) continue;
      const int64_t cell = vhead[j] - j + 1;
      const int64_t r = row[cell], c = r + dg[cell];
      const int64_t vs = cells[or_mcm_lin(r, r + j - 1, n)] + cells[or_mcm_lin(r + j, c, n)] +
                         p[r - 1] * p[r + j - 1] * p[c];
      waddr[nw] = cell;
      wval[nw++] = j == 1 ? vs : (cells[cell] < vs ? cells[cell] : vs);
    }
    for (int64_t w = 0; w < nw; ++w) {
      cells[waddr[w]] = wval[w];
      if (filled) filled[waddr[w]] = 1;
      done_w[waddr[w]]++;
    }
    for (int64_t j = 1; j <= lanes; ++j) {
      if (ldone[j] || !exec[j]) continue;
      if (++vhead[j] > last) ldone[j] = 1;
    }
    ++steps;
  }
  if (steps_out) *steps_out = steps;
  if (stall_out) *stall_out = steps - (last - first + 1);
out:
  free(row);
  free(dg);
  free(done_w);
  free(vhead);
  free(ldone);
  free(exec);
  free(wval);
  free(waddr);
  return rc;
}

/* table.cpp:12-25 */
uint64_t or_table_digest(const int64_t* cells, int64_t count) {
  uint64_t h = 14695981039346656037ull;
  const uint64_t prime = 1099511628211ull;
#define MIX(v)                                   \
  do {                                           \
    uint64_t _v = (uint64_t)(v);                 \
    for (int b = 0; b < 8; ++b) {                \
      h ^= (_v >> (8 * b)) & 0xffu;              \
      h *= prime;                                \
    }                                            \
  } while (0)
  MIX(count);
  for (int64_t i = 0; i < count; ++i) MIX(cells[i]);
#undef MIX
  return h;
}

/* std::mt19937_64 as pinned by the C++ standard (used by generate.cpp:26, 55) */
void or_mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

uint64_t or_mt64_next(or_mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ull : 0);
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* generate.cpp:15-17 */
static int64_t bounded(or_mt64* g, int64_t lo, int64_t hi) {
  return lo + (int64_t)(or_mt64_next(g) % (uint64_t)(hi - lo + 1));
}

static int cmp_desc(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}

/* generate.cpp:21-47.  The distinct set is an open-addressing table; only the
 * membership test matters, the final order comes from the descending sort. */
int or_generate_sdp(int64_t n, int64_t k, uint64_t seed, int consecutive, int64_t a1_cap,
                    int64_t* offs, int64_t* init, int64_t init_cap) {
  if (k < 1) return E_INVALID;
  or_mt64 g;
  or_mt64_seed(&g, seed);
  if (consecutive) {
    for (int64_t i = 0; i < k; ++i) offs[i] = k - i;
  } else {
    const int64_t cap = a1_cap > 0 ? a1_cap : 2 * k;
    if (cap < k) return E_INVALID;
    uint64_t tsize = 16;
    while (tsize < (uint64_t)(4 * k)) tsize <<= 1;
    int64_t* table = malloc(sizeof(int64_t) * tsize);
    if (!table) return E_INVALID;
    for (uint64_t i = 0; i < tsize; ++i) table[i] = 0;
    int64_t count = 0;
#define INSERT(v)                                                          \
  do {                                                                     \
    const int64_t _v = (v);                                                \
    uint64_t _h = ((uint64_t)_v * 0x9E3779B97F4A7C15ull) & (tsize - 1);    \
    while (table[_h] != 0 && table[_h] != _v) _h = (_h + 1) & (tsize - 1); \
    if (table[_h] == 0) {                                                  \
      table[_h] = _v;                                                      \
      offs[count++] = _v;                                                  \
    }                                                                      \
  } while (0)
    INSERT(cap);
    while (count < k) INSERT(bounded(&g, 1, cap - 1));
#undef INSERT
    free(table);
    qsort(offs, (size_t)k, sizeof(int64_t), cmp_desc);
  }
  const int64_t a1 = offs[0];
  if (n <= a1) return E_INVALID;
  if (init_cap < a1) return E_INVALID;
  for (int64_t i = 0; i < a1; ++i) init[i] = bounded(&g, 0, ((int64_t)1 << 20) - 1);
  return or_sdp_validate(offs, k, a1, n);
}

/* generate.cpp:49-60 */
int or_generate_mcm(int64_t n, uint64_t seed, int64_t lo, int64_t hi, int64_t* dims) {
  if (n < 1) return E_INVALID;
  if (lo < 1 || lo > hi) return E_INVALID;
  or_mt64 g;
  or_mt64_seed(&g, seed);
  for (int64_t i = 0; i <= n; ++i) dims[i] = bounded(&g, lo, hi);
  return or_mcm_validate(dims, n + 1);
}
