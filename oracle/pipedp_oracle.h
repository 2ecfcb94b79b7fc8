/*
 * pipedp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference library `pipedp` (arxiv/paper_2008_01938,
 * /root/reference/proj) for the hot path: the semigroup catalog, the S-DP
 * sequential solver, the MCM sequential solver with its split table, the MCM
 * pipeline lock-step engine semantics (paper-literal and stall-on-hazard), the
 * seeded instance generators and the FNV-1a table digest.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this code, and only as the checker / CPU baseline.  The product path
 * (paper_2008_01938_b200) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref, compiled from the reference sources by
 * oracle/Makefile) and against the SPEC known-answer vectors and the golden
 * digests in tests/golden/.
 *
 * Error returns follow the reference `errc` enumeration (error.hpp:8-20) as
 * 1 + enumerator index; 0 means success.
 */
#ifndef PIPEDP_ORACLE_H
#define PIPEDP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* OpKind order follows semigroup.hpp:13 */
enum { OR_OP_MIN = 0, OR_OP_MAX = 1, OR_OP_SAT_ADD = 2, OR_OP_MOD_ADD = 3 };

int64_t or_apply(int op, int64_t a, int64_t b);

int or_sdp_validate(const int64_t* offsets, int64_t k, int64_t init_len, int64_t n);
/* cells_out/filled_out: n entries each (filled_out may be NULL) */
int or_sdp_solve(const int64_t* offsets, int64_t k, const int64_t* init, int64_t init_len,
                 int64_t n, int op, int64_t* cells_out, uint8_t* filled_out);

int or_mcm_validate(const int64_t* dims, int64_t dims_len);
int64_t or_mcm_cell_count(int64_t n);
int64_t or_mcm_lin(int64_t row, int64_t col, int64_t n); /* -1 when out of range */
int or_mcm_coord(int64_t address, int64_t n, int64_t* row, int64_t* col);
/* cells_out/filled_out/split_out: cell_count(n)+1 entries (filled/split may be NULL) */
int or_mcm_solve(const int64_t* dims, int64_t dims_len, int64_t* cells_out, uint8_t* filled_out,
                 int64_t* split_out);
/* Lock-step engine semantics of McmProgram (mode 0 paper_literal, 1 stall_on_hazard). */
int or_mcm_pipeline(const int64_t* dims, int64_t dims_len, int mode, int64_t* cells_out,
                    uint8_t* filled_out, int64_t* steps_out, int64_t* stall_iterations_out);
int64_t or_mcm_bruteforce(const int64_t* dims, int64_t dims_len); /* -(errc+1) on error */

uint64_t or_table_digest(const int64_t* cells, int64_t count);

/* std::mt19937_64 (seeded with a single 64-bit value) restated */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_mt64;
void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);

/* generate_sdp: offsets_out has k entries; init_out has a_1 entries (a_1 = cap or k). */
int or_generate_sdp(int64_t n, int64_t k, uint64_t seed, int consecutive, int64_t a1_cap,
                    int64_t* offsets_out, int64_t* init_out, int64_t init_cap);
int or_generate_mcm(int64_t n, uint64_t seed, int64_t dims_min, int64_t dims_max,
                    int64_t* dims_out);

#ifdef __cplusplus
}
#endif
#endif
