/*
 * pipedp_cuda.h -- C ABI of the B200-native pipedp solvers (sm_100a).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams travel as `void*` = cudaStream_t).  Every entry point is the body
 * a reference FFI would bind in place of the reference's C++ solver
 * (/root/reference/proj, cited per function).  All host-buffer entry points
 * validate with the reference's exact rules and error codes BEFORE touching a
 * device and never fall back to a CPU path: with no usable GPU they return
 * PIPEDP_ERR_NO_DEVICE.
 *
 * Status codes: 0 = ok; 1 + index of the reference `errc` enumerator
 * (error.hpp:8-20) for validation errors; >= 100 for device errors.
 * pipedp_last_error() returns the message of the calling thread's last error,
 * prefixed like the reference's Error::what() ("InitLengthMismatch: ...").
 * Every function is thread-safe; concurrent callers get independent streams
 * and buffers.
 */
#ifndef PIPEDP_CUDA_H
#define PIPEDP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
enum {
  PIPEDP_OK = 0,
  PIPEDP_E_NON_DECREASING_OFFSETS = 1, /* errc::non_decreasing_offsets */
  PIPEDP_E_NON_POSITIVE_OFFSET = 2,    /* errc::non_positive_offset */
  PIPEDP_E_INIT_LENGTH_MISMATCH = 3,   /* errc::init_length_mismatch */
  PIPEDP_E_TABLE_TOO_SMALL = 4,        /* errc::table_too_small */
  PIPEDP_E_COORD_OUT_OF_RANGE = 5,     /* errc::coord_out_of_range */
  PIPEDP_E_ADDRESS_OUT_OF_RANGE = 6,   /* errc::address_out_of_range */
  PIPEDP_E_BASE_CELL_HAS_NO_DEPS = 7,  /* errc::base_cell_has_no_deps */
  PIPEDP_E_TOO_LARGE_FOR_BRUTE = 8,    /* errc::too_large_for_brute_force */
  PIPEDP_E_STALL_LIVELOCK = 9,         /* errc::stall_livelock */
  PIPEDP_E_WEIGHT_OVERFLOW = 10,       /* errc::weight_overflow */
  PIPEDP_E_INVALID_PARAMS = 11,        /* errc::invalid_params */
  PIPEDP_ERR_CUDA = 100,
  PIPEDP_ERR_NO_DEVICE = 101,
  PIPEDP_ERR_OUT_OF_MEMORY = 102,
  PIPEDP_ERR_UNSUPPORTED = 103
};

/* Semigroup kinds, OpKind order (semigroup.hpp:13). */
enum { PIPEDP_OP_MIN = 0, PIPEDP_OP_MAX = 1, PIPEDP_OP_SATURATING_ADD = 2, PIPEDP_OP_MODULAR_ADD = 3 };

/* S-DP methods (pipedp_sdp_plan_set_method / pipedp_sdp_solve_method) */
enum {
  PIPEDP_SDP_PIPELINE = 0,  /* the pipelined kernels (default) */
  PIPEDP_SDP_PREFIX = 1,    /* the paper's tournament per cell, O(n log k) steps */
  PIPEDP_SDP_NAIVE = 2      /* the paper's naive k-1-thread method with conflicts, O(nk) */
};

/* MCM kernels */
enum {
  PIPEDP_MCM_AUTO = 0,       /* shared-memory CTA for small n / batches, tiled pipeline otherwise */
  PIPEDP_MCM_WAVEFRONT = 1,  /* multi-SM dataflow pipeline, table in HBM */
  PIPEDP_MCM_SMEM = 2,       /* one CTA, table in shared memory (small n) */
  PIPEDP_MCM_TOURNAMENT = 3, /* the paper's O(n^2 log n) comparison kernel */
  PIPEDP_MCM_TILED = 4       /* blocked pipeline: 64x64 tiles, TMA-staged, split-K far terms */
};

/* McmMode (mcm_pipeline.hpp:88) */
enum { PIPEDP_MCM_PAPER_LITERAL = 0, PIPEDP_MCM_STALL_ON_HAZARD = 1 };

const char* pipedp_last_error(void);
const char* pipedp_version(void);
/* number of usable sm_100 devices (0 without a GPU; never fails) */
int32_t pipedp_device_count(void);

/* ---- host-only helpers (no device needed) -------------------------------- */
/* validate(SdpInstance) -- sdp.cpp:10-32 */
int32_t pipedp_sdp_validate(const int64_t* offsets, int64_t k, int64_t init_len, int64_t n);
/* validate(McmInstance) -- mcm.cpp:11-28 */
int32_t pipedp_mcm_validate(const int64_t* dims, int64_t dims_len);
/* table_digest over a cells array -- table.cpp:12-25 */
uint64_t pipedp_table_digest(const int64_t* cells, int64_t count);
/* generate_sdp -- generate.cpp:21-47 (offsets_out: k, init_out: a_1 <= init_cap) */
int32_t pipedp_generate_sdp(int64_t n, int64_t k, int32_t op, uint64_t seed, int32_t consecutive,
                            int64_t a1_cap, int64_t* offsets_out, int64_t* init_out,
                            int64_t init_cap, int64_t* a1_out);
/* generate_mcm -- generate.cpp:49-60 (dims_out: n+1) */
int32_t pipedp_generate_mcm(int64_t n, uint64_t seed, int64_t dims_min, int64_t dims_max,
                            int64_t* dims_out);
/* Batched generators for the batch driver: instance i = generate_* with seed
 * seed0 + i.  S-DP: offsets_out [count*k], init_out [count*a_1] (a_1 = a1_cap,
 * 2k when a1_cap == 0, or k when consecutive; returned in *a1_out).
 * MCM: dims_out [count*(n+1)]. */
int32_t pipedp_generate_sdp_batch(int64_t n, int64_t k, uint64_t seed0, int64_t count,
                                  int32_t consecutive, int64_t a1_cap, int64_t* offsets_out,
                                  int64_t* init_out, int64_t* a1_out);
int32_t pipedp_generate_mcm_batch(int64_t n, uint64_t seed0, int64_t count, int64_t dims_min,
                                  int64_t dims_max, int64_t* dims_out);

/* ---- S-DP, host buffers ---------------------------------------------------
 * Replaces the table computation of solve_sequential (sdp.cpp:84-89),
 * solve_prefix_parallel (sdp.cpp:91-100), solve_naive_parallel
 * (sdp.cpp:102-111) and solve_sdp_pipeline (sdp_pipeline.cpp:34-44).
 * cells_out: n entries; filled_out (nullable): n entries, all set to 1. */
int32_t pipedp_sdp_solve(const int64_t* offsets, int64_t k, const int64_t* init,
                         int64_t init_len, int64_t n, int32_t op, int64_t* cells_out,
                         uint8_t* filled_out);

/* solve_prefix_parallel / solve_naive_parallel (sdp.cpp:91-111) with the
 * paper's own methods on the device (method = PIPEDP_SDP_PREFIX / _NAIVE);
 * same table as pipedp_sdp_solve. */
int32_t pipedp_sdp_solve_method(const int64_t* offsets, int64_t k, const int64_t* init,
                                int64_t init_len, int64_t n, int32_t op, int32_t method,
                                int64_t* cells_out, uint8_t* filled_out);

/* Batch of independent instances sharing n, k and a_1 (SoA: offsets
 * [batch*k], init [batch*a_1], cells_out [batch*n]).  No reference
 * counterpart (the reference loops serially, commands.cpp:480-507); each
 * instance has solve_sequential's semantics.  device < 0: current device. */
int32_t pipedp_sdp_solve_batch(int64_t batch, int64_t n, int64_t k, int64_t a1,
                               const int64_t* offsets, const int64_t* init, int32_t op,
                               int64_t* cells_out, int32_t device);

/* ---- S-DP, device-resident plans (inputs already in HBM) ------------------ */
typedef struct pipedp_sdp_plan* pipedp_sdp_plan_t;
/* h_offsets / h_init: HOST copies of every instance's offsets and init values,
 * used for validation and value-width planning; uploaded once. */
int32_t pipedp_sdp_plan_create(int64_t batch, int64_t n, int64_t k, int64_t a1,
                               const int64_t* h_offsets, const int64_t* h_init, int32_t op,
                               int32_t device, pipedp_sdp_plan_t* plan_out);
/* d_init: device copy of init ([batch*a1]); d_cells: device table ([batch*n]);
 * stream: cudaStream_t or NULL.  Asynchronous. */
int32_t pipedp_sdp_plan_execute(pipedp_sdp_plan_t plan, const int64_t* d_init, int64_t* d_cells,
                                void* stream);
/* kernel name, value width (32/64) and kernel launches per execute */
int32_t pipedp_sdp_plan_describe(pipedp_sdp_plan_t plan, char* name, size_t name_cap,
                                 int32_t* value_bits, int32_t* launches);
/* switch a single-instance plan to the paper's prefix / naive method */
int32_t pipedp_sdp_plan_set_method(pipedp_sdp_plan_t plan, int32_t method);
/* chunked mode phase timing (CUDA events on the execute stream): set_timing
 * resets and enables; phase_ms returns the accumulated milliseconds of
 * [0] matrix powers, [1] entry-state chain, [2] chunk batch over `runs` executes */
int32_t pipedp_sdp_plan_set_timing(pipedp_sdp_plan_t plan, int32_t on);
int32_t pipedp_sdp_plan_phase_ms(pipedp_sdp_plan_t plan, double* out3, int64_t* runs);
int32_t pipedp_sdp_plan_destroy(pipedp_sdp_plan_t plan);

/* ---- MCM, host buffers ------------------------------------------------------
 * solve_mcm_sequential (mcm.cpp:85-110): cells_out / split_out (nullable) /
 * filled_out (nullable) have cell_count(n)+1 entries in the reference's
 * 1-based diagonal-major layout. */
int32_t pipedp_mcm_solve(const int64_t* dims, int64_t dims_len, int32_t kernel,
                         int64_t* cells_out, uint8_t* filled_out, int64_t* split_out);
/* solve_mcm_pipeline (mcm_pipeline.cpp:32-47): exact lock-step engine
 * semantics of McmProgram for both McmMode values: same table, same
 * steps_executed, same stall_iterations. */
int32_t pipedp_mcm_pipeline(const int64_t* dims, int64_t dims_len, int32_t mode,
                            int64_t* cells_out, uint8_t* filled_out, int64_t* steps_out,
                            int64_t* stall_iterations_out);
/* ---- lock-step engine with device-side trace analyses -------------------
 * The reference engine (engine.hpp:134-433) running McmProgram
 * (mcm_pipeline.hpp:22-84) or SdpProgram (sdp_pipeline.hpp:16-58) on the GPU,
 * iteration for iteration.  flags: PIPEDP_ENGINE_TRACE collects the access
 * records (PipelineTrace::records, canonical record_less order);
 * PIPEDP_ENGINE_ANALYSIS computes, on the device while the schedule runs,
 * the conflict groups of detect_conflicts (analysis.cpp:31-70) and the hazard
 * records of detect_hazards (analysis.cpp:72-103) without materialising the
 * trace.  The run handle owns the results until pipedp_engine_free. */
enum { PIPEDP_ENGINE_TRACE = 1, PIPEDP_ENGINE_ANALYSIS = 2 };
typedef struct pipedp_engine_run* pipedp_engine_t;
typedef struct {
  int64_t first_head;        /* head_range().first */
  int64_t steps_executed;    /* iterations, stalls included */
  int64_t stall_iterations;  /* steps_executed - head count */
  int64_t records;           /* access records (TRACE) */
  int64_t hazards;           /* hazard records (ANALYSIS) */
  int64_t conflict_groups;   /* conflict groups (ANALYSIS) */
  int64_t conflict_lanes;    /* lanes over all groups */
  int64_t max_group_size;    /* ConflictReport::max_group_size (1 if none) */
  int64_t stall_heads;       /* PipelineTrace::stall_heads entries */
} pipedp_engine_summary;
/* mode: PIPEDP_MCM_PAPER_LITERAL / PIPEDP_MCM_STALL_ON_HAZARD; cells_out
 * (nullable) cell_count(n)+1 entries */
int32_t pipedp_mcm_engine(const int64_t* dims, int64_t dims_len, int32_t mode, int32_t flags,
                          int64_t* cells_out, pipedp_engine_summary* summary, pipedp_engine_t* run_out);
/* SdpProgram has no stall mode in the reference (lock-step only); cells_out
 * (nullable) n entries */
int32_t pipedp_sdp_engine(const int64_t* offsets, int64_t k, const int64_t* init, int64_t init_len,
                          int64_t n, int32_t op, int32_t flags, int64_t* cells_out,
                          pipedp_engine_summary* summary, pipedp_engine_t* run_out);
/* records in record_less order: head, substep, lane, kind (0 read, 1 write), address */
int32_t pipedp_engine_records(pipedp_engine_t run, int64_t* head, int32_t* substep, int32_t* lane,
                              int32_t* kind, int64_t* address);
/* hazards [hazards][6]: head, substep, lane, address, finalization head, finalization substep,
 * sorted as detect_hazards sorts them */
int32_t pipedp_engine_hazards(pipedp_engine_t run, int64_t* out);
/* conflicts: groups [conflict_groups][4] head, substep, kind, address (detect_conflicts order);
 * group_sizes [conflict_groups]; lanes [conflict_lanes] concatenated, ascending per group;
 * per_step_cost [steps_executed] */
int32_t pipedp_engine_conflicts(pipedp_engine_t run, int64_t* groups, int32_t* group_sizes, int32_t* lanes,
                                int32_t* per_step_cost);
int32_t pipedp_engine_stall_heads(pipedp_engine_t run, int64_t* out);
void pipedp_engine_free(pipedp_engine_t run);

/* solve_mcm_bruteforce (mcm.cpp:130-138): the reference's independent oracle
 * (enumeration of every parenthesisation, n <= 12, else TooLargeForBruteForce),
 * run on the device. */
int32_t pipedp_mcm_bruteforce(const int64_t* dims, int64_t dims_len, int64_t* out);
/* batch of independent MCM instances of equal n (dims [batch*(n+1)],
 * cells/split [batch*(cell_count(n)+1)]) */
int32_t pipedp_mcm_solve_batch(int64_t batch, int64_t n, const int64_t* dims, int64_t* cells_out,
                               int64_t* split_out, int32_t device);

/* ---- MCM, device-resident plans ------------------------------------------ */
typedef struct pipedp_mcm_plan* pipedp_mcm_plan_t;
int32_t pipedp_mcm_plan_create(int64_t batch, int64_t n, const int64_t* h_dims, int32_t kernel,
                               int32_t device, pipedp_mcm_plan_t* plan_out);
/* d_cells / d_split: [batch*(cell_count(n)+1)].  Asynchronous (CUDA-graph
 * capturable): the 32-bit attempt raises a device-side overflow flag, and the
 * unpacked / 64-bit reruns queued behind it on `stream` run only if it did.
 * (Batches whose 64-bit table does not fit shared memory synchronise `stream`
 * once instead.)  describe() reports the value width that stood, waiting for
 * the last execute if needed. */
int32_t pipedp_mcm_plan_execute(pipedp_mcm_plan_t plan, int64_t* d_cells, int64_t* d_split,
                                void* stream);
int32_t pipedp_mcm_plan_describe(pipedp_mcm_plan_t plan, char* name, size_t name_cap,
                                 int32_t* value_bits, int32_t* launches);
int32_t pipedp_mcm_plan_destroy(pipedp_mcm_plan_t plan);

/* ---- device utilities -------------------------------------------------------- */
/* FNV-1a table_digest of ntables consecutive tables of `count` cells each. */
int32_t pipedp_digest_device(const int64_t* d_tables, int64_t count, int64_t ntables,
                             uint64_t* d_digests, void* stream);
/* Dependency-chain step microbenchmark: ns per warp-shuffle hand-off step of
 * the S-DP chain warp for `op` at `value_bits`. */
int32_t pipedp_chain_step_ns(int32_t op, int32_t value_bits, int32_t device, double* ns_out,
                             double* sm_clock_mhz_out);

/* Hardware floor of the S-DP dependency chain: latency of one dependent (x)
 * at `value_bits` in a single-thread register chain (ns and SM cycles). */
int32_t pipedp_op_latency_ns(int32_t op, int32_t value_bits, int32_t device, double* ns_out,
                             double* cycles_out);

/* Role-level cycle counters of the profiling build (-DPIPEDP_PROFILE,
 * tools/build_profile.sh); returns PIPEDP_ERR_UNSUPPORTED otherwise. */
int32_t pipedp_profile_read(uint64_t* out, int32_t count, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* PIPEDP_CUDA_H */
