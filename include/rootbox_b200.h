/*
 * rootbox_b200.h -- C ABI of the B200 (sm_100a) engine for the rootbox solver
 * hot path: global interval branch-and-bound with Hansen-Sengupta contraction.
 *
 * The library (paper_1802_00330_b200/librootbox_b200.so) replaces the
 * internals of the reference entry point
 *
 *     rootbox.bnb.solve(s: PolySystem, cfg: SolverConfig) -> SolveResult
 *                                       (rootbox/bnb.py:224-354, __init__.py:12)
 *
 * and its two per-round operators
 *
 *     bnb._chunk_batch((cs, lo, hi)) -> (lo, hi)                 (bnb.py:161-165)
 *     bnb._hs_pass(s, jac, lo, hi, contract_output) -> (lo, hi, cert)  (bnb.py:190-218)
 *
 * Plain C types only: pointers, sizes, IEEE binary64.  Box arrays crossing
 * the ABI are row-major (N x n), exactly the numpy layout of the reference
 * (_batch.py:9).  Every call is synchronous w.r.t. the caller's buffers,
 * thread-safe per handle (calls on one handle serialise), and does not hold
 * the Python GIL when invoked through ctypes.
 *
 * Return codes: 0 = ok; negative = error, message in rb_last_error().
 */
#ifndef ROOTBOX_B200_H
#define ROOTBOX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RB_OK 0
#define RB_ERR_ARG -1      /* invalid argument (reference: ValueError)        */
#define RB_ERR_CUDA -2     /* CUDA runtime error                             */
#define RB_ERR_NOMEM -3    /* device memory exhausted (reference: MemoryError) */
#define RB_ERR_LIMIT -4    /* system exceeds the compiled table limits        */
#define RB_ERR_STATE -5    /* call out of sequence (e.g. fetch before solve)  */

#define RB_MAX_DIM 16

/* status codes == bnb.py:40-42 */
#define RB_NO_REAL_SOLUTION 0 /* "no_real_solution" */
#define RB_WIDTH_REACHED 1    /* "width_reached"    */
#define RB_BUDGET_EXHAUSTED 2 /* "budget_exhausted" */

/* A compiled polynomial system (the flat form of _batch.compile_system,
 * _batch.py:156-164, extended with the Jacobian of PolySystem.jacobian,
 * poly.py:284-291).  Polynomials 0..n-1 are F in equation order; polynomial
 * n + i*n + j is dF_i/dx_j.  Terms of each polynomial are in the canonical
 * order of poly.py:159 (descending (degree, exponents)); factors of a term
 * are its nonzero (variable, exponent) pairs in ascending variable order. */
typedef struct rb_system {
    int32_t n;                /* dimension, 1..RB_MAX_DIM                 */
    int32_t n_polys;          /* n + n*n                                  */
    const int32_t* poly_off;  /* [n_polys + 1] term ranges                */
    const double* coeff;      /* [T] coefficients                         */
    const int32_t* fac_off;   /* [T + 1] factor ranges                    */
    const uint8_t* fac_var;   /* [Fc] variable index                      */
    const uint8_t* fac_exp;   /* [Fc] exponent >= 1                       */
    const double* init_lo;    /* [n] initial box (PolySystem.initial_box) */
    const double* init_hi;    /* [n]                                      */
} rb_system;

/* SolverConfig (bnb.py:49-86).  None is encoded as noted. worker_count,
 * batch_size and engine do not change results (bnb.py:9-11) and are not
 * passed. */
typedef struct rb_config {
    double target_width;      /* <= 0 or NaN: None (2^-10 x initial width) */
    int32_t hs_enable_round;  /* < 0: None                                  */
    int32_t hs_contract;      /* bool                                       */
    double hs_enable_width;   /* NaN: None                                  */
    int32_t max_rounds;
    int32_t exact_round_dedup;/* 1: exact per-round dedup (bnb.py:322-326)  */
    int64_t max_boxes;
    double max_seconds;       /* < 0 or NaN: None                           */
} rb_config;

/* RoundStats (bnb.py:89-96) plus engine counters. */
typedef struct rb_round_stats {
    int32_t round;
    int32_t hs_on;
    int64_t boxes_in;
    int64_t boxes_after_filter;
    int64_t boxes_after_hs;
    double width;
    double elapsed_seconds;
    int64_t children;          /* active parents x 2^n evaluated by the filter */
    int64_t hs_calls;          /* boxes contracted                              */
    int64_t filter_ops;        /* algorithmic directed ops in the filter        */
    int64_t hs_ops;            /* algorithmic directed ops in HS                */
    int64_t dups;              /* exact duplicates removed                      */
    int64_t exact_boxes;       /* boxes evaluated on the exact (guarded) path   */
    double filter_ms;          /* device time of the filter kernel(s)           */
    double hs_ms;              /* device time of the HS kernel(s)               */
    double classify_ms;        /* device time of the classify/compaction kernel */
    int64_t classify_bytes;    /* algorithmic HBM bytes of the classify kernel  */
    int64_t attempts;          /* 1 + redos after a buffer had to grow          */
} rb_round_stats;

typedef struct rb_result_info {
    int32_t status;            /* RB_NO_REAL_SOLUTION / RB_WIDTH_REACHED / RB_BUDGET_EXHAUSTED */
    int32_t nrounds;
    int64_t nboxes;
    double solve_seconds;      /* host wall time inside rb_solve */
    double device_ms;          /* CUDA-event time on the engine stream, first to last op */
    int64_t kernel_launches;   /* engine kernels launched by this solve (CUB sort passes excluded) */
} rb_result_info;

typedef struct rb_handle rb_handle;

/* Library version string. */
const char* rb_version(void);

/* Number of visible CUDA devices (>= 0), or a negative error code. */
int rb_device_count(void);

/* Create an engine for one system on one CUDA device (one handle per GPU /
 * per rank).  Copies the tables; the caller keeps ownership of `sys`.
 * Replaces: compile_system + PolySystem.jacobian setup in bnb.solve
 * (bnb.py:236-238). */
int rb_create(const rb_system* sys, int device, rb_handle** out);

/* Run bnb.solve (bnb.py:224-354) on the device.  Results stay on the device
 * until rb_fetch.  Replaces the whole round loop. */
int rb_solve(rb_handle* h, const rb_config* cfg, rb_result_info* info);

/* Copy the last solve's result into caller-allocated host buffers:
 * lo/hi [nboxes x n] row-major in canonical order (_batch.canonical_order,
 * _batch.py:244-250), cert/unsplit [nboxes] (RootBox.certified/unsplittable,
 * bnb.py:99-103), stats [nrounds].  Any pointer may be NULL to skip it. */
int rb_fetch(rb_handle* h, double* lo, double* hi, uint8_t* cert, uint8_t* unsplit,
             rb_round_stats* stats);

/* bnb._chunk_batch (bnb.py:161-165) on P parents (row-major P x n, all
 * non-degenerate): writes the feasible children, in the reference's order
 * (parents in input order, children in binary-counting order), to olo/ohi
 * (capacity `cap` rows); *M receives the survivor count even if > cap. */
int rb_filter(rb_handle* h, const double* plo, const double* phi, int64_t P, double* olo,
              double* ohi, int64_t cap, int64_t* M);

/* bnb._hs_pass (bnb.py:190-218) on M rows: writes the surviving rows in the
 * reference's order (forks as two consecutive rows) and their certified flags;
 * *M2 receives the output count even if > cap. */
int rb_hs(rb_handle* h, const double* lo, const double* hi, int64_t M, int contract_output,
          double* olo, double* ohi, uint8_t* cert, int64_t cap, int64_t* M2);

/* hansen.krawczyk (hansen.py:141-170) on M boxes (row-major M x n): the
 * Krawczyk operator K(X) intersected with X.  ok[r] = 0 where the reference
 * returns None (singular midpoint Jacobian or empty intersection); those rows
 * of olo/ohi are NaN.  Shares the HS preconditioning kernels (x, A J, A F(x)). */
int rb_krawczyk(rb_handle* h, const double* lo, const double* hi, int64_t M, double* olo, double* ohi,
                uint8_t* ok);

/* Last error message of this handle (or of the last failed rb_create when h is NULL). */
const char* rb_last_error(rb_handle* h);

void rb_destroy(rb_handle* h);

/* ---- sharded (multi-GPU) round protocol -------------------------------------
 * One handle per rank; the host performs the tiny per-round exchanges
 * (torch.distributed / NCCL) between the calls.  The same kernels as rb_solve. */

/* Load a shard of the frontier (row-major, host) as the current round input. */
int rb_shard_load(rb_handle* h, const double* lo, const double* hi, const uint8_t* cert,
                  const uint8_t* unsplit, int64_t N, double target_width);

/* Round part 1: classify + bisect + filter.  Outputs the local survivor
 * count and max child width (for the global HS trigger, bnb.py:289-296). */
int rb_round_filter(rb_handle* h, int32_t round_no, int64_t* carried, int64_t* survivors,
                    double* child_width, int64_t* children);

/* Round part 2: HS (hs_on decided globally by the caller).  The new frontier is
 * carried + HS rows, NOT yet deduplicated: route rows to their owners first
 * (rb_shard_partition + exchange), then rb_shard_dedup.  Outputs the local
 * frontier size and max width. */
int rb_round_hs(rb_handle* h, int32_t hs_on, int32_t hs_contract, int64_t* n_out,
                double* width, int64_t* hs_calls);

/* Copy `count` rows starting at `start` of the current frontier to host
 * buffers (any order; used for rebalancing and the final gather). */
int rb_shard_export(rb_handle* h, int64_t start, int64_t count, double* lo, double* hi,
                    uint8_t* cert, uint8_t* unsplit);

/* Keep only rows [0, keep) of the current frontier and append `count` rows
 * from host buffers (rebalancing receive). */
int rb_shard_import(rb_handle* h, int64_t keep, const double* lo, const double* hi,
                    const uint8_t* cert, const uint8_t* unsplit, int64_t count);

/* Current frontier size of the shard. */
int64_t rb_shard_size(rb_handle* h);

/* Reorder the shard owner-major: counts[r] rows (in rank order) belong to rank
 * r = row_hash(row) % world, the ownership that makes per-shard dedup global
 * (_batch.dedup_sorted, _batch.py:253-266). */
int rb_shard_partition(rb_handle* h, int32_t world, int64_t* counts);

/* Exact dedup of the shard with flag OR (after the owner exchange); outputs the
 * number of rows removed and the shard's max RN width (bnb.py:329). */
int rb_shard_dedup(rb_handle* h, int64_t* dups, double* width);

/* Device-pointer variants of export/import (row-major, e.g. torch CUDA tensors
 * exchanged with NCCL all_to_all).  Synchronous on the engine stream. */
int rb_shard_export_device(rb_handle* h, int64_t start, int64_t count, double* dlo, double* dhi, uint8_t* dcert,
                           uint8_t* duns);
int rb_shard_import_device(rb_handle* h, int64_t keep, const double* dlo, const double* dhi, const uint8_t* dcert,
                           const uint8_t* duns, int64_t count);

/* Frontier routing between shards: only rows with a component at
 * most 64 ulps wide can have an exact duplicate on another shard, so only those go
 * to their hash owner; the rest stay, except the surplus rows a rebalancing plan
 * moves.  rb_shard_route_count: thin rows per owner rank (thin_counts [world]) and
 * the number of other rows (*nonthin).  rb_shard_route (after route_count):
 * move[d] non-thin rows go to rank d (move[rank] ignored); reorders the shard as
 * [own rows | rows for rank 0 | rank 1 | ...] and returns the row count per
 * destination (send_counts[rank] = rows that stay).  The caller then exports rows
 * [send_counts[rank], size) for the exchange and imports the received rows with
 * keep = send_counts[rank].  Replaces the per-round row movement of the
 * reference's thread pool (bnb.py:183-187, 271-313), which has no shards. */
int rb_shard_route_count(rb_handle* h, int32_t world, int64_t* thin_counts, int64_t* nonthin);
int rb_shard_route(rb_handle* h, int32_t world, int32_t rank, const int64_t* move, int64_t* send_counts);

/* Canonical order (_batch.canonical_order, _batch.py:244-250) of the shard's rows
 * into the result buffers, so rb_fetch returns them (the gathered final frontier of
 * a sharded solve, bnb.py:322-326); *nboxes receives the row count. */
int rb_shard_finalize(rb_handle* h, int64_t* nboxes);

/* Kernels launched by the handle since its last rb_solve (the shard protocol's calls
 * accumulate): the launch count of a sharded solve, for the bench record. */
int64_t rb_kernel_launches(rb_handle* h);

/* Engine tuning knobs (results never depend on them):
 *   "filter_tab"  1: tabulated per-parent term filter (k_filter_tab, a block per
 *                 parent) when the tables fit; 0: direct per-child evaluation (k_filter).
 *                 Default: on for n >= 10 (2^n >= 1024 children per parent).
 *   "filter_wt"   1: warp-tabulated filter (k_filter_wt, a warp per parent or per 1024 of its
 *                 children, 5 <= n <= 16),
 *                 ahead of "filter_tab"; 0: off; -1: the default, on unless more than
 *                 half of the equations have tables above 2^(min(n, 10) - 2) entries
 *                 (such equations are evaluated per child inside k_filter_wt).
 *   "force_exact" 0 (default): exponent guards pick IEEE directed rounding wherever it
 *                 provably equals the reference; 1: every guard fails, so every box
 *                 runs the Exact policy (the reference's error-free transformations,
 *                 interval.py:66-205).  For the parity tests of that path.
 *   "graph"       1 (default): rounds whose worst case fits the survivor buffer run
 *                 in one CUDA graph (device-side WHILE loop, no host round trip);
 *                 0: host-driven rounds (per-kernel CUDA-event timings in the stats).
 *   "device_timing" 1 (default): rb_solve waits for the stream and reports CUDA-event
 *                 device time in rb_result_info.device_ms; 0: a solve the round graph
 *                 finishes returns as soon as its results are visible in mapped host
 *                 memory (completion flag), device_ms = -1.
 *   "jconst"      1 (default): J entries without a variable ([c, c] for every box) are
 *                 neither stored by k_hs_eval nor loaded by k_hs_lin_tps; 0: every
 *                 entry through the HS scratch.
 *   "hs_fused"    1 (default): k_hs_fused (one warp per box) for small survivor counts,
 *                 k_hs_eval / k_hs_lin_tps / k_hs_sweep above; 0: the three kernels
 *                 always; 2: k_hs_fused always.
 *   "lin_tpb"     Gauss-Jordan of the three-kernel HS: 2 (default) one thread per box,
 *                 tableau in shared memory (n <= 8; two threads per box for 8 < n <= 12);
 *                 3 two threads per box at every n <= 12; 1 tableau in registers
 *                 (n <= 8); 0 G lanes per box.
 *   "hs_tile"     1: k_hs_tile (a tile's whole HS in shared memory, n <= 8); 0 (default).
 *   "codegen"     1 (default): system-specialised (NVRTC) kernels once compiled;
 *                 0: table kernels.  "codegen_wait" 1: block until the compile is done.
 *   "stream_parents" P > 0: every host-driven round processes its parents in chunks
 *                 of P (otherwise only rounds whose survivors exceed the buffer do).
 *   "mem_budget_mb" engine memory budget (0: the default, a share of free memory).
 *   Round-graph structure (dev knobs, defaults measured best): "pingpong", "graph_cf",
 *   "append_dedup", "graph_unroll", "graph_prologue", "graph_fused_only", "hs_cond",
 *   "small_rounds" (persistent small-round kernel, with "mk_bps" / "mk_cap"),
 *   "tail_blocks_x4", "pdl". */
int rb_set_option(rb_handle* h, const char* key, int64_t value);

/* ---- system-specialised kernels ----------------------------------------------
 * rb_create compiles the system's F equations into straight-line filter kernels
 * (NVRTC, sm_100a; replaces the per-term walk over compile_system's tables,
 * _batch.py:144-186, with identical operations) and caches the cubin on disk.
 * rb_codegen_prepare fills that cache without a device (e.g. at build time);
 * on success err receives the cache key.
 * rb_codegen_active returns 1 when the handle runs the specialised kernels, 0
 * when it runs the table kernels (reason in why).  RB_CODEGEN=0 disables it. */
int rb_codegen_prepare(const rb_system* sys, char* err, int64_t err_len);
int rb_codegen_active(rb_handle* h, char* why, int64_t why_len);

/* ---- post-processing -----------------------------------
 * Backtracking merge of a solve result: snap_to_grid of every box, then
 * merge_to_width (rootbox/backtrack.py:118-242), in exact integer arithmetic on
 * the host.  lo/hi [N x n] row-major, cert [N]; stop_width < 0 or NaN = None.
 * Outputs the merged boxes in canonical order (out_lo/out_hi [M x n], out_cert
 * [M]) and the merge levels (levels [K x 2] = (width, count)); *M and *K get
 * the true sizes even when they exceed cap / cap_levels.  Errors (the
 * reference's NotOnGrid) return RB_ERR_ARG with the message in err. */
int rb_merge(int n, const double* init_lo, const double* init_hi, const double* lo, const double* hi,
             const uint8_t* cert, int64_t N, double stop_width, int stop_on_plateau, double* out_lo,
             double* out_hi, uint8_t* out_cert, int64_t cap, int64_t* M, double* levels, int64_t cap_levels,
             int64_t* K, char* err, int64_t err_len);

/* The same merge on `device`: snapping per box in 128-bit
 * integers, then per merge level a radix sort of the (level, index) keys, exact-duplicate
 * merge with flag OR, nested-cell absorption and parent index halving on the GPU.
 * Same arguments and results as rb_merge.  Applies when every initial width is a power of
 * two and every snapped level is at most 53; otherwise returns RB_ERR_LIMIT (message in
 * err) and the caller runs rb_merge. */
int rb_merge_device(int device, int n, const double* init_lo, const double* init_hi, const double* lo,
                    const double* hi, const uint8_t* cert, int64_t N, double stop_width, int stop_on_plateau,
                    double* out_lo, double* out_hi, uint8_t* out_cert, int64_t cap, int64_t* M, double* levels,
                    int64_t cap_levels, int64_t* K, char* err, int64_t err_len);

/* ---- interval-layer known-answer hook (tests) --------------------------------
 * m operand pairs through one device operation of interval.cuh on `device`
 * (host arrays in and out).  x = [xl, xh], y = [yl, yh]; policy 0 = Fast (IEEE
 * directed instructions), 1 = Exact (the reference's emulation,
 * interval.py:66-205), 2 = guarded (what the kernels run: Fast when the exponent
 * guard proves it equal to Exact, else Exact).
 *   op 0..5   scalar _add_rd/_add_ru/_mul_rd/_mul_ru/_div_rd/_div_ru (xl, yl) -> o0
 *   op 10     interval product x*y -> [o0, o1]       (interval.py:322-326)
 *   op 11     recip(x) -> [o0, o1]                    (interval.py:347-351)
 *   op 12     mid(x) -> o0                            (interval.py:269-281)
 *   op 20+k   x**k (k = 0..9) -> [o0, o1]              (interval.py:328-345)
 *   op 40     div_extended(x, y) -> kind, [o0, o1], [o2, o3]  (interval.py:394-432);
 *             policy 0 = div_extended_fast (reciprocal fast path), 1 = forced Exact,
 *             2 = div_extended with the guarded product
 * Replaces no reference entry point: it exposes the device twins of the
 * reference's scalar/interval functions to tests/test_gpu_exact.py. */
int rb_interval_kat(int device, int op, int policy, int64_t m, const double* xl, const double* xh,
                    const double* yl, const double* yh, double* o0, double* o1, double* o2, double* o3,
                    int8_t* kind);

/* ---- report writer ---------------------------------------
 * The raw-box sections of the reference's reports for N boxes (lo/hi [N x n],
 * cert [N]): fmt 0 = the elements of RunReport.to_json's "roots" list exactly as
 * json.dumps(indent=2) lays them out inside the report object (cli.py:54-86),
 * fmt 1 = RunReport.to_csv's rows (cli.py:88-100); floats as Python's repr().
 * Writes at most cap bytes to out (may be null); *len receives the full length. */
int rb_format_boxes(int n, const double* lo, const double* hi, const uint8_t* cert, int64_t N, int fmt, char* out,
                    int64_t cap, int64_t* len);

/* ---- measurement utility ----------------------------------------------------
 * Measured throughput of the FP64 pipe on `device` for the directed-rounding
 * instructions the engine issues (DMUL.RM/RP, DADD.RM/RP; one op each), in
 * ops/s: the roofline denominator for the filter and HS kernels. */
int rb_fp64_peak(int device, double* ops_per_second);

#ifdef __cplusplus
}
#endif
#endif /* ROOTBOX_B200_H */
