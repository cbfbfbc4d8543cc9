// engine.cuh -- host-side engine state and the per-dimension launchers.
//
// Shared by engine.cu (orchestration + C ABI) and kinst.cu, which explicitly
// instantiates the launchers (and with them every kernel) for a few dimensions
// per translation unit so the sm_100a build runs in parallel.
#pragma once
#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <future>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/rootbox_b200.h"
#include "codegen.h"
#include "kernels.cuh"

using namespace rb;

#define RB_VERSION "rootbox_b200 0.1.0 (sm_100a)"

namespace rbe {

// Stream-ordered allocations from the handle's memory pool (memory is retained
// across rounds and solves, so growth never stalls the device); set per API call.
inline thread_local cudaMemPool_t t_pool = nullptr;
inline thread_local cudaStream_t t_stream = nullptr;

inline void dfree(void* p) {
    if (!p) return;
    if (t_pool) cudaFreeAsync(p, t_stream);
    else cudaFree(p);
}


struct DevFront {
    Front f{};
    int n = 0;
    void release() {
        dfree(f.lo);
        dfree(f.hi);
        dfree(f.cert);
        dfree(f.unsplit);
        f = Front{};
    }
};

struct CudaError {
    cudaError_t e;
    const char* what;
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError{e, what};
}

struct ArgError {
    int code;
    std::string msg;
};

}  // namespace rbe

using namespace rbe;

struct rb_handle {
    std::mutex mu;
    int dev = 0;
    int n = 0;
    int sms = 148;
    cudaStream_t st = nullptr;
    cudaMemPool_t pool = nullptr;
    cudaEvent_t ev[8] = {};
    int64_t launches = 0;
    TabMeta meta{};
    uint8_t* d_tab = nullptr;
    std::vector<double> init_lo, init_hi;

    DevFront F[2];
    int cur = 0;
    int64_t n_cur = 0;       // rows in F[cur]
    uint32_t* parents = nullptr;
    int64_t cap_par = 0;
    SBuf S{};
    Counters* d_ctr = nullptr;
    Counters* h_ctr = nullptr;  // pinned
    int64_t* d_tags = nullptr;
    int64_t cap_tags = 0;
    // dedup scratch (table kept all-zero between rounds)
    unsigned* d_table = nullptr;
    size_t table_slots = 0;
    unsigned* d_slot = nullptr;
    uint8_t* d_dead = nullptr;
    int64_t cap_dead = 0;
    // capacity prediction from the previous round
    size_t mem_budget = 0;     // bytes the engine may hold
    size_t mem_budget_default = 0;
    // sort scratch
    void* d_cub = nullptr;
    size_t cub_bytes = 0;
    unsigned long long* d_keys[2] = {nullptr, nullptr};
    unsigned* d_perm[2] = {nullptr, nullptr};
    int64_t cap_sort = 0;
    // result (device, row-major, canonical order)
    double* r_lo = nullptr;
    double* r_hi = nullptr;
    uint8_t* r_cert = nullptr;
    uint8_t* r_uns = nullptr;
    int64_t r_n = 0;
    bool r_on_host = false;  // small results are ordered on the host
    bool r_ready = false;    // the result buffers already hold this solve's result
    int64_t cap_r = 0;
    // mapped pinned memory the round graph reads its start state from and writes back to
    uint8_t* pin = nullptr;      // mapped pinned block holding h_ctr, h_state, hx, stats and result rows
    size_t pin_bytes = 0;
    DevRoundStats* hx_stats_own = nullptr;
    HostX* hx = nullptr;
    HostX* hx_dev = nullptr;
    DevRoundStats* hx_stats = nullptr;
    DevRoundStats* hx_stats_dev = nullptr;
    int cap_hx_stats = 0;
    double *hx_lo = nullptr, *hx_hi = nullptr, *hx_lo_dev = nullptr, *hx_hi_dev = nullptr;
    uint8_t *hx_c = nullptr, *hx_u = nullptr, *hx_c_dev = nullptr, *hx_u_dev = nullptr;
    std::vector<double> hr_lo, hr_hi;
    std::vector<uint8_t> hr_cert, hr_uns;
    bool have_result = false;
    std::vector<rb_round_stats> stats;
    // adaptive filter equation order (device copy; host mirror for host-driven rounds)
    int* d_order = nullptr;
    int h_order[16] = {};
    // device-resident round loop (CUDA graph with a WHILE node)
    bool use_graph = true;
    DevState* d_state = nullptr;
    DevState* h_state = nullptr;  // pinned
    DevRoundStats* d_rstats = nullptr;
    int cap_rstats = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    std::vector<uintptr_t> graph_key;
    int64_t graph_launches_per_iter = 0;
    int graph_unroll = 6;        // rounds per WHILE iteration of the round graph (measured: 6 > 4 > 2)
    bool graph_fused_only = true;  // round graph: k_hs_fused for every count (no eval/lin/sweep nodes)
    bool graph_cf = true;        // round graph: k_classify_filter instead of k_classify + k_filter
    bool pingpong = true;        // round graph: ping-pong frontiers, round end in k_hs_fused
    bool graph_prologue = true;  // ping-pong round graph: the first U rounds outside the WHILE node
    unsigned long long* d_etable = nullptr;  // epoch dedup table (ping-pong round graph)
    size_t cap_etable = 0;
    unsigned epoch_next = 1;
    int graph_rounds_per_iter = 1;
    bool ev_end_valid = false;   // ev[6] already marks the end of this solve's device work
    double tail_blocks_per_sm = 2.0;  // k_round_tail grid
    // system-specialised filter kernels (codegen.cpp); the table kernels when unavailable
    rbg::SystemTerms terms;
    rbg::Loaded gen;
    bool use_gen = true;
    bool gen_pending = false;                              // compiling in the background
    std::future<std::pair<bool, rbg::Compiled>> gen_job;
    std::string gen_err;
    int gen_cf_bps = 1, gen_filter_bps = 1, gen_hsf_bps = 1, gen_hse_bps = 1, gen_ftab_bps = 1;
    bool append_dedup = true;    // round graph: exact dedup at append time instead of k_dedup_insert
    // sharded protocol state
    double shard_target = 0.0;
    int64_t shard_carried = 0;
    int shard_round = 0;
    int64_t shard_need_f = 0;
    std::string err;
    // launch shapes
    int filter_threads = 256;
    int hs_threads = 128;
    int filter_blocks_per_sm = 1;
    int eval_blocks_per_sm = 1, lin_blocks_per_sm = 1, sweep_blocks_per_sm = 1;
    size_t filter_smem = 0, eval_smem = 0, lin_smem = 0, sweep_smem = 0, ftab_smem = 0;
    int ftab_blocks_per_sm = 1;
    bool use_ftab = true;
    // warp-tabulated filter (k_filter_wt, 5 <= n <= 16): shared memory, blocks per SM (table / specialised)
    bool use_fwt = false, fwt_auto = false;
    // constant entries of J (no variable): mask + values (device), used by the three-kernel
    // HS with k_hs_lin_tps ("jconst" option)
    unsigned long long jmask[4] = {0, 0, 0, 0};
    double* d_jc = nullptr;
    bool jconst = true;
    size_t fwt_smem = 0;
    int fwt_bps = 0, gen_fwt_bps = 0;
    bool hs_fused = true;        // k_hs_fused (tile in shared memory) for small HS batches
    int64_t fused_rows = 0;      // largest HS batch k_hs_fused takes (set from the SM count)
    cudaStream_t st_side = nullptr;  // captures the IF branch of the round graph
    bool hs_cond = true;
    bool pdl = false;            // programmatic dependent launch between round kernels
    bool use_mk = false;         // k_small_rounds (persistent grid) for the smallest rounds (experimental)
    int64_t mk_cap = 1 << 16;    // ... while n_cur * 2^n <= mk_cap
    size_t mk_smem = 0;
    int mk_blocks_per_sm = 0;
    int mk_bps = 1;              // blocks per SM of k_small_rounds
    unsigned* d_bar = nullptr;         // graph: IF node around eval/lin/sweep (else they early-exit)
    // RB_TRACE=1: device timestamps (%globaltimer) at the phase boundaries of every
    // round, printed to stderr after each solve (a profiling aid; adds one tiny launch per phase)
    bool trace = false;
    bool device_timing = true;   // false: a graph-finished solve returns on HostX::done_seq, device_ms = -1
    unsigned long long solve_seq = 0;
    bool graph_fast_return = false;  // this solve's graph ended on done_seq (no stream sync yet)
    double t_solve0 = 0.0;
    unsigned long long* d_trace = nullptr;
    size_t fused_smem = 0;
    int fused_blocks_per_sm = 1;
    HsScratch W{};
    int smem_optin = 48 * 1024;
    // rb_set_option("force_exact"): every exponent guard fails, so the filter, HS and
    // sweep run the Exact policy (interval.cuh) on every box -- the parity tests of
    // that path; the guard constants of build_tables are kept here to restore them
    bool force_exact = false;
    // k_hs_tile (throughput HS, n <= 8): boxes per tile (= threads per block), shared memory,
    // blocks per SM; table-evaluator and specialised builds
    bool hs_tile = false;  // k_hs_tile measured slower than eval/lin/sweep (6 vs 19 warps per SM): off
    int64_t stream_parents = 0;
    // k_hs_lin_tpb (thread per box Gauss-Jordan, n <= 8) in the three-kernel HS
    int lin_tpb = 2;  // 2: shared memory (k_hs_lin_tps, measured best), 1: registers (k_hs_lin_tpb), 0: G lanes per box
    size_t lin_tp2_smem = 0;  // k_hs_lin_tp2 (lin_tpb = 3): two threads per box
    int lin_tp2_bps = 1;
    int lin_tpb_threads = 0, lin_tpb_bps = 1, lin_tps_bps = 1;
    size_t lin_tpb_smem = 0, lin_tps_smem = 0;  // > 0: host-driven rounds stream parents in chunks of this size (tests)
    int tile_tb = 0, gen_tile_tb = 0;
    size_t tile_smem = 0, gen_tile_smem = 0;
    int tile_bps = 1, gen_tile_bps = 1;
    unsigned* d_route = nullptr;   // per-row destination of the shard routing (RouteCountK / RouteK)
    int64_t cap_route = 0;
    int guard_f_ecmin = 0, guard_j_ecmin = 0;
};

struct PoolScope {
    explicit PoolScope(rb_handle* h) {
        t_pool = h->pool;
        t_stream = h->st;
    }
    ~PoolScope() {
        t_pool = nullptr;
        t_stream = nullptr;
    }
};

// ---------------------------------------------------------------- dispatch on n

template <template <int> class F, typename... Args>
static void dispatch_n(int n, Args&&... args) {
    switch (n) {
#define RB_CASE(k) \
    case k: F<k>::run(std::forward<Args>(args)...); break;
        RB_CASE(1) RB_CASE(2) RB_CASE(3) RB_CASE(4) RB_CASE(5) RB_CASE(6) RB_CASE(7) RB_CASE(8)
        RB_CASE(9) RB_CASE(10) RB_CASE(11) RB_CASE(12) RB_CASE(13) RB_CASE(14) RB_CASE(15) RB_CASE(16)
#undef RB_CASE
        default: throw ArgError{RB_ERR_LIMIT, "dimension out of range"};
    }
}

static int grid_for(int64_t work, int threads, int max_blocks) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

// dynamic shared memory limit = opt-in maximum minus the kernel's static shared memory
template <typename K>
static void set_max_dyn_smem(K kernel, int optin) {
    cudaFuncAttributes fa;
    ck(cudaFuncGetAttributes(&fa, kernel), "func attrs");
    ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes),
       "attr");
}

// RB_TRACE buffer layout (words): per-round phase stamps, k_hs_fused block-0 clocks and
// per-block (start, end, smid), k_classify_filter per-block (start, tables, loop, end)
constexpr int kTraceRounds = 256, kTracePhases = 8;
constexpr size_t kTraceHsBlkOff = (size_t)kTraceRounds * kTracePhases + 16 + 32;
constexpr size_t kTraceCfOff = kTraceHsBlkOff + 3 * (size_t)kTraceBlocks;
constexpr size_t kTraceBoxAbs = (size_t)kTraceRounds * kTracePhases + kTraceBoxOff;
static_assert(kTraceBoxAbs == kTraceCfOff + 4 * (size_t)kTraceBlocks, "trace layout");
constexpr size_t kTraceWords = kTraceCfOff + 4 * (size_t)kTraceBlocks + 8 * (size_t)kTraceBoxes;

template <int N>
struct SetupK {
    static void run(rb_handle* h);
};

// Kernel launch on the handle's stream; with h->pdl the launch allows programmatic
// dependent launch (the kernel's blocks start while the previous kernel drains and
// wait in pdl_enter() for its completion).
template <typename... KArgs, typename... Args>
static void klaunch(rb_handle* h, void (*k)(KArgs...), int grid, int block, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = h->pdl ? 1 : 0;
    ck(cudaLaunchKernelEx(&cfg, k, args...), "kernel launch");
}

// launch of a kernel handle (NVRTC-compiled, codegen.cpp) with typed arguments
template <typename... Args>
static void klaunch_k(rb_handle* h, cudaKernel_t k, int grid, int block, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = h->pdl ? 1 : 0;
    void* pa[] = {(void*)&args...};
    ck(cudaLaunchKernelExC(&cfg, (const void*)k, pa), "kernel launch (specialised)");
}

static inline bool gen_on(const rb_handle* h) { return h->use_gen && h->gen.ok; }

// k_hs_tile shape: the tile size (32/64/128 boxes, one thread each) with the most
// resident warps per SM under the tile's shared memory; ties go to the larger tile
template <typename K>
static void choose_tile(rb_handle* h, K kernel, int n, int tab_bytes, int& tb_out, size_t& smem_out, int& bps_out) {
    tb_out = 0;
    int best = 0;
    for (int tb : {128, 64, 32}) {
        const size_t sm = tile_smem_bytes(n, tb, tab_bytes);
        if ((int)sm > h->smem_optin - 256) continue;
        int nb = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, tb, sm), "occ tile");
        if (nb * tb > best) {
            best = nb * tb;
            tb_out = tb;
            smem_out = sm;
            bps_out = std::max(1, nb);
        }
    }
}

// launch attributes of the specialised kernels (same shared-memory layouts as the
// table kernels, whose sizes SetupK computed)
static inline void gen_configure(rb_handle* h) {
    if (!h->gen.ok) return;
    for (cudaKernel_t k : {h->gen.cf, h->gen.filter, h->gen.hs_fused, h->gen.hs_eval, h->gen.hs_tile, h->gen.filter_tab, h->gen.filter_wt}) {
        cudaFuncAttributes fa;
        ck(cudaFuncGetAttributes(&fa, (const void*)k), "gen attrs");
        ck(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                h->smem_optin - (int)fa.sharedSizeBytes), "gen attr");
    }
    int nb = 0;
    const int T = h->hs_threads;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)h->gen.cf, 256, h->filter_smem), "occ");
    h->gen_cf_bps = std::max(1, nb);
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)h->gen.filter, h->filter_threads,
                                                     h->filter_smem), "occ");
    h->gen_filter_bps = std::max(1, nb);
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)h->gen.hs_eval, T, h->eval_smem), "occ");
    h->gen_hse_bps = std::max(1, nb);
    if (h->hs_fused) {
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)h->gen.hs_fused, T, h->fused_smem), "occ");
        h->gen_hsf_bps = std::max(1, nb);
    }
    choose_tile(h, (const void*)h->gen.hs_tile, h->n, 0, h->gen_tile_tb, h->gen_tile_smem, h->gen_tile_bps);
    if (h->meta.ftab && h->ftab_smem <= (size_t)h->smem_optin) {
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)h->gen.filter_tab, 256, h->ftab_smem), "occ");
        h->gen_ftab_bps = std::max(1, nb);
    }
    h->gen_fwt_bps = 0;
    if (h->fwt_bps > 0) {
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)h->gen.filter_wt, 256, h->fwt_smem), "occ");
        h->gen_fwt_bps = nb;
    }
    // the specialised direct filter beats the tabulated one up to n = 8 (katsura6 6.7 vs 9.3 ms, brown8
    // 4.7 vs 6.2, eco8 26.2 vs 25.8 ms); with 2^n >= 1024 children per parent the tables pay
    // (broyden_banded12 3.25 -> 2.35 ms, tools/hs_bench.py --opt filter_tab=1)
    h->use_ftab = h->n >= 10 && h->meta.ftab;
}

template <int N>
struct ClassifyK {
    static void run(rb_handle* h, double target, const DevState* st = nullptr, int64_t bound = -1,
                    DedupCtx dd = DedupCtx{});
};

// classify + filter in one launch (round graph): at most `bound` children
template <int N>
struct ClassifyFilterK {
    static void run(rb_handle* h, DedupCtx dd, int64_t bound);
};

template <int N>
struct AllParentsK {
    static void run(rb_handle* h);
};

template <int N>
struct FilterK {
    static void run(rb_handle* h, int64_t max_parents, int64_t* tags, int64_t p0 = 0, int64_t pcount = -1);
};

// K2a + K2b + K2c over rows [b0, b0 + W.B) of S (n_in read on the device when prm.count_from_ctr)
template <int N>
struct HsK {
    static void run(rb_handle* h, int64_t b0, int64_t n_in, HsParams prm, int64_t* tags, int64_t batch_bound);
};

// tiled K2 (k_hs_tile) over all n_in rows of S (n_in read on the device when prm.count_from_ctr)
template <int N>
struct HsTileK {
    static void run(rb_handle* h, int64_t n_in, HsParams prm, int64_t* tags, int64_t bound);
};

// fused K2 over all n_in rows of S (n_in read on the device when prm.count_from_ctr); `bound`
// is the most rows it can see, which sizes the grid
template <int N>
struct HsFusedK {
    static void run(rb_handle* h, int64_t n_in, HsParams prm, int64_t* tags, int64_t bound);
};

// K2a + K2b + Krawczyk over rows [b0, b_end) of S; results at the same rows of `out`
template <int N>
struct KrawczykK {
    static void run(rb_handle* h, int64_t b0, int64_t b_end, Front out, uint8_t* ok);
};

// persistent small rounds (cooperative: every block resident for the grid barrier)
template <int N>
struct SmallRoundsK {
    static void run(rb_handle* h, const HsParams& prm, bool dedup, int64_t scap, cudaGraphConditionalHandle hw);
};

template <int N>
struct DedupInsertK {
    static void run(rb_handle* h, Front next);
};

// dedup finish + F[1] -> F[0] + round end (graph mode)
template <int N>
struct TailK {
    static void run(rb_handle* h, bool dedup, int64_t bound, int64_t scap, cudaGraphConditionalHandle hw);
};

template <int N>
struct SettleK {
    static void run(rb_handle* h, int64_t bound);
};

template <int N>
struct DedupK {
    static void run(rb_handle* h, Front next, Front other);
};

template <typename T>
static void dalloc(T** p, size_t count) {
    if (*p) dfree(*p);
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = t_pool ? cudaMallocFromPoolAsync((void**)p, count * sizeof(T), t_pool, t_stream)
                           : cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        throw ArgError{RB_ERR_NOMEM, "device memory exhausted allocating " + std::to_string(count * sizeof(T)) +
                                         " bytes"};
    }
}

template <int N>
struct PartitionK {
    static void run(rb_handle* h, int world, int64_t* counts);
};

template <int N>
struct WidthK {
    static void run(rb_handle* h);
};

// frontier routing between shards: thin rows to their hash owner, `move[d]` surplus
// rows to rank d; F[cur] becomes [own rows | rows for rank 0 | rank 1 | ...]
template <int N>
struct RouteCountK {
    static void run(rb_handle* h, int world, int64_t* thin_counts, int64_t* nonthin);
};
template <int N>
struct RouteK {
    static void run(rb_handle* h, int world, int rank, const int64_t* move, int64_t* send_counts);
};


// every launcher template, for explicit instantiation (kinst.cu) and extern declarations (engine.cu)
#define RB_LAUNCHERS(X, K)                                                                              \
    X SetupK<K>; X ClassifyK<K>; X ClassifyFilterK<K>; X AllParentsK<K>; X FilterK<K>; X HsK<K>; X HsTileK<K>; X HsFusedK<K>; X KrawczykK<K>; \
    X SmallRoundsK<K>; X DedupInsertK<K>; X TailK<K>; X SettleK<K>; X DedupK<K>; X PartitionK<K>; X WidthK<K>; \
    X RouteCountK<K>; X RouteK<K>;
