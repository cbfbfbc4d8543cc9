// engine.cu -- host orchestration + C ABI (include/rootbox_b200.h).
//
// One rb_handle = one CUDA device + one compiled system.  rb_solve runs the
// round loop of rootbox.bnb.solve (bnb.py:224-354) with the frontier resident
// in HBM; per round:
//
//   memset counters -> K3 classify (carried rows straight into F_next, parents list)
//   -> K1 filter (implicit 2^n children, survivors to S) -> K2 HS (trigger decided
//   on device from the survivors' max width; outputs appended to F_next)
//   -> 1 small D2H of the counters (sync) -> overflow retry if a buffer was short
//   -> exact dedup (hash insert; compaction only when duplicates exist)
//
// so a round costs 3 kernel launches + 1-2 tiny syncs, independent of frontier size.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/rootbox_b200.h"
#include "kernels.cuh"

using namespace rb;

#define RB_VERSION "rootbox_b200 0.1.0 (sm_100a)"

namespace {

std::string g_create_error;

struct DevFront {
    Front f{};
    int n = 0;
    void release() {
        if (f.lo) cudaFree(f.lo);
        if (f.hi) cudaFree(f.hi);
        if (f.cert) cudaFree(f.cert);
        if (f.unsplit) cudaFree(f.unsplit);
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

}  // namespace

struct rb_handle {
    std::mutex mu;
    int dev = 0;
    int n = 0;
    int sms = 148;
    cudaStream_t st = nullptr;
    cudaEvent_t ev[6] = {};
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
    // dedup scratch
    unsigned* d_table = nullptr;
    size_t table_slots = 0;
    uint8_t* d_dead = nullptr;
    int64_t cap_dead = 0;
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
    bool have_result = false;
    std::vector<rb_round_stats> stats;
    // sharded protocol state
    double shard_target = 0.0;
    int64_t shard_carried = 0;
    int shard_round = 0;
    std::string err;
    // launch shapes
    int filter_threads = 256;
    int hs_threads = 128;
    int filter_blocks_per_sm = 1;
    int hs_blocks_per_sm = 1;
    size_t filter_smem = 0, hs_smem = 0;
    int smem_optin = 48 * 1024;
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

template <int N>
struct SetupK {
    static void run(rb_handle* h) {
        const size_t fs = stab_bytes(h->meta, true) + (size_t)2 * N * h->filter_threads * sizeof(double);
        const size_t hsm = stab_bytes(h->meta, false) +
                           (size_t)(h->hs_threads / 32) * HsLayout<N>::BPW * HsLayout<N>::doubles * sizeof(double);
        h->filter_smem = fs;
        h->hs_smem = hsm;
        // the attribute is per kernel (shared by every handle of this n): set it to the opt-in maximum
        if ((int)fs > h->smem_optin || (int)hsm > h->smem_optin)
            throw ArgError{RB_ERR_LIMIT, "system tables exceed the shared-memory budget"};
        ck(cudaFuncSetAttribute(k_filter<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_optin),
           "attr filter");
        ck(cudaFuncSetAttribute(k_hs<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_optin), "attr hs");
        int nb = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_filter<N>, h->filter_threads, fs), "occ filter");
        h->filter_blocks_per_sm = std::max(1, nb);
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs<N>, h->hs_threads, hsm), "occ hs");
        h->hs_blocks_per_sm = std::max(1, nb);
    }
};

template <int N>
struct ClassifyK {
    static void run(rb_handle* h, double target) {
        Front cur = h->F[h->cur].f, next = h->F[h->cur ^ 1].f;
        const int blocks = grid_for(h->n_cur, 256, h->sms * 8);
        k_classify<N><<<blocks, 256, 0, h->st>>>(h->meta, cur, h->n_cur, next, h->parents, h->d_ctr, target);
        ck(cudaGetLastError(), "classify launch");
    }
};

template <int N>
struct AllParentsK {
    static void run(rb_handle* h) {
        const int blocks = grid_for(h->n_cur, 256, h->sms * 8);
        k_all_parents<N><<<blocks, 256, 0, h->st>>>(h->meta, h->F[h->cur].f, h->n_cur, h->parents, h->d_ctr);
        ck(cudaGetLastError(), "parents launch");
    }
};

template <int N>
struct FilterK {
    static void run(rb_handle* h, int64_t max_parents, int64_t* tags) {
        const int64_t work = max_parents << N;
        const int blocks = grid_for(work, h->filter_threads, h->sms * h->filter_blocks_per_sm);
        k_filter<N><<<blocks, h->filter_threads, h->filter_smem, h->st>>>(h->meta, h->d_tab, h->F[h->cur].f,
                                                                         h->parents, h->d_ctr, h->S, tags);
        ck(cudaGetLastError(), "filter launch");
    }
};

template <int N>
struct HsK {
    static void run(rb_handle* h, int64_t max_in, int64_t n_in, HsParams prm, int64_t* tags) {
        const int per_block_boxes = (h->hs_threads / 32) * HsLayout<N>::BPW;
        const int blocks = grid_for(max_in * 1, per_block_boxes, h->sms * h->hs_blocks_per_sm);
        k_hs<N><<<std::max(blocks, 1), h->hs_threads, h->hs_smem, h->st>>>(
            h->meta, h->d_tab, h->S, n_in, prm, h->F[h->cur ^ 1].f, h->d_ctr, tags);
        ck(cudaGetLastError(), "hs launch");
    }
};

template <int N>
struct DedupK {
    static void run(rb_handle* h, Front f, int64_t n, size_t slots) {
        const int blocks = grid_for(n, 256, h->sms * 8);
        k_dedup_insert<N><<<blocks, 256, 0, h->st>>>(f, n, h->d_table, (unsigned long long)(slots - 1),
                                                     h->d_dead, h->d_ctr);
        ck(cudaGetLastError(), "dedup launch");
    }
};

template <int N>
struct CompactK {
    static void run(rb_handle* h, Front src, int64_t n, Front dst, unsigned long long* counter) {
        const int blocks = grid_for(n, 256, h->sms * 8);
        k_compact<N><<<blocks, 256, 0, h->st>>>(src, n, h->d_dead, dst, counter);
        ck(cudaGetLastError(), "compact launch");
    }
};

// ---------------------------------------------------------------- memory helpers

template <typename T>
static void dalloc(T** p, size_t count) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        throw ArgError{RB_ERR_NOMEM, "device memory exhausted allocating " + std::to_string(count * sizeof(T)) +
                                         " bytes"};
    }
}

static int64_t grow_cap(int64_t need) {
    int64_t c = 4096;
    while (c < need) c = c + c / 2;
    return c;
}

// (re)allocate a frontier for at least `need` rows, preserving the first `keep` rows
static void front_reserve(rb_handle* h, DevFront& F, int64_t need, int64_t keep) {
    if (F.f.cap >= need && F.f.lo) return;
    const int n = h->n;
    const int64_t cap = grow_cap(need);
    DevFront G;
    G.n = n;
    dalloc(&G.f.lo, (size_t)cap * n);
    dalloc(&G.f.hi, (size_t)cap * n);
    dalloc(&G.f.cert, (size_t)cap);
    dalloc(&G.f.unsplit, (size_t)cap);
    G.f.cap = cap;
    if (keep > 0 && F.f.lo) {
        ck(cudaMemcpy2DAsync(G.f.lo, cap * sizeof(double), F.f.lo, F.f.cap * sizeof(double), keep * sizeof(double), n,
                             cudaMemcpyDeviceToDevice, h->st), "grow copy lo");
        ck(cudaMemcpy2DAsync(G.f.hi, cap * sizeof(double), F.f.hi, F.f.cap * sizeof(double), keep * sizeof(double), n,
                             cudaMemcpyDeviceToDevice, h->st), "grow copy hi");
        ck(cudaMemcpyAsync(G.f.cert, F.f.cert, keep, cudaMemcpyDeviceToDevice, h->st), "grow copy cert");
        ck(cudaMemcpyAsync(G.f.unsplit, F.f.unsplit, keep, cudaMemcpyDeviceToDevice, h->st), "grow copy uns");
        ck(cudaStreamSynchronize(h->st), "grow sync");
    }
    F.release();
    F = G;
}

static void surv_reserve(rb_handle* h, int64_t need) {
    if (h->S.cap >= need && h->S.lo) return;
    const int64_t cap = grow_cap(need);
    if (h->S.lo) cudaFree(h->S.lo);
    if (h->S.hi) cudaFree(h->S.hi);
    h->S.lo = h->S.hi = nullptr;
    dalloc(&h->S.lo, (size_t)cap * h->n);
    dalloc(&h->S.hi, (size_t)cap * h->n);
    h->S.cap = cap;
}

static void parents_reserve(rb_handle* h, int64_t need) {
    if (h->cap_par >= need && h->parents) return;
    const int64_t cap = grow_cap(need);
    dalloc(&h->parents, (size_t)cap);
    h->cap_par = cap;
}

static void tags_reserve(rb_handle* h, int64_t need) {
    if (h->cap_tags >= need && h->d_tags) return;
    const int64_t cap = grow_cap(need);
    dalloc(&h->d_tags, (size_t)cap);
    h->cap_tags = cap;
}

static void sync_counters(rb_handle* h) {
    ck(cudaMemcpyAsync(h->h_ctr, h->d_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, h->st), "ctr d2h");
    ck(cudaStreamSynchronize(h->st), "ctr sync");
}

static double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

// ---------------------------------------------------------------- tables

static void build_tables(rb_handle* h, const rb_system* sys) {
    const int n = sys->n;
    if (n < 1 || n > RB_MAX_DIM) throw ArgError{RB_ERR_LIMIT, "dimension must be in 1..16"};
    if (sys->n_polys != n + n * n) throw ArgError{RB_ERR_ARG, "n_polys must be n + n*n"};
    const int P = sys->n_polys;
    const int T = sys->poly_off[P];
    const int Fc = sys->fac_off[T];
    if (T >= 65535 || Fc >= 65535) throw ArgError{RB_ERR_LIMIT, "too many terms for the u16 tables"};
    TabMeta m{};
    m.n = n;
    m.T = T;
    m.Fc = Fc;
    m.P = P;
    m.TF = sys->poly_off[n];
    m.FcF = sys->fac_off[m.TF];
    m.off_poly = align8(8 * T);
    m.off_fac_off = m.off_poly + align8(2 * (P + 1));
    m.off_fac = m.off_fac_off + align8(2 * (T + 1));
    m.bytes = m.off_fac + align8(2 * Fc);
    std::vector<uint8_t> buf(m.bytes, 0);
    std::memcpy(buf.data(), sys->coeff, 8 * (size_t)T);
    auto* po = reinterpret_cast<uint16_t*>(buf.data() + m.off_poly);
    auto* fo = reinterpret_cast<uint16_t*>(buf.data() + m.off_fac_off);
    auto* fa = reinterpret_cast<uint16_t*>(buf.data() + m.off_fac);
    for (int i = 0; i <= P; i++) {
        if (i > 0 && sys->poly_off[i] < sys->poly_off[i - 1]) throw ArgError{RB_ERR_ARG, "poly_off not monotone"};
        po[i] = (uint16_t)sys->poly_off[i];
    }
    for (int i = 0; i <= T; i++) fo[i] = (uint16_t)sys->fac_off[i];
    for (int i = 0; i < Fc; i++) {
        if (sys->fac_var[i] >= n || sys->fac_exp[i] == 0) throw ArgError{RB_ERR_ARG, "bad factor"};
        fa[i] = (uint16_t)(sys->fac_var[i] | (sys->fac_exp[i] << 8));
    }
    // guard constants + algorithmic op counts
    auto term_ops = [&](int q) {
        int ops = 2;
        for (int f = sys->fac_off[q]; f < sys->fac_off[q + 1]; f++) ops += 2 + 2 * (sys->fac_exp[f] - 1);
        return ops;
    };
    auto group = [&](int p0, int p1, int& ecmin, int& ecmax, int& deg, int& ops) {
        ecmin = 4096;
        ecmax = -4096;
        deg = 0;
        ops = 0;
        for (int p = p0; p < p1; p++)
            for (int q = sys->poly_off[p]; q < sys->poly_off[p + 1]; q++) {
                const double c = sys->coeff[q];
                if (!std::isfinite(c)) throw ArgError{RB_ERR_ARG, "non-finite coefficient"};
                if (c != 0.0) {
                    int e;
                    std::frexp(c, &e);
                    ecmin = std::min(ecmin, e - 1);
                    ecmax = std::max(ecmax, e - 1);
                }
                int d = 0;
                for (int f = sys->fac_off[q]; f < sys->fac_off[q + 1]; f++) d += sys->fac_exp[f];
                deg = std::max(deg, d);
                ops += term_ops(q);
            }
        if (ecmin > ecmax) ecmin = ecmax = 0;
    };
    int ops_f = 0, ops_j = 0;
    group(0, n, m.f_ecmin, m.f_ecmax, m.f_deg, ops_f);
    group(n, P, m.j_ecmin, m.j_ecmax, m.j_deg, ops_j);
    for (int e = 0; e < n; e++) {
        int ops = 0;
        for (int q = sys->poly_off[e]; q < sys->poly_off[e + 1]; q++) ops += term_ops(q);
        m.ops_eq[e] = ops;
    }
    int ops_gj = 0;
    for (int k = 0; k < n; k++) ops_gj += (2 * n - k) + 1 + 2 * (n - 1) * (2 * n - k);
    // ops_HS = ops_J + 2n^2 (mid) + ops_GJ + 2n (mid x) + ops_F + 4n^2 (g) + 4n^3 (M) + sweep
    m.ops_hs_pre = ops_j + 2 * n * n + ops_gj + 2 * n + ops_f + 4 * n * n + 4 * n * n * n;
    m.ops_hs_row = 6 * (n - 1) + 8;
    h->meta = m;
    dalloc(&h->d_tab, (size_t)m.bytes);
    ck(cudaMemcpy(h->d_tab, buf.data(), m.bytes, cudaMemcpyHostToDevice), "tables h2d");
    h->init_lo.assign(sys->init_lo, sys->init_lo + n);
    h->init_hi.assign(sys->init_hi, sys->init_hi + n);
    for (int j = 0; j < n; j++)
        if (!std::isfinite(h->init_lo[j]) || !std::isfinite(h->init_hi[j]) || h->init_lo[j] > h->init_hi[j])
            throw ArgError{RB_ERR_ARG, "initial box must be bounded with lo <= hi"};
}

// ---------------------------------------------------------------- rounds

static void load_rows(rb_handle* h, DevFront& F, int64_t off, const double* lo, const double* hi,
                      const uint8_t* cert, const uint8_t* uns, int64_t N) {
    if (N <= 0) return;
    const int n = h->n;
    double *dlo = nullptr, *dhi = nullptr;
    uint8_t *dc = nullptr, *du = nullptr;
    dalloc(&dlo, (size_t)N * n);
    dalloc(&dhi, (size_t)N * n);
    ck(cudaMemcpyAsync(dlo, lo, sizeof(double) * N * n, cudaMemcpyHostToDevice, h->st), "rows h2d");
    ck(cudaMemcpyAsync(dhi, hi, sizeof(double) * N * n, cudaMemcpyHostToDevice, h->st), "rows h2d");
    if (cert) {
        dalloc(&dc, (size_t)N);
        ck(cudaMemcpyAsync(dc, cert, N, cudaMemcpyHostToDevice, h->st), "rows h2d");
    }
    if (uns) {
        dalloc(&du, (size_t)N);
        ck(cudaMemcpyAsync(du, uns, N, cudaMemcpyHostToDevice, h->st), "rows h2d");
    }
    k_rows_to_soa<<<grid_for(N, 256, h->sms * 8), 256, 0, h->st>>>(dlo, dhi, dc, du, n, N, F.f, off);
    ck(cudaGetLastError(), "rows_to_soa");
    ck(cudaStreamSynchronize(h->st), "rows sync");
    cudaFree(dlo);
    cudaFree(dhi);
    if (dc) cudaFree(dc);
    if (du) cudaFree(du);
}

struct RoundOut {
    int64_t boxes_in, carried, survivors, after_hs, children, hs_calls, dups, exact;
    double child_width, width;
    bool hs_on;
    unsigned long long filter_ops, hs_ops;
    double classify_ms, filter_ms, hs_ms;
};

// classify + filter, with overflow retry of the survivor buffer
static void round_filter(rb_handle* h, double target, RoundOut& ro) {
    const int n = h->n;
    DevFront& next = h->F[h->cur ^ 1];
    // the carried rows can never exceed the current frontier
    front_reserve(h, next, std::max<int64_t>(h->n_cur, 1), 0);
    parents_reserve(h, std::max<int64_t>(h->n_cur, 1));
    surv_reserve(h, std::max<int64_t>(h->S.cap, 4096));
    ck(cudaMemsetAsync(h->d_ctr, 0, sizeof(Counters), h->st), "ctr memset");
    ck(cudaEventRecord(h->ev[0], h->st), "ev");
    if (h->n_cur > 0) dispatch_n<ClassifyK>(n, h, target);
    ck(cudaEventRecord(h->ev[1], h->st), "ev");
    if (h->n_cur > 0) dispatch_n<FilterK>(n, h, h->n_cur, (int64_t*)nullptr);
    ck(cudaEventRecord(h->ev[2], h->st), "ev");
    sync_counters(h);
    if (h->h_ctr->n_surv > (unsigned long long)h->S.cap) {
        // retry the filter into a buffer of the exact size
        surv_reserve(h, (int64_t)h->h_ctr->n_surv);
        Counters c = *h->h_ctr;
        c.n_surv = 0;
        c.child_wmax = 0;
        c.filter_ops = 0;
        c.exact_boxes = 0;
        ck(cudaMemcpyAsync(h->d_ctr, &c, sizeof(Counters), cudaMemcpyHostToDevice, h->st), "ctr h2d");
        ck(cudaEventRecord(h->ev[1], h->st), "ev");
        dispatch_n<FilterK>(n, h, h->n_cur, (int64_t*)nullptr);
        ck(cudaEventRecord(h->ev[2], h->st), "ev");
        sync_counters(h);
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
    ro.classify_ms = ms;
    cudaEventElapsedTime(&ms, h->ev[1], h->ev[2]);
    ro.filter_ms = ms;
    ro.boxes_in = h->n_cur;
    ro.carried = (int64_t)h->h_ctr->n_carried;
    ro.survivors = (int64_t)h->h_ctr->n_surv;
    ro.children = (int64_t)(h->h_ctr->n_par << n);
    ro.child_width = bits_to_double(h->h_ctr->child_wmax);
    ro.filter_ops = h->h_ctr->filter_ops;
    ro.exact = (int64_t)h->h_ctr->exact_boxes;
}

// HS (or pass-through) into F_next after the carried rows, with overflow retry; then dedup
static void round_hs(rb_handle* h, const HsParams& prm0, bool dedup, RoundOut& ro) {
    const int n = h->n;
    DevFront& next = h->F[h->cur ^ 1];
    const int64_t carried = ro.carried;
    const int64_t surv = ro.survivors;
    HsParams prm = prm0;
    prm.count_from_ctr = 1;
    // F_next must hold carried + up to 2 outputs per survivor; try the current
    // capacity first (forks are rare), grow exactly on overflow
    front_reserve(h, next, carried + surv + 1, carried);
    ck(cudaEventRecord(h->ev[3], h->st), "ev");
    if (surv > 0) dispatch_n<HsK>(n, h, surv, (int64_t)0, prm, (int64_t*)nullptr);
    ck(cudaEventRecord(h->ev[4], h->st), "ev");
    sync_counters(h);
    if (h->h_ctr->n_next > (unsigned long long)next.f.cap) {
        front_reserve(h, next, (int64_t)h->h_ctr->n_next, carried);
        Counters c = *h->h_ctr;
        c.n_next = carried;  // keep wmax: a max over the same rows the retry rewrites
        c.hs_ops = 0;
        c.hs_calls = 0;
        c.exact_boxes = 0;
        ck(cudaMemcpyAsync(h->d_ctr, &c, sizeof(Counters), cudaMemcpyHostToDevice, h->st), "ctr h2d");
        ck(cudaEventRecord(h->ev[3], h->st), "ev");
        dispatch_n<HsK>(n, h, surv, (int64_t)0, prm, (int64_t*)nullptr);
        ck(cudaEventRecord(h->ev[4], h->st), "ev");
        sync_counters(h);
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev[3], h->ev[4]);
    ro.hs_ms = ms;
    ro.hs_on = h->h_ctr->hs_on != 0;
    ro.hs_calls = (int64_t)h->h_ctr->hs_calls;
    ro.hs_ops = h->h_ctr->hs_ops;
    ro.exact = (int64_t)h->h_ctr->exact_boxes;
    int64_t n_next = (int64_t)h->h_ctr->n_next;
    ro.width = bits_to_double(h->h_ctr->wmax);
    ro.dups = 0;
    if (dedup && n_next >= 2) {
        // open-addressing table of >= 2 n slots (power of two)
        size_t slots = 1;
        while (slots < (size_t)(2 * n_next)) slots <<= 1;
        if (slots > h->table_slots || !h->d_table) {
            dalloc(&h->d_table, slots);
            h->table_slots = slots;
        }
        if (h->cap_dead < n_next || !h->d_dead) {
            dalloc(&h->d_dead, (size_t)grow_cap(n_next));
            h->cap_dead = grow_cap(n_next);
        }
        // use exactly `slots` entries (mask = slots - 1)
        ck(cudaMemsetAsync(h->d_table, 0, slots * sizeof(unsigned), h->st), "table memset");
        dispatch_n<DedupK>(n, h, next.f, n_next, slots);
        sync_counters(h);
        const int64_t dups = (int64_t)h->h_ctr->dups;
        if (dups > 0) {
            DevFront& other = h->F[h->cur];  // consumed input frontier, free now
            front_reserve(h, other, n_next - dups, 0);
            unsigned long long* cnt = &h->d_ctr->pad[0];
            ck(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), h->st), "cnt memset");
            dispatch_n<CompactK>(n, h, next.f, n_next, other.f, cnt);
            ck(cudaStreamSynchronize(h->st), "compact sync");
            // the compacted frontier now lives in F[cur]; swap roles so that
            // F[cur ^ 1] is the next frontier
            std::swap(h->F[0], h->F[1]);
            n_next -= dups;
        }
        ro.dups = dups;
    }
    ro.after_hs = n_next;
}

static void release_all(rb_handle* h) {
    h->F[0].release();
    h->F[1].release();
    auto fr = [](void* p) {
        if (p) cudaFree(p);
    };
    fr(h->parents);
    fr(h->S.lo);
    fr(h->S.hi);
    fr(h->d_ctr);
    fr(h->d_tags);
    fr(h->d_table);
    fr(h->d_dead);
    fr(h->d_cub);
    fr(h->d_keys[0]);
    fr(h->d_keys[1]);
    fr(h->d_perm[0]);
    fr(h->d_perm[1]);
    fr(h->r_lo);
    fr(h->r_hi);
    fr(h->r_cert);
    fr(h->r_uns);
    fr(h->d_tab);
    if (h->h_ctr) cudaFreeHost(h->h_ctr);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->st) cudaStreamDestroy(h->st);
}

// canonical order of F[cur] rows [0, N) -> result buffers (row-major)
static void finalize_sorted(rb_handle* h) {
    const int n = h->n;
    const int64_t N = h->n_cur;
    Front f = h->F[h->cur].f;
    dalloc(&h->r_lo, (size_t)std::max<int64_t>(N, 1) * n);
    dalloc(&h->r_hi, (size_t)std::max<int64_t>(N, 1) * n);
    dalloc(&h->r_cert, (size_t)std::max<int64_t>(N, 1));
    dalloc(&h->r_uns, (size_t)std::max<int64_t>(N, 1));
    h->r_n = N;
    if (N == 0) return;
    const unsigned* perm = nullptr;
    if (N > 1) {
        if (h->cap_sort < N) {
            const int64_t cap = grow_cap(N);
            for (int b = 0; b < 2; b++) {
                dalloc(&h->d_keys[b], (size_t)cap);
                dalloc(&h->d_perm[b], (size_t)cap);
            }
            h->cap_sort = cap;
            size_t bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, bytes, h->d_keys[0], h->d_keys[1], h->d_perm[0], h->d_perm[1],
                                            (int)cap, 0, 64, h->st);
            dalloc((uint8_t**)&h->d_cub, bytes);
            h->cub_bytes = bytes;
        }
        const int blocks = grid_for(N, 256, h->sms * 8);
        k_iota<<<blocks, 256, 0, h->st>>>(h->d_perm[0], N);
        // LSD over the 2n keys of np.lexsort order: least significant first (hi_{n-1}), most
        // significant last (lo_0); each pass is a stable radix sort.
        int cur = 0;
        for (int k = 2 * n - 1; k >= 0; k--) {
            k_sort_keys<<<blocks, 256, 0, h->st>>>(f, n, N, k, h->d_perm[cur], h->d_keys[0]);
            size_t bytes = h->cub_bytes;
            ck(cub::DeviceRadixSort::SortPairs(h->d_cub, bytes, h->d_keys[0], h->d_keys[1], h->d_perm[cur],
                                               h->d_perm[cur ^ 1], (int)N, 0, 64, h->st),
               "radix sort");
            cur ^= 1;
        }
        perm = h->d_perm[cur];
    }
    k_gather_rows<<<grid_for(N, 256, h->sms * 8), 256, 0, h->st>>>(f, n, N, perm, h->r_lo, h->r_hi, h->r_cert,
                                                                    h->r_uns);
    ck(cudaGetLastError(), "gather");
    ck(cudaStreamSynchronize(h->st), "finalize sync");
}

static double now_s() {
    using namespace std::chrono;
    return duration<double>(steady_clock::now().time_since_epoch()).count();
}

static void solve_impl(rb_handle* h, const rb_config* cfg, rb_result_info* info) {
    const int n = h->n;
    const double t_start = now_s();
    h->stats.clear();
    h->have_result = false;
    if (cfg->max_rounds < 1) throw ArgError{RB_ERR_ARG, "max_rounds must be at least 1"};
    if (cfg->max_boxes < 1) throw ArgError{RB_ERR_ARG, "max_boxes must be at least 1"};
    // initial frontier = the initial box (bnb.py:229-232)
    front_reserve(h, h->F[0], 4096, 0);
    front_reserve(h, h->F[1], 4096, 0);
    h->cur = 0;
    {
        uint8_t z = 0;
        load_rows(h, h->F[0], 0, h->init_lo.data(), h->init_hi.data(), &z, &z, 1);
    }
    h->n_cur = 1;
    double init_width = 0.0;
    for (int j = 0; j < n; j++) {
        const double d = h->init_hi[j] - h->init_lo[j];
        init_width = j == 0 ? d : std::max(init_width, d);
    }
    const bool has_target = cfg->target_width > 0;  // NaN and <= 0 mean None
    const double target = has_target ? cfg->target_width : init_width * 0x1p-10;
    const bool hs_possible = cfg->hs_enable_round >= 0 || !std::isnan(cfg->hs_enable_width);
    const bool has_max_seconds = cfg->max_seconds >= 0;
    int status = RB_BUDGET_EXHAUSTED;
    if (init_width <= target) {
        status = RB_WIDTH_REACHED;
    } else {
        for (int round_no = 1; round_no <= cfg->max_rounds; round_no++) {
            const double t0 = now_s();
            RoundOut ro{};
            round_filter(h, target, ro);
            HsParams prm{};
            prm.round_no = round_no;
            prm.hs_mode = 0;
            prm.hs_enable_round = cfg->hs_enable_round;
            prm.hs_possible = hs_possible ? 1 : 0;
            prm.hs_enable_width = cfg->hs_enable_width;
            prm.contract_output = cfg->hs_contract ? 1 : 0;
            round_hs(h, prm, cfg->exact_round_dedup != 0, ro);
            h->cur ^= 1;
            h->n_cur = ro.after_hs;
            rb_round_stats st{};
            st.round = round_no;
            st.hs_on = ro.hs_on;
            st.boxes_in = ro.boxes_in;
            st.boxes_after_filter = ro.carried + ro.survivors;
            st.boxes_after_hs = ro.after_hs;
            st.width = ro.after_hs ? ro.width : 0.0;
            st.children = ro.children;
            st.hs_calls = ro.hs_calls;
            st.filter_ops = (int64_t)ro.filter_ops;
            st.hs_ops = (int64_t)ro.hs_ops;
            st.dups = ro.dups;
            st.exact_boxes = ro.exact;
            st.filter_ms = ro.filter_ms;
            st.hs_ms = ro.hs_ms;
            st.classify_ms = ro.classify_ms;
            // classify reads every row (16n + 2 B) and writes carried rows + 4 B per parent
            st.classify_bytes = ro.boxes_in * (16 * n + 2) + ro.carried * (16 * n + 2) +
                                (ro.boxes_in - ro.carried) * 4;
            st.elapsed_seconds = now_s() - t0;
            h->stats.push_back(st);
            // termination (bnb.py:339-352)
            if (ro.after_hs == 0) {
                status = RB_NO_REAL_SOLUTION;
                break;
            }
            if (st.width <= target) {
                status = RB_WIDTH_REACHED;
                break;
            }
            if (ro.after_hs > cfg->max_boxes) {
                status = RB_BUDGET_EXHAUSTED;
                break;
            }
            if (has_max_seconds && now_s() - t_start > cfg->max_seconds) {
                status = RB_BUDGET_EXHAUSTED;
                break;
            }
        }
    }
    finalize_sorted(h);
    h->have_result = true;
    if (info) {
        info->status = status;
        info->nrounds = (int32_t)h->stats.size();
        info->nboxes = h->r_n;
        info->solve_seconds = now_s() - t_start;
    }
}

// ---------------------------------------------------------------- C ABI

#define RB_GUARD(h, ...)                                                                   \
    try {                                                                                  \
        __VA_ARGS__;                                                                            \
        return RB_OK;                                                                      \
    } catch (const CudaError& ce) {                                                        \
        (h)->err = std::string(ce.what) + ": " + cudaGetErrorString(ce.e);                 \
        cudaGetLastError();                                                                \
        return ce.e == cudaErrorMemoryAllocation ? RB_ERR_NOMEM : RB_ERR_CUDA;             \
    } catch (const ArgError& ae) {                                                         \
        (h)->err = ae.msg;                                                                 \
        return ae.code;                                                                    \
    } catch (const std::exception& ex) {                                                   \
        (h)->err = ex.what();                                                              \
        return RB_ERR_CUDA;                                                                \
    }

extern "C" {

const char* rb_version(void) { return RB_VERSION; }

int rb_device_count(void) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? 0 : RB_ERR_CUDA;
    }
    return c;
}

int rb_create(const rb_system* sys, int device, rb_handle** out) {
    if (!out || !sys) {
        g_create_error = "null argument";
        return RB_ERR_ARG;
    }
    *out = nullptr;
    rb_handle* h = new rb_handle();
    h->dev = device;
    h->n = sys->n;
    try {
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "props");
        if (prop.major < 10) throw ArgError{RB_ERR_CUDA, "device is not sm_100 class (B200 required)"};
        h->sms = prop.multiProcessorCount;
        h->smem_optin = (int)prop.sharedMemPerBlockOptin;
        ck(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking), "stream");
        for (auto& e : h->ev) ck(cudaEventCreate(&e), "event");
        build_tables(h, sys);
        dalloc(&h->d_ctr, 1);
        ck(cudaMallocHost((void**)&h->h_ctr, sizeof(Counters)), "pinned ctr");
        dispatch_n<SetupK>(h->n, h);
        *out = h;
        return RB_OK;
    } catch (const CudaError& ce) {
        g_create_error = std::string(ce.what) + ": " + cudaGetErrorString(ce.e);
        cudaGetLastError();
    } catch (const ArgError& ae) {
        g_create_error = ae.msg;
        release_all(h);
        delete h;
        return ae.code;
    }
    release_all(h);
    delete h;
    return RB_ERR_CUDA;
}

int rb_solve(rb_handle* h, const rb_config* cfg, rb_result_info* info) {
    if (!h || !cfg) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        solve_impl(h, cfg, info);
    })
}

int rb_fetch(rb_handle* h, double* lo, double* hi, uint8_t* cert, uint8_t* unsplit, rb_round_stats* stats) {
    if (!h) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->have_result) {
        h->err = "rb_fetch before a successful rb_solve";
        return RB_ERR_STATE;
    }
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        const int64_t N = h->r_n;
        if (N > 0) {
            if (lo) ck(cudaMemcpyAsync(lo, h->r_lo, sizeof(double) * N * h->n, cudaMemcpyDeviceToHost, h->st), "d2h");
            if (hi) ck(cudaMemcpyAsync(hi, h->r_hi, sizeof(double) * N * h->n, cudaMemcpyDeviceToHost, h->st), "d2h");
            if (cert) ck(cudaMemcpyAsync(cert, h->r_cert, N, cudaMemcpyDeviceToHost, h->st), "d2h");
            if (unsplit) ck(cudaMemcpyAsync(unsplit, h->r_uns, N, cudaMemcpyDeviceToHost, h->st), "d2h");
            ck(cudaStreamSynchronize(h->st), "fetch sync");
        }
        if (stats && !h->stats.empty()) std::memcpy(stats, h->stats.data(), sizeof(rb_round_stats) * h->stats.size());
    })
}

int rb_filter(rb_handle* h, const double* plo, const double* phi, int64_t P, double* olo, double* ohi, int64_t cap,
              int64_t* M) {
    if (!h || !M || P < 0 || (P > 0 && (!plo || !phi))) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    h->have_result = false;
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        const int n = h->n;
        *M = 0;
        if (P == 0) return RB_OK;
        h->cur = 0;
        front_reserve(h, h->F[0], P, 0);
        load_rows(h, h->F[0], 0, plo, phi, nullptr, nullptr, P);
        h->n_cur = P;
        parents_reserve(h, P);
        const int64_t bound = P << n;
        surv_reserve(h, std::min<int64_t>(bound, std::max<int64_t>(4096, P * 64)));
        for (int attempt = 0; attempt < 2; attempt++) {
            tags_reserve(h, h->S.cap);
            ck(cudaMemsetAsync(h->d_ctr, 0, sizeof(Counters), h->st), "ctr memset");
            dispatch_n<AllParentsK>(n, h);
            dispatch_n<FilterK>(n, h, P, h->d_tags);
            sync_counters(h);
            if (h->h_ctr->n_surv <= (unsigned long long)h->S.cap) break;
            surv_reserve(h, (int64_t)h->h_ctr->n_surv);
        }
        const int64_t m = (int64_t)h->h_ctr->n_surv;
        *M = m;
        std::vector<double> slo((size_t)m * n), shi((size_t)m * n);
        std::vector<int64_t> tags(m);
        for (int j = 0; j < n; j++) {
            ck(cudaMemcpyAsync(slo.data() + (size_t)j * m, h->S.lo + (size_t)j * h->S.cap, sizeof(double) * m,
                               cudaMemcpyDeviceToHost, h->st), "d2h");
            ck(cudaMemcpyAsync(shi.data() + (size_t)j * m, h->S.hi + (size_t)j * h->S.cap, sizeof(double) * m,
                               cudaMemcpyDeviceToHost, h->st), "d2h");
        }
        ck(cudaMemcpyAsync(tags.data(), h->d_tags, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaStreamSynchronize(h->st), "sync");
        std::vector<int64_t> order(m);
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return tags[a] < tags[b]; });
        const int64_t w = std::min(m, cap);
        for (int64_t r = 0; r < w; r++)
            for (int j = 0; j < n; j++) {
                olo[r * n + j] = slo[(size_t)j * m + order[r]];
                ohi[r * n + j] = shi[(size_t)j * m + order[r]];
            }
    })
}

int rb_hs(rb_handle* h, const double* lo, const double* hi, int64_t M, int contract_output, double* olo, double* ohi,
          uint8_t* cert, int64_t cap, int64_t* M2) {
    if (!h || !M2 || M < 0 || (M > 0 && (!lo || !hi))) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    h->have_result = false;
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        const int n = h->n;
        *M2 = 0;
        if (M == 0) return RB_OK;
        surv_reserve(h, M);
        // stage rows into S via a temporary frontier view
        Front sview{h->S.lo, h->S.hi, nullptr, nullptr, h->S.cap};
        DevFront tmp;
        tmp.f = sview;
        load_rows(h, tmp, 0, lo, hi, nullptr, nullptr, M);
        h->cur = 0;
        DevFront& out = h->F[1];
        front_reserve(h, out, 2 * M, 0);
        tags_reserve(h, out.f.cap);
        HsParams prm{};
        prm.hs_mode = 1;
        prm.contract_output = contract_output ? 1 : 0;
        prm.count_from_ctr = 0;
        ck(cudaMemsetAsync(h->d_ctr, 0, sizeof(Counters), h->st), "ctr memset");
        dispatch_n<HsK>(n, h, M, M, prm, h->d_tags);
        sync_counters(h);
        const int64_t m = (int64_t)h->h_ctr->n_next;
        *M2 = m;
        std::vector<double> slo((size_t)m * n), shi((size_t)m * n);
        std::vector<uint8_t> c(m);
        std::vector<int64_t> tags(m);
        for (int j = 0; j < n; j++) {
            ck(cudaMemcpyAsync(slo.data() + (size_t)j * m, out.f.lo + (size_t)j * out.f.cap, sizeof(double) * m,
                               cudaMemcpyDeviceToHost, h->st), "d2h");
            ck(cudaMemcpyAsync(shi.data() + (size_t)j * m, out.f.hi + (size_t)j * out.f.cap, sizeof(double) * m,
                               cudaMemcpyDeviceToHost, h->st), "d2h");
        }
        ck(cudaMemcpyAsync(c.data(), out.f.cert, m, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaMemcpyAsync(tags.data(), h->d_tags, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaStreamSynchronize(h->st), "sync");
        std::vector<int64_t> order(m);
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return tags[a] < tags[b]; });
        const int64_t w = std::min(m, cap);
        for (int64_t r = 0; r < w; r++) {
            for (int j = 0; j < n; j++) {
                olo[r * n + j] = slo[(size_t)j * m + order[r]];
                ohi[r * n + j] = shi[(size_t)j * m + order[r]];
            }
            if (cert) cert[r] = c[order[r]];
        }
    })
}

const char* rb_last_error(rb_handle* h) {
    if (!h) return g_create_error.c_str();
    return h->err.c_str();
}

void rb_destroy(rb_handle* h) {
    if (!h) return;
    {
        std::lock_guard<std::mutex> lk(h->mu);
        cudaSetDevice(h->dev);
        release_all(h);
    }
    delete h;
}

// ---------------------------------------------------------------- sharded protocol

int rb_shard_load(rb_handle* h, const double* lo, const double* hi, const uint8_t* cert, const uint8_t* unsplit,
                  int64_t N, double target_width) {
    if (!h || N < 0) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        h->cur = 0;
        front_reserve(h, h->F[0], std::max<int64_t>(N, 1), 0);
        front_reserve(h, h->F[1], std::max<int64_t>(N, 1), 0);
        load_rows(h, h->F[0], 0, lo, hi, cert, unsplit, N);
        h->n_cur = N;
        h->shard_target = target_width;
        h->have_result = false;
    })
}

int rb_round_filter(rb_handle* h, int32_t round_no, int64_t* carried, int64_t* survivors, double* child_width,
                    int64_t* children) {
    if (!h) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        RoundOut ro{};
        round_filter(h, h->shard_target, ro);
        h->shard_carried = ro.carried;
        h->shard_round = round_no;
        if (carried) *carried = ro.carried;
        if (survivors) *survivors = ro.survivors;
        if (child_width) *child_width = ro.child_width;
        if (children) *children = ro.children;
    })
}

int rb_round_hs(rb_handle* h, int32_t hs_on, int32_t hs_contract, int64_t* n_out, double* width, int64_t* hs_calls) {
    if (!h) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        RoundOut ro{};
        ro.carried = h->shard_carried;
        ro.survivors = (int64_t)h->h_ctr->n_surv;
        HsParams prm{};
        prm.round_no = h->shard_round;
        prm.hs_mode = hs_on ? 1 : 2;
        prm.contract_output = hs_contract ? 1 : 0;
        round_hs(h, prm, true, ro);
        h->cur ^= 1;
        h->n_cur = ro.after_hs;
        if (n_out) *n_out = ro.after_hs;
        if (width) *width = ro.after_hs ? ro.width : 0.0;
        if (hs_calls) *hs_calls = ro.hs_calls;
    })
}

int rb_shard_export(rb_handle* h, int64_t start, int64_t count, double* lo, double* hi, uint8_t* cert,
                    uint8_t* unsplit) {
    if (!h || start < 0 || count < 0) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    if (start + count > h->n_cur) {
        h->err = "export range beyond the shard";
        return RB_ERR_ARG;
    }
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        const int n = h->n;
        if (count == 0) return RB_OK;
        Front f = h->F[h->cur].f;
        double *dlo = nullptr, *dhi = nullptr;
        uint8_t *dc = nullptr, *du = nullptr;
        dalloc(&dlo, (size_t)count * n);
        dalloc(&dhi, (size_t)count * n);
        dalloc(&dc, (size_t)count);
        dalloc(&du, (size_t)count);
        Front sub = f;
        sub.lo = f.lo + start;
        sub.hi = f.hi + start;
        sub.cert = f.cert + start;
        sub.unsplit = f.unsplit + start;
        k_gather_rows<<<grid_for(count, 256, h->sms * 8), 256, 0, h->st>>>(sub, n, count, nullptr, dlo, dhi, dc, du);
        ck(cudaGetLastError(), "export gather");
        if (lo) ck(cudaMemcpyAsync(lo, dlo, sizeof(double) * count * n, cudaMemcpyDeviceToHost, h->st), "d2h");
        if (hi) ck(cudaMemcpyAsync(hi, dhi, sizeof(double) * count * n, cudaMemcpyDeviceToHost, h->st), "d2h");
        if (cert) ck(cudaMemcpyAsync(cert, dc, count, cudaMemcpyDeviceToHost, h->st), "d2h");
        if (unsplit) ck(cudaMemcpyAsync(unsplit, du, count, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaStreamSynchronize(h->st), "export sync");
        cudaFree(dlo);
        cudaFree(dhi);
        cudaFree(dc);
        cudaFree(du);
    })
}

int rb_shard_import(rb_handle* h, int64_t keep, const double* lo, const double* hi, const uint8_t* cert,
                    const uint8_t* unsplit, int64_t count) {
    if (!h || keep < 0 || count < 0) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    if (keep > h->n_cur) {
        h->err = "keep beyond the shard";
        return RB_ERR_ARG;
    }
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        DevFront& F = h->F[h->cur];
        front_reserve(h, F, keep + count, keep);
        load_rows(h, F, keep, lo, hi, cert, unsplit, count);
        h->n_cur = keep + count;
    })
}

int64_t rb_shard_size(rb_handle* h) { return h ? h->n_cur : -1; }

}  // extern "C"
