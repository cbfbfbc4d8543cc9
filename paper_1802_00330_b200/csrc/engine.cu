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
#include "engine.cuh"

namespace {
std::string g_create_error;
}  // namespace

// launchers are instantiated in kinst.cu (one TU per few dimensions, built in parallel)
#define RB_EXTERN(K) RB_LAUNCHERS(extern template struct, K)
RB_EXTERN(1) RB_EXTERN(2) RB_EXTERN(3) RB_EXTERN(4) RB_EXTERN(5) RB_EXTERN(6) RB_EXTERN(7) RB_EXTERN(8)
RB_EXTERN(9) RB_EXTERN(10) RB_EXTERN(11) RB_EXTERN(12) RB_EXTERN(13) RB_EXTERN(14) RB_EXTERN(15) RB_EXTERN(16)
#undef RB_EXTERN

// One stream-ordered memory pool per device for the whole process, retaining
// its memory (release threshold = max): a new handle for the next system reuses
// the frontier buffers of the last one instead of mapping fresh memory.
static cudaMemPool_t device_pool(int device) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)pools.size() <= device) pools.resize(device + 1, nullptr);
    if (!pools[device]) {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = device;
        ck(cudaMemPoolCreate(&pools[device], &pp), "mempool");
        uint64_t thr = UINT64_MAX;
        ck(cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &thr), "mempool attr");
    }
    return pools[device];
}

// ---------------------------------------------------------------- memory helpers

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
    }
    F.release();
    F = G;
}

static void surv_reserve(rb_handle* h, int64_t need) {
    if (h->S.cap >= need && h->S.lo) return;
    const int64_t cap = grow_cap(need);
    dfree(h->S.lo);
    dfree(h->S.hi);
    h->S.lo = h->S.hi = nullptr;
    dalloc(&h->S.lo, (size_t)cap * h->n);
    dalloc(&h->S.hi, (size_t)cap * h->n);
    h->S.cap = cap;
}

// HS scratch: batch capacity B <= S.cap, bounded so the scratch stays small
static void scratch_reserve(rb_handle* h, int64_t want) {
    const int n = h->n;
    const size_t per_box = (size_t)(2 * n * n + 3 * n) * sizeof(double) + 1;
    const size_t cap_bytes = std::min<size_t>((size_t)4 << 30, h->mem_budget / 5);
    int64_t B = std::min<int64_t>(want, std::max<int64_t>(65536, (int64_t)(cap_bytes / per_box)));
    B = std::max<int64_t>(B, 1024);
    if (h->W.B >= B && h->W.x) return;
    auto fr = [](void* p) { dfree(p); };
    fr(h->W.x); fr(h->W.jl); fr(h->W.jh); fr(h->W.fl); fr(h->W.fh); fr(h->W.flags);
    h->W = HsScratch{};
    dalloc(&h->W.x, (size_t)B * n);
    dalloc(&h->W.jl, (size_t)B * n * n);
    dalloc(&h->W.jh, (size_t)B * n * n);
    dalloc(&h->W.fl, (size_t)B * n);
    dalloc(&h->W.fh, (size_t)B * n);
    dalloc(&h->W.flags, (size_t)B);
    h->W.B = B;
}

// all batches of the HS pipeline over at most `bound` survivors: the tiled kernel
// (one launch, no scratch) when it applies, else eval/lin/sweep per scratch batch
static void launch_hs_three(rb_handle* h, int64_t bound, int64_t n_in, const HsParams& prm, int64_t* tags) {
    if (h->hs_tile) {
        dispatch_n<HsTileK>(h->n, h, n_in, prm, tags, bound);
        return;
    }
    scratch_reserve(h, std::max<int64_t>(bound, 1));
    const int64_t B = h->W.B;
    for (int64_t b0 = 0; b0 == 0 || b0 < bound; b0 += B)
        dispatch_n<HsK>(h->n, h, b0, n_in, prm, tags, std::min<int64_t>(B, bound - b0));
}

// HS over the survivors: k_hs_fused (one launch, latency-optimal) for counts up to
// h->fused_rows, eval/lin/sweep (throughput-optimal) above.  When the count is only
// known on the device both are enqueued and each exits unless the count is its own;
// inside a graph capture the fused kernel instead sets an IF node around the other three.
static void launch_hs_batches(rb_handle* h, int64_t bound, int64_t n_in, const HsParams& prm0, int64_t* tags) {
    HsParams prm = prm0;
    prm.has_cond = 0;
    const int64_t thr = h->hs_fused ? h->fused_rows : -1;
    const int64_t rows = prm.count_from_ctr ? bound : n_in;
    if (rows <= thr) {
        prm.fused_max = LLONG_MAX;
        dispatch_n<HsFusedK>(h->n, h, n_in, prm, tags, bound);
        return;
    }
    if (!prm.count_from_ctr || thr < 0) {
        prm.fused_max = -1;
        launch_hs_three(h, bound, n_in, prm, tags);
        return;
    }
    prm.fused_max = thr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    ck(cudaStreamIsCapturing(h->st, &cs), "capture status");
    if (cs != cudaStreamCaptureStatusActive || !h->hs_cond) {
        dispatch_n<HsFusedK>(h->n, h, n_in, prm, tags, thr);
        launch_hs_three(h, bound, n_in, prm, tags);
        return;
    }
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    ck(cudaStreamGetCaptureInfo(h->st, &cs, nullptr, &cg, &deps, &ndeps), "capture info");
    ck(cudaGraphConditionalHandleCreate(&prm.big_cond, cg, 0, 0), "cond handle");
    prm.has_cond = 1;
    dispatch_n<HsFusedK>(h->n, h, n_in, prm, tags, thr);
    ck(cudaStreamGetCaptureInfo(h->st, &cs, nullptr, &cg, &deps, &ndeps), "capture info");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = prm.big_cond;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    ck(cudaGraphAddNode(&node, cg, deps, ndeps, &cp), "if node");
    ck(cudaStreamUpdateCaptureDependencies(h->st, &node, 1, cudaStreamSetCaptureDependencies), "capture deps");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStream_t main_st = h->st;
    ck(cudaStreamBeginCaptureToGraph(h->st_side, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
       "begin side capture");
    h->st = h->st_side;
    prm.has_cond = 0;
    try {
        launch_hs_three(h, bound, n_in, prm, tags);
    } catch (...) {
        h->st = main_st;
        throw;
    }
    h->st = main_st;
    cudaGraph_t side = nullptr;
    ck(cudaStreamEndCapture(h->st_side, &side), "end side capture");
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

static void reset_order(rb_handle* h) {
    for (int k = 0; k < 16; k++) h->h_order[k] = k;  // reference order to start
    ck(cudaMemcpyAsync(h->d_order, h->h_order, sizeof(h->h_order), cudaMemcpyHostToDevice, h->st), "order h2d");
}

// host-driven rounds: next round's filter order from this round's counts
static void update_order(rb_handle* h) {
    filter_order(h->h_ctr->f_eval, h->h_ctr->f_rej, h->meta.cost_eq, h->n, h->h_order);
    ck(cudaMemcpyAsync(h->d_order, h->h_order, sizeof(h->h_order), cudaMemcpyHostToDevice, h->st), "order h2d");
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
    // tabulated-filter metadata: per F term its entry base inside its equation's
    // table, and per equation the (term, combo) entries to build
    std::vector<uint16_t> tbase(std::max(1, m.TF));
    std::vector<uint16_t> ent_off(n + 1, 0);
    std::vector<uint32_t> ent;
    m.e_max = 1;
    m.ftab = 1;
    for (int e = 0; e < n; e++) {
        int base = 0;
        for (int q = sys->poly_off[e]; q < sys->poly_off[e + 1]; q++) {
            const int d = sys->fac_off[q + 1] - sys->fac_off[q];
            if (d > 15 || base + (1 << d) > 60000) {
                m.ftab = 0;
                break;
            }
            tbase[q] = (uint16_t)base;
            for (int combo = 0; combo < (1 << d); combo++) ent.push_back((uint32_t)q | ((uint32_t)combo << 16));
            base += 1 << d;
        }
        if (!m.ftab) break;
        ent_off[e + 1] = (uint16_t)ent.size();
        m.e_max = std::max(m.e_max, base);
        if (ent.size() > 60000) {
            m.ftab = 0;
            break;
        }
    }
    if (!m.ftab) {
        ent.clear();
        std::fill(ent_off.begin(), ent_off.end(), 0);
    }
    m.ent_total = (int)ent.size();
    // k_filter_wt: an equation whose table exceeds a quarter of a work unit's children
    // (2^min(n, 10) / 4) is evaluated per child; the table area fits the largest of the others
    m.fwt_direct = 0;
    m.fwt_emax = 1;
    if (m.ftab) {
        const int lim = 1 << (std::min(n, 10) - 2);
        for (int e = 0; e < n; e++) {
            const int E = ent_off[e + 1] - ent_off[e];
            if (E > lim) m.fwt_direct |= 1 << e;
            else m.fwt_emax = std::max(m.fwt_emax, E);
        }
    }
    // the tables pay off when terms multiply several variables (measured: eco8 1.6x
    // faster filter, linear-term systems slightly slower): mean (d - 1) >= 1
    {
        int extra = 0;
        for (int q = 0; q < m.TF; q++) extra += std::max(0, sys->fac_off[q + 1] - sys->fac_off[q] - 1);
        h->use_ftab = m.TF > 0 && extra >= m.TF;
    }
    m.off_tbase = m.bytes;
    m.off_ent_off = m.off_tbase + align8(2 * std::max(1, m.TF));
    m.off_ent = m.off_ent_off + align8(2 * (n + 1));
    m.bytes2 = m.off_ent + align8(4 * std::max(1, m.ent_total));
    m.off_termp = align16(m.bytes2);
    m.bytes3 = m.off_termp + 16 * std::max(1, m.TF);
    std::vector<uint8_t> buf(m.bytes3, 0);
    for (int q = 0; q < m.TF; q++) {
        TermP tp{};
        tp.c = sys->coeff[q];
        const int f0 = sys->fac_off[q], f1 = sys->fac_off[q + 1];
        tp.nf = (uint16_t)(f1 - f0);
        tp.packed = (f1 - f0) <= 4 ? 1 : 0;
        for (int f = f0; f < f1 && tp.packed; f++) {
            if (sys->fac_var[f] >= 16 || sys->fac_exp[f] < 1 || sys->fac_exp[f] > 16) tp.packed = 0;
            else tp.fpack |= (uint32_t)(sys->fac_var[f] | ((sys->fac_exp[f] - 1) << 4)) << (8 * (f - f0));
        }
        if (!tp.packed) tp.fpack = 0;
        std::memcpy(buf.data() + m.off_termp + 16 * q, &tp, sizeof(TermP));
    }
    std::memcpy(buf.data() + m.off_tbase, tbase.data(), 2 * (size_t)std::max(1, m.TF));
    std::memcpy(buf.data() + m.off_ent_off, ent_off.data(), 2 * (size_t)(n + 1));
    if (!ent.empty()) std::memcpy(buf.data() + m.off_ent, ent.data(), 4 * ent.size());
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
        int ops = 0, cost = 0;
        for (int q = sys->poly_off[e]; q < sys->poly_off[e + 1]; q++) {
            ops += term_ops(q);
            // instruction-cost model of one term in k_filter: point x interval product,
            // full interval products, power chains, the accumulate
            const int nf = sys->fac_off[q + 1] - sys->fac_off[q];
            cost += 4 + (nf >= 1 ? 8 : 0) + 20 * std::max(0, nf - 1);
            for (int f = sys->fac_off[q]; f < sys->fac_off[q + 1]; f++) cost += 6 * (sys->fac_exp[f] - 1);
        }
        m.ops_eq[e] = ops;
        m.cost_eq[e] = std::max(1, cost);
    }
    int ops_gj = 0;
    for (int k = 0; k < n; k++) ops_gj += (2 * n - k) + 1 + 2 * (n - 1) * (2 * n - k);
    // ops_HS = ops_J + 2n^2 (mid) + ops_GJ + 2n (mid x) + ops_F + 4n^2 (g) + 4n^3 (M) + sweep
    m.ops_hs_pre = ops_j + 2 * n * n + ops_gj + 2 * n + ops_f + 4 * n * n + 4 * n * n * n;
    m.ops_hs_row = 6 * (n - 1) + 8;
    h->guard_f_ecmin = m.f_ecmin;
    h->guard_j_ecmin = m.j_ecmin;
    h->meta = m;
    // constant J entries: no term, or one term without factors -- the value [c, c] that
    // eval_poly (and the specialised evaluator, codegen.cpp evJ) computes for every box
    {
        std::vector<double> jc((size_t)n * n, 0.0);
        for (int w = 0; w < 4; w++) h->jmask[w] = 0;
        for (int q = 0; q < n * n; q++) {
            const int t0 = sys->poly_off[n + q], t1 = sys->poly_off[n + q + 1];
            const bool cst = t1 == t0 || (t1 - t0 == 1 && sys->fac_off[t0 + 1] == sys->fac_off[t0]);
            if (!cst) continue;
            h->jmask[q >> 6] |= 1ull << (q & 63);
            jc[q] = t1 == t0 ? 0.0 : 0.0 + sys->coeff[t0];  // [0,0] + [c,c] (+0 for a zero c)
        }
        dalloc(&h->d_jc, (size_t)n * n);
        ck(cudaMemcpyAsync(h->d_jc, jc.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, h->st), "jc h2d");
    }
    dalloc(&h->d_tab, (size_t)m.bytes3);
    ck(cudaMemcpyAsync(h->d_tab, buf.data(), m.bytes3, cudaMemcpyHostToDevice, h->st), "tables h2d");
    ck(cudaStreamSynchronize(h->st), "tables sync");
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
    h->launches++;
    k_rows_to_soa<<<grid_for(N, 256, h->sms * 8), 256, 0, h->st>>>(dlo, dhi, dc, du, n, N, F.f, off);
    ck(cudaGetLastError(), "rows_to_soa");
    ck(cudaStreamSynchronize(h->st), "rows sync");
    dfree(dlo);
    dfree(dhi);
    dfree(dc);
    dfree(du);
}

struct RoundOut {
    int64_t boxes_in, carried, survivors, after_hs, children, hs_calls, dups, exact;
    double child_width, width;
    bool hs_on;
    unsigned long long filter_ops, hs_ops;
    double classify_ms, filter_ms, hs_ms;
    int attempts;
};

// both frontier buffers share one capacity (the dedup compaction may target
// either); the current one keeps its rows when grown
static void fronts_reserve(rb_handle* h, int64_t need, int64_t keep_next = 0) {
    front_reserve(h, h->F[h->cur], need, h->n_cur);
    front_reserve(h, h->F[h->cur ^ 1], h->F[h->cur].f.cap, keep_next);
    if (h->F[h->cur ^ 1].f.cap != h->F[h->cur].f.cap) front_reserve(h, h->F[h->cur], h->F[h->cur ^ 1].f.cap, h->n_cur);
    const int64_t cap = h->F[h->cur].f.cap;
    if (h->cap_dead < cap || !h->d_dead) {
        dalloc(&h->d_dead, (size_t)cap);
        dalloc(&h->d_slot, (size_t)cap);
        h->cap_dead = cap;
    }
    size_t slots = 1;
    while (slots < (size_t)(2 * cap)) slots <<= 1;
    if (slots > h->table_slots || !h->d_table) {
        dalloc(&h->d_table, slots);
        ck(cudaMemsetAsync(h->d_table, 0, slots * sizeof(unsigned), h->st), "table memset");
        h->table_slots = slots;
    }
}

static void record(rb_handle* h, int i) { ck(cudaEventRecord(h->ev[i], h->st), "event"); }

static float elapsed(rb_handle* h, int a, int b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]);
    return ms;
}

// K3 classify + K1 filter (no sync)

__global__ void k_stamp(unsigned long long* buf, const DevState* st, int round_host, int phase, int delta) {
    if (st && (st->done || st->bail) && delta == 0) return;  // unrolled round after the end
    const int r = (st ? st->round_no : round_host) + delta;
    if (r >= 0 && r < kTraceRounds) buf[r * kTracePhases + phase] = gtimer();
}
static void stamp(rb_handle* h, const DevState* st, int round_host, int phase, int delta = 0) {
    if (!h->trace) return;
    k_stamp<<<1, 1, 0, h->st>>>(h->d_trace, st, round_host, phase, delta);
}
static void trace_report(rb_handle* h, int rounds) {
    if (!h->trace) return;
    std::vector<unsigned long long> t(kTraceWords);
    ck(cudaMemcpy(t.data(), h->d_trace, t.size() * 8, cudaMemcpyDeviceToHost), "trace d2h");
    static const char* names[] = {"classify", "filter", "hs", "dedup", "tail", "round_end", "loop"};
    {
        const unsigned long long* g = &t[(size_t)(kTraceRounds - 1) * kTracePhases];
        const unsigned long long r1 = t[(size_t)1 * kTracePhases];
        if (g[0] && g[3] && r1)
            std::fprintf(stderr, "[rb trace] graph: start kernel %.1f us, to round 1 %.1f us, rounds (start -> finish) "
                                 "%.1f us, finish kernel %.1f us, total %.1f us\n", (g[1] - g[0]) * 1e-3,
                         (r1 - g[1]) * 1e-3, (g[2] - g[1]) * 1e-3, (g[3] - g[2]) * 1e-3, (g[3] - g[0]) * 1e-3);
    }
    for (int r = 1; r <= std::min(rounds, kTraceRounds - 1); r++) {
        const unsigned long long* p = &t[(size_t)r * kTracePhases];
        if (!p[0]) continue;
        std::fprintf(stderr, "[rb trace] round %2d:", r);
        const unsigned long long nxt = r + 1 < kTraceRounds ? t[(size_t)(r + 1) * kTracePhases] : 0;
        for (int k = 0; k < 7; k++) {
            if (k == 5) continue;  // no stamp between the round tail and the round end (one kernel)
            const unsigned long long b = k == 4 ? p[6] : (k < 6 ? p[k + 1] : nxt);
            if (p[k] && b >= p[k]) std::fprintf(stderr, " %s %.1f", names[k], (b - p[k]) * 1e-3);
        }
        std::fprintf(stderr, " us");
        std::fprintf(stderr, "\n");
    }
    const unsigned long long* q = &t[(size_t)kTraceRounds * kTracePhases];
    if (q[1]) {
        std::fprintf(stderr, "[rb trace] last k_hs_fused, block 0 (cycles): ctr %llu, tables %llu, box load %llu, eval %llu, "
                             "lin %llu, sweep %llu, output %llu, rest %llu; kernel %.1f us\n",
                     q[2] - q[1], q[3] - q[2], q[4] - q[3], q[5] - q[4], q[6] - q[5], q[7] - q[6], q[8] - q[7],
                     q[9] - q[8], (q[10] - q[0]) * 1e-3);
        std::fprintf(stderr, "[rb trace]   lin: loads %llu, scale %llu, gauss-jordan %llu, guards %llu, products %llu\n",
                     q[11] - q[5], q[12] - q[11], q[13] - q[12], q[14] - q[13], q[6] - q[14]);
    }
    {
        const unsigned long long* bt = &t[kTraceHsBlkOff];
        unsigned long long t0 = ~0ull, t1 = 0;
        int nb = 0;
        for (int b = 0; b < kTraceBlocks; b++)
            if (bt[3 * b] && bt[3 * b + 1]) {
                nb++;
                t0 = std::min(t0, bt[3 * b]);
                t1 = std::max(t1, bt[3 * b + 1]);
            }
        if (nb) {
            std::vector<double> st, en;
            for (int b = 0; b < kTraceBlocks; b++)
                if (bt[3 * b] && bt[3 * b + 1]) st.push_back((bt[3 * b] - t0) * 1e-3), en.push_back((bt[3 * b + 1] - t0) * 1e-3);
            std::vector<double> s2 = st, e2 = en;
            std::sort(s2.begin(), s2.end());
            std::sort(e2.begin(), e2.end());
            auto q = [](const std::vector<double>& v, double f) { return v[(size_t)(f * (v.size() - 1))]; };
            std::fprintf(stderr, "[rb trace] last k_hs_fused blocks %d: start p0 %.1f p50 %.1f p100 %.1f, end p0 %.1f "
                                 "p50 %.1f p90 %.1f p100 %.1f us (from first block start)\n",
                         nb, q(s2, 0), q(s2, .5), q(s2, 1), q(e2, 0), q(e2, .5), q(e2, .9), q(e2, 1));
        }
    }
    {
        const unsigned long long* bt = &t[kTraceCfOff];
        std::vector<double> a, b, c, d;
        unsigned long long t0 = ~0ull;
        for (int k = 0; k < kTraceBlocks; k++)
            if (bt[4 * k] && bt[4 * k + 3]) t0 = std::min(t0, bt[4 * k]);
        for (int k = 0; k < kTraceBlocks; k++)
            if (bt[4 * k] && bt[4 * k + 3]) {
                a.push_back((bt[4 * k] - t0) * 1e-3);
                b.push_back((bt[4 * k + 1] - t0) * 1e-3);
                c.push_back((bt[4 * k + 2] - t0) * 1e-3);
                d.push_back((bt[4 * k + 3] - t0) * 1e-3);
            }
        if (!a.empty()) {
            for (auto* v : {&a, &b, &c, &d}) std::sort(v->begin(), v->end());
            auto q = [](const std::vector<double>& v, double f) { return v[(size_t)(f * (v.size() - 1))]; };
            std::fprintf(stderr, "[rb trace] last k_classify_filter blocks %zu (p50/p100 us from first start): start "
                                 "%.1f/%.1f tables %.1f/%.1f loop %.1f/%.1f end %.1f/%.1f\n",
                         a.size(), q(a, .5), q(a, 1), q(b, .5), q(b, 1), q(c, .5), q(c, 1), q(d, .5), q(d, 1));
        }
    }
    {  // per-box k_hs_fused records of the last round that ran HS
        const unsigned long long* br = &t[kTraceBoxAbs];
        std::vector<unsigned long long> rounds_seen;  // a later round overwrites the first records
        for (int b = 0; b < kTraceBoxes; b++)
            if (br[8 * b + 4] &&
                std::find(rounds_seen.begin(), rounds_seen.end(), br[8 * b + 6]) == rounds_seen.end())
                rounds_seen.push_back(br[8 * b + 6]);
        std::sort(rounds_seen.begin(), rounds_seen.end());
        for (unsigned long long rmax : rounds_seen) {
        std::vector<int> ids;
        for (int b = 0; b < kTraceBoxes; b++)
            if (br[8 * b + 4] && br[8 * b + 6] == rmax) ids.push_back(b);
        if (!ids.empty()) {
            unsigned long long t0 = ~0ull;
            for (int b : ids) t0 = std::min(t0, br[8 * b]);
            std::sort(ids.begin(), ids.end(), [&](int a, int b) { return br[8 * a + 4] < br[8 * b + 4]; });
            double ph[4] = {0, 0, 0, 0};
            int rows_hist[17] = {0};
            for (int b : ids) {
                for (int k = 0; k < 4; k++) ph[k] += (br[8 * b + k + 1] - br[8 * b + k]) * 1e-3;
                rows_hist[std::min<int>(16, br[8 * b + 5] & 0xff)]++;
            }
            std::fprintf(stderr, "[rb trace] round %llu k_hs_fused boxes %zu: mean us eval %.2f lin %.2f sweep %.2f out %.2f; "
                                 "rows:", (unsigned long long)rmax, ids.size(), ph[0] / ids.size(), ph[1] / ids.size(),
                         ph[2] / ids.size(), ph[3] / ids.size());
            for (int r = 0; r <= 16; r++)
                if (rows_hist[r]) std::fprintf(stderr, " %d:%d", r, rows_hist[r]);
            std::fprintf(stderr, "\n");
            for (int q : {(int)ids.size() / 2, (int)(ids.size() * 9 / 10), (int)ids.size() - 1}) {
                const unsigned long long* x = &br[8 * ids[q]];
                std::fprintf(stderr, "[rb trace]   box %d (end rank %d): start %.2f eval %.2f lin %.2f sweep %.2f out %.2f "
                                     "(to loop end %.2f) end %.2f us, rows %llu kind %llu sm %llu\n",
                             ids[q], q, (x[0] - t0) * 1e-3, (x[1] - x[0]) * 1e-3, (x[2] - x[1]) * 1e-3,
                             (x[3] - x[2]) * 1e-3, (x[4] - x[3]) * 1e-3, x[7] ? (x[7] - x[3]) * 1e-3 : 0.0,
                             (x[4] - t0) * 1e-3, x[5] & 0xff, (x[5] >> 8) & 0xff, x[5] >> 16 & 0xffff);
            }
        }
        }
    }
    ck(cudaMemset(h->d_trace, 0, t.size() * 8), "trace clear");
}

static void launch_filter_phase(rb_handle* h, double target, int round_no = -1) {
    const int n = h->n;
    ck(cudaMemsetAsync(h->d_ctr, 0, sizeof(Counters), h->st), "ctr memset");
    stamp(h, nullptr, round_no, 0);
    record(h, 0);
    if (h->n_cur > 0) dispatch_n<ClassifyK>(n, h, target);
    record(h, 1);
    stamp(h, nullptr, round_no, 1);
    if (h->n_cur > 0) dispatch_n<FilterK>(n, h, h->n_cur, (int64_t*)nullptr);
    record(h, 2);
    stamp(h, nullptr, round_no, 2);
}

// K2 HS (or pass-through) + exact dedup (no sync)
static void launch_hs_phase(rb_handle* h, const HsParams& prm0, bool dedup) {
    HsParams prm = prm0;
    prm.count_from_ctr = 1;
    if (h->n_cur > 0) launch_hs_batches(h, std::min<int64_t>(h->S.cap, h->n_cur << h->n), 0, prm, nullptr);
    record(h, 3);
    stamp(h, nullptr, prm0.round_no, 3);
    if (dedup) dispatch_n<DedupK>(h->n, h, h->F[h->cur ^ 1].f, h->F[h->cur].f);
    stamp(h, nullptr, prm0.round_no, 4);
}

// Capacities for the coming round.  S keeps the largest size a round has
// needed (it grows, with a redo, when a round overflows it); F is sized so that
// it can never overflow: carried rows <= n_cur and HS emits <= 2 rows per survivor.
static void plan_capacity(rb_handle* h, int64_t& need_s, int64_t& need_f) {
    need_s = std::max<int64_t>(h->S.cap, 4096);
    need_f = h->n_cur + 2 * need_s + 1;
}
static void fill_round_out(rb_handle* h, RoundOut& ro) {
    const Counters& c = *h->h_ctr;
    ro.boxes_in = h->n_cur;
    ro.carried = (int64_t)c.n_carried;
    ro.survivors = (int64_t)c.n_surv;
    ro.children = (int64_t)(c.n_par << h->n);
    ro.child_width = bits_to_double(c.child_wmax);
    ro.filter_ops = c.filter_ops;
    ro.exact = (int64_t)c.exact_boxes;
    ro.hs_on = c.hs_on != 0;
    ro.hs_calls = (int64_t)c.hs_calls;
    ro.hs_ops = c.hs_ops;
    ro.width = bits_to_double(c.wmax);
    ro.dups = (int64_t)c.dups;
    ro.after_hs = (int64_t)c.n_next - ro.dups;
}

// After a completed round: make F[cur] the new frontier.
static void commit_round(rb_handle* h, RoundOut& ro) {
    if (ro.dups == 0) h->cur ^= 1;  // else k_dedup_finish compacted into F[cur]
    h->n_cur = ro.after_hs;
}

// One round of bnb.solve (bnb.py:248-337) with a single host sync; buffers that
// turn out too small are grown and the round is redone (the input is untouched).
struct NvtxRange {  // profiler-visible round ranges (ncu --nvtx --nvtx-include "rb_round_5/")
    explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Largest survivor buffer a round may use (a quarter of the engine's memory budget);
// a round with more survivors streams its parents in chunks (run_round_streamed).
static int64_t s_cap_limit(rb_handle* h) {
    return std::max<int64_t>(65536, (int64_t)(h->mem_budget / 4 / (16 * (size_t)h->n)));
}

// One round with its parents processed in chunks (bnb.py:271-313 chunks them by
// batch_size for its thread pool): the chunk's 2^n children per parent fit the survivor
// buffer S, and each chunk's survivors are contracted (or passed through) into F_next
// before the next chunk is filtered, so a round needs S for one chunk and F_next for the
// next frontier -- bounded by max_boxes -- instead of S for every survivor of the round.
// The HS trigger (bnb.py:289-296) depends on the widest survivor of the WHOLE round, so a
// first pass filters every parent without storing (counts + max width only); the chunks
// then run with the decision fixed.  Results are identical to the unchunked round: every
// output row is a function of its parent alone and the frontier is order-free.
static void run_round_streamed(rb_handle* h, double target, const HsParams& prm0, bool dedup, RoundOut& ro) {
    const int n = h->n;
    int64_t scap = h->stream_parents > 0 ? std::max<int64_t>(4096, h->stream_parents << n)
                                         : std::max<int64_t>(h->S.cap, (int64_t)1 << n);
    scap = std::min<int64_t>(scap, std::max<int64_t>(s_cap_limit(h), (int64_t)1 << n));
    surv_reserve(h, scap);
    scap = h->S.cap;
    const int64_t chunk = h->stream_parents > 0 ? h->stream_parents : std::max<int64_t>(1, scap >> n);
    fronts_reserve(h, h->n_cur + 2 * std::min<int64_t>(scap, h->n_cur << n) + 1);
    parents_reserve(h, std::max<int64_t>(h->n_cur, 1));
    // pass 1: classify (carried rows into F_next, the parents list) + a count-only filter
    ck(cudaMemsetAsync(h->d_ctr, 0, sizeof(Counters), h->st), "ctr memset");
    record(h, 0);
    dispatch_n<ClassifyK>(n, h, target);
    record(h, 1);
    const SBuf S0 = h->S;
    h->S.cap = 0;  // nothing stored: n_surv and child_wmax only
    dispatch_n<FilterK>(n, h, h->n_cur, (int64_t*)nullptr);
    h->S = S0;
    record(h, 2);
    sync_counters(h);
    const Counters c1 = *h->h_ctr;
    const int64_t npar = (int64_t)c1.n_par;
    bool hs_on = false;  // hs_count's trigger, on the whole round's survivors
    if (c1.n_surv > 0 && prm0.hs_possible) {
        if (prm0.hs_enable_round >= 0 && prm0.round_no >= prm0.hs_enable_round) hs_on = true;
        if (!std::isnan(prm0.hs_enable_width) && bits_to_double(c1.child_wmax) <= prm0.hs_enable_width) hs_on = true;
    }
    double classify_ms = elapsed(h, 0, 1), filter_ms = 0.0, hs_ms = 0.0;
    // the chunks re-count survivors, filter work and exact boxes
    {
        Counters z = c1;
        z.n_surv = 0;
        z.filter_ops = 0;
        z.exact_boxes = 0;
        ck(cudaMemcpyAsync(h->d_ctr, &z, sizeof(Counters), cudaMemcpyHostToDevice, h->st), "ctr h2d");
    }
    HsParams prm = prm0;
    prm.hs_mode = hs_on ? 1 : 2;
    prm.count_from_ctr = 1;
    int64_t surv_total = 0, n_next = (int64_t)c1.n_next;
    unsigned long long filter_ops = 0, exact = 0;
    for (int64_t p0 = 0; p0 < npar; p0 += chunk) {
        const int64_t pc = std::min<int64_t>(chunk, npar - p0);
        const int64_t worst = std::min<int64_t>(scap, pc << n);
        if (n_next + 2 * worst + 1 > h->F[h->cur ^ 1].f.cap)  // F_next keeps its rows when it grows
            fronts_reserve(h, grow_cap(n_next + 2 * worst + 1), n_next);
        scratch_reserve(h, std::max<int64_t>(1, worst));
        ck(cudaMemsetAsync(&h->d_ctr->n_surv, 0, sizeof(unsigned long long), h->st), "memset");
        record(h, 1);
        dispatch_n<FilterK>(n, h, pc, (int64_t*)nullptr, p0, pc);
        record(h, 2);
        launch_hs_batches(h, worst, 0, prm, nullptr);
        record(h, 3);
        sync_counters(h);
        const Counters& c = *h->h_ctr;
        if (c.n_surv > (unsigned long long)scap) throw ArgError{RB_ERR_STATE, "streamed chunk overflowed S"};
        surv_total += (int64_t)c.n_surv;
        n_next = (int64_t)c.n_next;
        filter_ms += elapsed(h, 1, 2);
        hs_ms += elapsed(h, 2, 3);
    }
    filter_ops = h->h_ctr->filter_ops;
    exact = h->h_ctr->exact_boxes;
    if (dedup) {
        dispatch_n<DedupK>(n, h, h->F[h->cur ^ 1].f, h->F[h->cur].f);
        sync_counters(h);
    }
    fill_round_out(h, ro);
    ro.survivors = surv_total;
    ro.filter_ops = filter_ops;
    ro.exact = (int64_t)exact;
    ro.hs_on = hs_on;
    update_order(h);
    ro.attempts = 1;
    ro.classify_ms = classify_ms;
    ro.filter_ms = filter_ms;
    ro.hs_ms = hs_ms;
}

static void run_round(rb_handle* h, double target, const HsParams& prm, bool dedup, RoundOut& ro) {
    char nv[32];
    std::snprintf(nv, sizeof(nv), "rb_round_%d", prm.round_no);
    NvtxRange range(nv);
    if (h->stream_parents > 0 && h->n_cur > 0) {  // forced (tests): every round in chunks
        run_round_streamed(h, target, prm, dedup, ro);
        return;
    }
    int64_t need_s, need_f;
    plan_capacity(h, need_s, need_f);
    for (int attempt = 1;; attempt++) {
        fronts_reserve(h, need_f);
        surv_reserve(h, need_s);
        parents_reserve(h, std::max<int64_t>(h->n_cur, 1));
        scratch_reserve(h, std::max<int64_t>(1, std::min<int64_t>(h->S.cap, h->n_cur << h->n)));
        launch_filter_phase(h, target, prm.round_no);
        launch_hs_phase(h, prm, dedup);
        record(h, 4);
        stamp(h, nullptr, prm.round_no, 5);
        sync_counters(h);
        const Counters& c = *h->h_ctr;
        if (c.n_surv > (unsigned long long)h->S.cap) {
            need_s = (int64_t)(c.n_surv + c.n_surv / 4);
            if (need_s > s_cap_limit(h)) {  // too many survivors for one buffer: stream the parents
                run_round_streamed(h, target, prm, dedup, ro);
                ro.attempts = attempt + 1;
                return;
            }
            need_f = h->n_cur + 2 * need_s + 1;
            continue;
        }
        if (c.n_next > (unsigned long long)h->F[h->cur ^ 1].f.cap) {  // cannot happen (see plan_capacity)
            need_f = (int64_t)(c.n_next + c.n_next / 4);
            continue;
        }
        fill_round_out(h, ro);
        update_order(h);
        ro.attempts = attempt;
        ro.classify_ms = elapsed(h, 0, 1);
        ro.filter_ms = elapsed(h, 1, 2);
        ro.hs_ms = elapsed(h, 2, 3);
        return;
    }
}

static void graph_release(rb_handle* h) {
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->graph) cudaGraphDestroy(h->graph);
    h->graph_exec = nullptr;
    h->graph = nullptr;
    h->graph_key.clear();
}

// Mapped pinned host blocks, kept by the process and reused across handles
// (pinning host memory costs milliseconds; a new engine for the next system reuses one).
constexpr int64_t kHostSortRows = 16384;  // final sets up to this size are ordered on the host
constexpr int kPinnedRounds = 256;        // round statistics held in the pinned block
static std::mutex g_pin_mu;
static std::vector<std::pair<void*, size_t>> g_pin_free;
static void* pinned_acquire(size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        for (size_t i = 0; i < g_pin_free.size(); i++)
            if (g_pin_free[i].second >= bytes) {
                void* p = g_pin_free[i].first;
                g_pin_free.erase(g_pin_free.begin() + (long)i);
                return p;
            }
    }
    void* p = nullptr;
    ck(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable), "pinned block");
    return p;
}
static void pinned_release(void* p, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.emplace_back(p, bytes);
}

static void release_all(rb_handle* h) {
    h->F[0].release();
    h->F[1].release();
    auto fr = [](void* p) { dfree(p); };
    fr(h->parents);
    fr(h->S.lo);
    fr(h->S.hi);
    fr(h->d_ctr);
    fr(h->d_tags);
    fr(h->d_table);
    fr(h->d_etable);
    fr(h->d_dead);
    fr(h->d_slot);
    fr(h->d_rstats);
    fr(h->d_order);
    fr(h->d_state);
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
    fr(h->d_jc);
    fr(h->W.x);
    fr(h->W.jl);
    fr(h->W.jh);
    fr(h->W.fl);
    fr(h->W.fh);
    fr(h->W.flags);
    fr(h->d_trace);
    fr(h->d_bar);
    fr(h->d_route);
    if (h->st) cudaStreamSynchronize(h->st);  // frees are stream-ordered; the pool is shared
    h->pool = nullptr;
    graph_release(h);
    if (h->hx_stats_own) cudaFreeHost(h->hx_stats_own);
    h->hx_stats_own = nullptr;
    if (h->pin) pinned_release(h->pin, h->pin_bytes);
    h->pin = nullptr;
    h->h_ctr = nullptr;
    h->h_state = nullptr;
    h->hx = nullptr;
    h->hx_stats = nullptr;
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->st) cudaStreamDestroy(h->st);
    if (h->st_side) cudaStreamDestroy(h->st_side);
}

// canonical order of F[cur] rows [0, N) -> result buffers (row-major)

// canonical order of N row-major rows on the host -> hr_* result arrays
static void sort_on_host(rb_handle* h, int64_t N, const double* lo, const double* hi, const uint8_t* c,
                         const uint8_t* u) {
    const int n = h->n;
    std::vector<int64_t> ord(N);
    std::iota(ord.begin(), ord.end(), 0);
    // np.lexsort keys: lo_0..lo_{n-1}, then hi_0..hi_{n-1} (_batch.py:244-250); stable
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        for (int j = 0; j < n; j++) {
            const double x = lo[a * n + j], y = lo[b * n + j];
            if (x < y) return true;
            if (y < x) return false;
        }
        for (int j = 0; j < n; j++) {
            const double x = hi[a * n + j], y = hi[b * n + j];
            if (x < y) return true;
            if (y < x) return false;
        }
        return false;
    });
    h->hr_lo.resize((size_t)N * n);
    h->hr_hi.resize((size_t)N * n);
    h->hr_cert.resize(N);
    h->hr_uns.resize(N);
    for (int64_t r = 0; r < N; r++) {
        std::memcpy(&h->hr_lo[r * n], &lo[ord[r] * n], sizeof(double) * n);
        std::memcpy(&h->hr_hi[r * n], &hi[ord[r] * n], sizeof(double) * n);
        h->hr_cert[r] = c[ord[r]];
        h->hr_uns[r] = u[ord[r]];
    }
    h->r_n = N;
    h->r_on_host = true;
    h->r_ready = true;
}

static void finalize_sorted(rb_handle* h) {
    const int n = h->n;
    const int64_t N = h->n_cur;
    Front f = h->F[h->cur].f;
    if (h->cap_r < std::max<int64_t>(N, 1)) {
        const int64_t cap = grow_cap(std::max<int64_t>(N, 1));
        dalloc(&h->r_lo, (size_t)cap * n);
        dalloc(&h->r_hi, (size_t)cap * n);
        dalloc(&h->r_cert, (size_t)cap);
        dalloc(&h->r_uns, (size_t)cap);
        h->cap_r = cap;
    }
    h->r_n = N;
    h->r_ready = true;
    h->r_on_host = false;
    if (N == 0) return;
    if (N <= kHostSortRows) {
        // small final sets: one gather + D2H, then canonical order on the host
        // (cheaper than 2n radix passes of launch latency)
        h->launches++;
        k_gather_rows<<<grid_for(N, 256, h->sms * 8), 256, 0, h->st>>>(f, n, N, nullptr, h->r_lo, h->r_hi,
                                                                        h->r_cert, h->r_uns);
        ck(cudaGetLastError(), "gather");
        ck(cudaMemcpyAsync(h->hx_lo, h->r_lo, sizeof(double) * N * n, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaMemcpyAsync(h->hx_hi, h->r_hi, sizeof(double) * N * n, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaMemcpyAsync(h->hx_c, h->r_cert, N, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaMemcpyAsync(h->hx_u, h->r_uns, N, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaStreamSynchronize(h->st), "finalize sync");
        sort_on_host(h, N, h->hx_lo, h->hx_hi, h->hx_c, h->hx_u);
        return;
    }
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
        h->launches++;
        k_iota<<<blocks, 256, 0, h->st>>>(h->d_perm[0], N);
        // LSD over the 2n keys of np.lexsort order: least significant first (hi_{n-1}), most
        // significant last (lo_0); each pass is a stable radix sort.
        int cur = 0;
        for (int k = 2 * n - 1; k >= 0; k--) {
            h->launches++;
            k_sort_keys<<<blocks, 256, 0, h->st>>>(f, n, N, k, h->d_perm[cur], h->d_keys[0]);
            size_t bytes = h->cub_bytes;
            ck(cub::DeviceRadixSort::SortPairs(h->d_cub, bytes, h->d_keys[0], h->d_keys[1], h->d_perm[cur],
                                               h->d_perm[cur ^ 1], (int)N, 0, 64, h->st),
               "radix sort");
            cur ^= 1;
        }
        perm = h->d_perm[cur];
    }
    h->launches++;
    k_gather_rows<<<grid_for(N, 256, h->sms * 8), 256, 0, h->st>>>(f, n, N, perm, h->r_lo, h->r_hi, h->r_cert,
                                                                    h->r_uns);
    ck(cudaGetLastError(), "gather");
    ck(cudaStreamSynchronize(h->st), "finalize sync");
}

static double now_s() {
    using namespace std::chrono;
    return duration<double>(steady_clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------- device round loop

// Rounds whose worst case (n_cur * 2^n children) fits the survivor buffer run
// inside one CUDA graph: a WHILE node whose body is one round (classify, filter,
// HS, dedup, settle, k_round_end).  No host round trip per round; the frontier
// always comes back to F[0] (k_settle), so the body's parameters are fixed.
static int64_t graph_small_cap(int n) {
    int64_t c = (int64_t)1 << std::min(30, n + 10);
    return std::min<int64_t>(std::max<int64_t>(c, (int64_t)1 << 16), (int64_t)1 << 18);
}



static void build_round_graph(rb_handle* h, const HsParams& prm, bool dedup, int64_t scap,
                              const std::vector<uintptr_t>& key) {
    graph_release(h);
    const int n = h->n;
    cudaGraph_t g = nullptr;
    ck(cudaGraphCreate(&g, 0), "graph create");
    cudaGraphConditionalHandle hw;
    ck(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault), "cond handle");
    const bool fused_hs = h->graph_fused_only && h->hs_fused;
    // exact dedup at append time needs every appender to insert: classify / k_classify_filter
    // (carried rows) and k_hs_fused (HS outputs, pass-through)
    const bool append_dedup = dedup && fused_hs && h->append_dedup;
    const bool cf = h->graph_cf && !(h->meta.ftab && h->use_ftab);
    // ping-pong rounds: round u reads F[u & 1] and writes F[u & 1 ^ 1]; the last k_hs_fused
    // block ends the round (no round-tail kernel, no frontier copy), duplicates go through
    // the epoch table (no cleanup pass), and one small kernel per U rounds sets the WHILE
    // condition.  Needs the fused HS, the classify-filter kernel and dedup at append time.
    const bool pp = h->pingpong && cf && fused_hs && (append_dedup || !dedup);
    const int U_pp = std::max(2, h->graph_unroll + (h->graph_unroll & 1));
    auto pp_rounds = [&]() {
        DedupCtx de{};
        if (dedup) de = DedupCtx{nullptr, (unsigned long long)(h->table_slots - 1), h->d_slot, h->d_dead, h->d_etable,
                                 (const DevState*)h->d_state};
        for (int u = 0; u < U_pp; u++) {
            h->cur = u & 1;
            stamp(h, h->d_state, 0, 0);
            dispatch_n<ClassifyFilterK>(n, h, de, scap);
            stamp(h, h->d_state, 0, 1);
            stamp(h, h->d_state, 0, 2);
            HsParams p = prm;
            p.count_from_ctr = 1;
            p.st = h->d_state;
            p.dd = de;
            p.fused_max = LLONG_MAX;
            p.has_cond = 0;
            p.round_end = 1;
            p.rstats = h->d_rstats;
            p.eq_order = h->d_order;
            p.s_cap = scap;
            dispatch_n<HsFusedK>(n, h, (int64_t)0, p, (int64_t*)nullptr, scap);
            stamp(h, h->d_state, 0, 3);
            stamp(h, h->d_state, 0, 4);
            stamp(h, h->d_state, 0, 6, -1);
        }
        k_set_cond<<<1, 32, 0, h->st>>>(h->d_state, hw);
        ck(cudaGetLastError(), "set cond launch");
        h->launches++;
        h->cur = 0;
    };
    // top level: k_solve_start -> [U rounds] -> WHILE(U rounds) -> k_solve_finish; the first U
    // rounds sit before the loop, so a solve that ends in them never pays for a WHILE iteration
    ck(cudaStreamBeginCaptureToGraph(h->st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
       "begin capture");
    {
        InitBox box{};
        for (int j = 0; j < n; j++) {
            box.lo[j] = h->init_lo[j];
            box.hi[j] = h->init_hi[j];
        }
        stamp(h, nullptr, kTraceRounds - 1, 0);
        k_solve_start<<<1, 32, 0, h->st>>>(h->d_state, h->hx_dev, h->F[0].f, h->d_ctr, h->d_order, box, n);
        ck(cudaGetLastError(), "start launch");
        stamp(h, nullptr, kTraceRounds - 1, 1);
    }
    if (h->use_mk) dispatch_n<SmallRoundsK>(n, h, prm, dedup, scap, hw);
    const int64_t l_pro = h->launches;
    if (pp && h->graph_prologue) pp_rounds();
    h->launches = l_pro;
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t cg = nullptr;
    ck(cudaStreamGetCaptureInfo(h->st, &cs, nullptr, &cg, &deps, &ndeps), "capture info");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hw;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    ck(cudaGraphAddNode(&node, cg, deps, ndeps, &cp), "while node");
    ck(cudaStreamUpdateCaptureDependencies(h->st, &node, 1, cudaStreamSetCaptureDependencies), "capture deps");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    stamp(h, nullptr, kTraceRounds - 1, 2);
    k_solve_finish<<<grid_for(kHostSortRows, 256, h->sms * 4), 256, 0, h->st>>>(
        h->d_state, h->d_rstats, h->d_order, h->hx_dev, h->hx_stats_dev, h->F[0].f, h->F[1].f, n, (long long)kHostSortRows,
        h->hx_lo_dev, h->hx_hi_dev, h->hx_c_dev, h->hx_u_dev);
    ck(cudaGetLastError(), "finish launch");
    stamp(h, nullptr, kTraceRounds - 1, 3);
    {
        cudaGraph_t top = nullptr;
        ck(cudaStreamEndCapture(h->st, &top), "end capture");
    }
    ck(cudaStreamBeginCaptureToGraph(h->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
       "begin capture");
    const int64_t l0 = h->launches;
    h->cur = 0;
    const int64_t fcap = h->F[0].f.cap;
    // U rounds per WHILE iteration: an iteration costs ~5 us on B200 (tools/microbench/
    // graph_nodes.cu) against ~0.8 us per kernel node, so rounds are unrolled; the
    // rounds after the one that ends the solve find st->done / st->bail and exit at once.
    DedupCtx dd{};
    if (append_dedup) dd = DedupCtx{h->d_table, (unsigned long long)(h->table_slots - 1), h->d_slot, h->d_dead};
    if (pp) pp_rounds();
    for (int u = 0; u < (pp ? 0 : h->graph_unroll); u++) {
        stamp(h, h->d_state, 0, 0);
        if (cf) {
            dispatch_n<ClassifyFilterK>(n, h, dd, scap);
            stamp(h, h->d_state, 0, 1);
        } else {
            dispatch_n<ClassifyK>(n, h, 0.0, (const DevState*)h->d_state, std::min<int64_t>(fcap, scap), dd);
            stamp(h, h->d_state, 0, 1);
            dispatch_n<FilterK>(n, h, std::max<int64_t>(1, scap >> n), (int64_t*)nullptr);
        }
        stamp(h, h->d_state, 0, 2);
        HsParams p = prm;
        p.count_from_ctr = 1;
        p.st = h->d_state;
        p.dd = dd;
        if (fused_hs) {  // no early-exit eval/lin/sweep nodes in the round
            p.fused_max = LLONG_MAX;
            p.has_cond = 0;
            dispatch_n<HsFusedK>(n, h, (int64_t)0, p, (int64_t*)nullptr, scap);
        } else {
            launch_hs_batches(h, scap, 0, p, nullptr);
        }
        stamp(h, h->d_state, 0, 3);
        if (dedup && !append_dedup) dispatch_n<DedupInsertK>(n, h, h->F[1].f);
        stamp(h, h->d_state, 0, 4);
        dispatch_n<TailK>(n, h, dedup, std::min<int64_t>(fcap, 3 * scap), scap, hw);
        stamp(h, h->d_state, 0, 6, -1);
    }
    h->launches++;
    cudaGraph_t captured = nullptr;
    ck(cudaStreamEndCapture(h->st, &captured), "end capture");
    h->graph_launches_per_iter = h->launches - l0;
    h->graph_rounds_per_iter = pp ? U_pp : h->graph_unroll;
    h->launches = l0;
    ck(cudaGraphInstantiate(&h->graph_exec, g, 0), "graph instantiate");
    h->graph = g;
    h->graph_key = key;
}

// Runs rounds on the device while they fit; returns true when the solve finished
// (status in *status), false when the host must continue from h->stats.size() + 1.
static bool graph_rounds(rb_handle* h, const rb_config* cfg, double target, bool hs_possible, int* status) {
    const int n = h->n;
    int64_t scap = graph_small_cap(n);
    surv_reserve(h, scap);
    scap = std::min<int64_t>(h->S.cap, (int64_t)1 << 20);
    scratch_reserve(h, scap);
    if (h->W.B < scap) scap = h->W.B;
    fronts_reserve(h, (scap >> n) + 2 * scap + 1);
    parents_reserve(h, std::max<int64_t>(1, (scap >> n) + 1));
    if (h->cap_rstats < cfg->max_rounds) {
        dalloc(&h->d_rstats, (size_t)cfg->max_rounds);
        h->cap_rstats = cfg->max_rounds;
    }
    if (h->cap_hx_stats < cfg->max_rounds) {  // beyond the pinned block's kPinnedRounds
        if (h->hx_stats_own) ck(cudaFreeHost(h->hx_stats_own), "free mapped stats");
        h->hx_stats_own = nullptr;
        ck(cudaHostAlloc((void**)&h->hx_stats_own, sizeof(DevRoundStats) * cfg->max_rounds, cudaHostAllocMapped),
           "mapped stats");
        h->hx_stats = h->hx_stats_own;
        ck(cudaHostGetDevicePointer((void**)&h->hx_stats_dev, h->hx_stats, 0), "mapped ptr");
        h->cap_hx_stats = cfg->max_rounds;
    }
    if (!h->d_state) dalloc(&h->d_state, 1);
    if (h->pingpong && (h->cap_etable < h->table_slots || !h->d_etable)) {  // epoch dedup table, zero = epoch 0
        dalloc(&h->d_etable, h->table_slots);
        ck(cudaMemsetAsync(h->d_etable, 0, h->table_slots * sizeof(unsigned long long), h->st), "etable memset");
        h->cap_etable = h->table_slots;
        h->epoch_next = 1;
    }
    HsParams prm{};
    prm.hs_mode = 0;
    prm.hs_enable_round = cfg->hs_enable_round;
    prm.hs_possible = hs_possible ? 1 : 0;
    prm.hs_enable_width = cfg->hs_enable_width;
    prm.contract_output = cfg->hs_contract ? 1 : 0;
    const bool dedup = cfg->exact_round_dedup != 0;
    uint64_t hw_bits;
    std::memcpy(&hw_bits, &cfg->hs_enable_width, 8);
    std::vector<uintptr_t> key = {
        (uintptr_t)h->F[0].f.lo, (uintptr_t)h->F[0].f.hi, (uintptr_t)h->F[0].f.cert, (uintptr_t)h->F[0].f.unsplit,
        (uintptr_t)h->F[1].f.lo, (uintptr_t)h->F[1].f.hi, (uintptr_t)h->F[1].f.cert, (uintptr_t)h->F[1].f.unsplit,
        (uintptr_t)h->F[0].f.cap, (uintptr_t)h->F[1].f.cap, (uintptr_t)h->S.lo, (uintptr_t)h->S.hi,
        (uintptr_t)h->S.cap, (uintptr_t)h->parents, (uintptr_t)h->W.x, (uintptr_t)h->W.jl, (uintptr_t)h->W.jh,
        (uintptr_t)h->W.fl, (uintptr_t)h->W.fh, (uintptr_t)h->W.flags, (uintptr_t)h->W.B, (uintptr_t)h->d_table,
        (uintptr_t)h->table_slots, (uintptr_t)h->d_slot, (uintptr_t)h->d_dead, (uintptr_t)h->d_rstats,
        (uintptr_t)h->d_state, (uintptr_t)scap, (uintptr_t)dedup, (uintptr_t)prm.hs_enable_round,
        (uintptr_t)prm.hs_possible, (uintptr_t)hw_bits, (uintptr_t)prm.contract_output,
        (uintptr_t)(h->use_ftab ? 1 : 0), (uintptr_t)(h->hs_fused ? 1 : 0), (uintptr_t)h->fused_rows,
        (uintptr_t)(h->use_fwt ? 1 : 0), (uintptr_t)(h->jconst ? 1 : 0)};
    key.push_back((uintptr_t)h->hs_cond);
    key.push_back((uintptr_t)h->graph_unroll);
    key.push_back((uintptr_t)h->graph_fused_only);
    key.push_back((uintptr_t)h->graph_cf);
    key.push_back((uintptr_t)h->pingpong);
    key.push_back((uintptr_t)h->graph_prologue);
    key.push_back((uintptr_t)h->d_etable);
    key.push_back((uintptr_t)(h->tail_blocks_per_sm * 64));
    key.push_back((uintptr_t)gen_on(h));
    key.push_back((uintptr_t)h->append_dedup);
    key.push_back((uintptr_t)h->use_mk);
    key.push_back((uintptr_t)h->mk_cap);
    key.push_back((uintptr_t)h->mk_bps);
    key.push_back((uintptr_t)h->hx_stats_dev);
    key.push_back((uintptr_t)h->pdl);
    key.push_back((uintptr_t)h->trace);
    key.push_back((uintptr_t)h->force_exact);
    key.push_back((uintptr_t)h->hs_tile);
    key.push_back((uintptr_t)h->lin_tpb);
    if (key != h->graph_key || !h->graph_exec) build_round_graph(h, prm, dedup, scap, key);
    DevState st{};
    st.n_cur = 1;
    st.target = target;
    st.max_boxes = cfg->max_boxes;
    st.round_no = 1;
    st.max_rounds = cfg->max_rounds;
    st.status = RB_BUDGET_EXHAUSTED;
    st.cur = 0;
    st.epoch = h->epoch_next;
    HostX& X = *h->hx;
    st.finish_blocks = 0;
    // process-wide sequence: the pinned block of a destroyed handle is reused by the next
    // one, whose HostX may still hold an old done_seq
    static std::atomic<unsigned long long> g_solve_seq{0};
    st.seq = ++g_solve_seq;
    h->solve_seq = st.seq;
    X.done_seq = 0;
    X.start = st;
    X.rows = -1;
    if (h->trace) X.state.nrounds = -7;  // sentinel for the visibility measurement below
    std::atomic_thread_fence(std::memory_order_seq_cst);
    const double tg0 = now_s();
    ck(cudaGraphLaunch(h->graph_exec, h->st), "graph launch");
    // end-of-device-work event in the same stream pass: a solve that finishes inside the
    // graph needs no second record + synchronise round trip (solve_impl)
    ck(cudaEventRecord(h->ev[6], h->st), "ev end");
    h->ev_end_valid = true;
    const double tg1 = now_s();
    double tflag = 0.0;
    if (h->trace) {  // when the finish kernel's state write becomes visible to the host (measurement only)
        const volatile int* nr = &X.state.nrounds;
        while (*nr == -7 && now_s() - tg1 < 0.1) {
        }
        tflag = now_s();
    }
    h->graph_fast_return = false;
    if (!h->device_timing) {
        // spin on the completion flag the finish kernel publishes after its mapped writes;
        // the stream is polled now and then so a fault or an early end is still seen
        const volatile unsigned long long* ds = &X.done_seq;
        for (unsigned it = 1;; it++) {
            if (*ds == st.seq) {
                h->graph_fast_return = true;
                break;
            }
            if ((it & 1023u) == 0) {
                const cudaError_t e = cudaStreamQuery(h->st);
                if (e == cudaSuccess) break;
                if (e != cudaErrorNotReady) ck(e, "graph");
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    }
    if (!h->graph_fast_return) ck(cudaStreamSynchronize(h->st), "graph sync");
    const double tg2 = now_s();
    if (h->trace)
        std::fprintf(stderr, "[rb trace] host: solve start -> graph launch %.1f us, launch call %.1f us, sync %.1f us "
                             "(state visible after %.1f us)\n",
                     (tg0 - h->t_solve0) * 1e6, (tg1 - tg0) * 1e6, (tg2 - tg1) * 1e6, (tflag - tg1) * 1e6);
    const DevState r = X.state;
    const int first = (int)h->stats.size();
    const int nr = r.nrounds - first;
    for (int i = 0; i < nr; i++) {
        const DevRoundStats& x = h->hx_stats[first + i];
        rb_round_stats o{};
        o.round = (int32_t)x.round;
        o.hs_on = (int32_t)x.hs_on;
        o.boxes_in = x.boxes_in;
        o.boxes_after_filter = x.after_filter;
        o.boxes_after_hs = x.after_hs;
        o.width = x.width;
        o.elapsed_seconds = x.elapsed;
        o.children = x.children;
        o.hs_calls = x.hs_calls;
        o.filter_ops = x.filter_ops;
        o.hs_ops = x.hs_ops;
        o.dups = x.dups;
        o.exact_boxes = x.exact;
        o.attempts = 1;
        o.classify_bytes = x.boxes_in * (16 * n + 2);
        h->stats.push_back(o);
    }
    {
        const int U = h->graph_rounds_per_iter;
        h->launches += (int64_t)((nr + U - 1) / U) * h->graph_launches_per_iter + 2;
    }
    h->cur = r.cur;  // ping-pong rounds leave the frontier in F[cur]
    h->epoch_next = r.epoch + 1;
    h->n_cur = (int64_t)r.n_cur;
    for (int k = 0; k < 16; k++) h->h_order[k] = X.order[k];
    if (r.done && X.rows >= 0) sort_on_host(h, X.rows, h->hx_lo, h->hx_hi, h->hx_c, h->hx_u);
    if (r.done) *status = r.status;
    return r.done != 0;
}

static void solve_impl(rb_handle* h, const rb_config* cfg, rb_result_info* info) {
    const int n = h->n;
    const double t_start = now_s();
    h->t_solve0 = t_start;
    h->launches = 0;
    ck(cudaEventRecord(h->ev[5], h->st), "ev start");
    h->stats.clear();
    h->have_result = false;
    h->r_ready = false;
    h->ev_end_valid = false;
    if (cfg->max_rounds < 1) throw ArgError{RB_ERR_ARG, "max_rounds must be at least 1"};
    if (cfg->max_boxes < 1) throw ArgError{RB_ERR_ARG, "max_boxes must be at least 1"};
    h->cur = 0;
    h->n_cur = 0;
    fronts_reserve(h, 4096);
    // initial frontier = the initial box (bnb.py:229-232); the device round loop writes it itself
    auto host_init = [&]() {
        reset_order(h);
        Front f = h->F[0].f;
        ck(cudaMemcpy2DAsync(f.lo, f.cap * sizeof(double), h->init_lo.data(), sizeof(double), sizeof(double), n,
                             cudaMemcpyHostToDevice, h->st), "init lo");
        ck(cudaMemcpy2DAsync(f.hi, f.cap * sizeof(double), h->init_hi.data(), sizeof(double), sizeof(double), n,
                             cudaMemcpyHostToDevice, h->st), "init hi");
        ck(cudaMemsetAsync(f.cert, 0, 1, h->st), "init cert");
        ck(cudaMemsetAsync(f.unsplit, 0, 1, h->st), "init uns");
    };
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
    bool finished = false;
    if (init_width <= target) {
        host_init();
        status = RB_WIDTH_REACHED;
        finished = true;
    } else if (h->use_graph && !has_max_seconds && h->stream_parents == 0) {
        finished = graph_rounds(h, cfg, target, hs_possible, &status);
    } else {
        host_init();
    }
    if (!finished) {
        h->ev_end_valid = false;  // host-driven rounds follow
        for (int round_no = (int)h->stats.size() + 1; round_no <= cfg->max_rounds; round_no++) {
            const double t0 = now_s();
            RoundOut ro{};
            HsParams prm{};
            prm.round_no = round_no;
            prm.hs_mode = 0;
            prm.hs_enable_round = cfg->hs_enable_round;
            prm.hs_possible = hs_possible ? 1 : 0;
            prm.hs_enable_width = cfg->hs_enable_width;
            prm.contract_output = cfg->hs_contract ? 1 : 0;
            run_round(h, target, prm, cfg->exact_round_dedup != 0, ro);
            commit_round(h, ro);
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
            st.attempts = ro.attempts;
            // classify reads every row (16n + 2 B) and writes carried rows (16n + 2 B) + 4 B per parent
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
    if (!h->r_ready) {
        h->ev_end_valid = false;
        finalize_sorted(h);
    }
    if (h->trace) std::fprintf(stderr, "[rb trace] host: solve total %.1f us\n", (now_s() - t_start) * 1e6);
    trace_report(h, (int)h->stats.size());
    float dev_ms = -1.f;
    if (h->graph_fast_return && h->ev_end_valid && h->r_ready && h->r_on_host) {
        // the graph finished the solve and its results are on the host: no stream wait
        // (the events complete on their own; device time is not measured in this mode)
    } else {
        if (!h->ev_end_valid) ck(cudaEventRecord(h->ev[6], h->st), "ev end");
        ck(cudaEventSynchronize(h->ev[6]), "ev sync");
        cudaEventElapsedTime(&dev_ms, h->ev[5], h->ev[6]);
    }
    h->ev_end_valid = false;
    h->graph_fast_return = false;
    h->have_result = true;
    if (info) {
        info->device_ms = dev_ms;
        info->kernel_launches = h->launches;
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

static rbg::SystemTerms terms_of(const rb_system* sys) {
    rbg::SystemTerms t;
    t.n = sys->n;
    const int P = sys->n + sys->n * sys->n;
    t.poly_off.assign(sys->poly_off, sys->poly_off + P + 1);
    const int T = sys->poly_off[P];
    t.coeff.assign(sys->coeff, sys->coeff + T);
    t.fac_off.assign(sys->fac_off, sys->fac_off + T + 1);
    const int Fc = sys->fac_off[T];
    t.fac_var.assign(sys->fac_var, sys->fac_var + Fc);
    t.fac_exp.assign(sys->fac_exp, sys->fac_exp + Fc);
    return t;
}

static int codegen_mode() {  // 0 off, 1 background compile on a cache miss, 2 synchronous
    const char* e = std::getenv("RB_CODEGEN");
    if (e && e[0] == '0') return 0;
    if (e && (e[0] == 's' || e[0] == '2')) return 2;
    return 1;
}

// Specialised kernels for this system (compiled once per machine, cached on disk).
// A cached system loads at once; otherwise NVRTC compiles it on a background
// thread while the table kernels run, and the specialised ones take over at the
// next API call after it finishes (codegen_poll).  Both are device code with
// identical results; rb_codegen_active reports which one is in use.
static void codegen_setup(rb_handle* h, const rb_system* sys) {
    h->terms = terms_of(sys);
    const int mode = codegen_mode();
    if (mode == 0) {
        h->gen_err = "disabled (RB_CODEGEN=0)";
        return;
    }
    rbg::Compiled c;
    std::string err;
    if (rbg::cached(h->terms, c) || (mode == 2 && rbg::compile(h->terms, c, err))) {
        if (!rbg::load(c, h->dev, h->gen, err)) {
            h->gen = rbg::Loaded{};
            h->gen_err = err;
        }
        return;
    }
    if (mode == 2) {
        h->gen_err = err;
        return;
    }
    h->gen_err = "compiling";
    h->gen_pending = true;
    const rbg::SystemTerms t = h->terms;
    h->gen_job = std::async(std::launch::async, [t]() {
        std::pair<bool, rbg::Compiled> r;
        std::string e;
        r.first = rbg::compile(t, r.second, e);
        if (!r.first) r.second.key = e;  // carries the reason
        return r;
    });
}

// take over the specialised kernels once the background compile is done (or wait for it)
static void codegen_poll(rb_handle* h, bool wait = false) {
    if (!h->gen_pending) return;
    if (!wait && h->gen_job.wait_for(std::chrono::seconds(0)) != std::future_status::ready) return;
    std::pair<bool, rbg::Compiled> r = h->gen_job.get();
    h->gen_pending = false;
    std::string err;
    if (!r.first) {
        h->gen_err = r.second.key;
        return;
    }
    if (!rbg::load(r.second, h->dev, h->gen, err)) {
        h->gen = rbg::Loaded{};
        h->gen_err = err;
        return;
    }
    h->gen_err.clear();
    gen_configure(h);
}

int rb_codegen_prepare(const rb_system* sys, char* err, int64_t err_len) {
    if (!sys) return RB_ERR_ARG;
    if (sys->n < 1 || sys->n > RB_MAX_DIM) return RB_ERR_LIMIT;
    rbg::Compiled c;
    std::string e;
    if (!rbg::compile(terms_of(sys), c, e)) {
        if (err && err_len > 0) std::snprintf(err, (size_t)err_len, "%s", e.c_str());
        return RB_ERR_CUDA;
    }
    if (err && err_len > 0) std::snprintf(err, (size_t)err_len, "%s", c.key.c_str());  // cache key on success
    return RB_OK;
}

int rb_codegen_active(rb_handle* h, char* why, int64_t why_len) {
    if (!h) return RB_ERR_ARG;
    if (why && why_len > 0) std::snprintf(why, (size_t)why_len, "%s", h->gen.ok ? "" : h->gen_err.c_str());
    return gen_on(h) ? 1 : 0;
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
        const double tc0 = now_s();
        ck(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking), "stream");
        ck(cudaStreamCreateWithFlags(&h->st_side, cudaStreamNonBlocking), "stream");
        h->fused_rows = (int64_t)h->sms * 80;  // measured crossover, tools/hs_ab.py
        if (const char* tr = std::getenv("RB_TRACE")) h->trace = tr[0] == '1';
        h->pool = device_pool(device);  // process-wide per device: memory outlives handles
        PoolScope ps(h);
        for (auto& e : h->ev) ck(cudaEventCreate(&e), "event");
        const double tc1 = now_s();
        build_tables(h, sys);
        const double tc2 = now_s();
        size_t free_b = 0, total_b = 0;
        ck(cudaMemGetInfo(&free_b, &total_b), "meminfo");
        h->mem_budget = (size_t)(0.80 * (double)free_b);
        h->mem_budget_default = h->mem_budget;
        dalloc(&h->d_ctr, 1);
        dalloc(&h->d_bar, 2);
        ck(cudaMemsetAsync(h->d_bar, 0, 2 * sizeof(unsigned), h->st), "barrier clear");
        if (h->trace) {
            dalloc(&h->d_trace, kTraceWords);
            ck(cudaMemsetAsync(h->d_trace, 0, kTraceWords * 8, h->st), "trace clear");
        }
        dalloc(&h->d_order, 16);
        reset_order(h);
        const double tc3 = now_s();
        // one mapped pinned block (reused across handles): counters, state, the graph's
        // start/readback area, kPinnedRounds of statistics and up to kHostSortRows result rows
        {
            size_t off = 0;
            auto take = [&](size_t bytes) {
                const size_t o = off;
                off = (off + bytes + 127) & ~size_t(127);  // Counters is 128-byte aligned
                return o;
            };
            const size_t o_ctr = take(sizeof(Counters)), o_state = take(sizeof(DevState)), o_hx = take(sizeof(HostX));
            const size_t o_stats = take(sizeof(DevRoundStats) * kPinnedRounds);
            const size_t o_lo = take(sizeof(double) * kHostSortRows * h->n);
            const size_t o_hi = take(sizeof(double) * kHostSortRows * h->n);
            const size_t o_c = take(kHostSortRows), o_u = take(kHostSortRows);
            h->pin_bytes = off;
            h->pin = static_cast<uint8_t*>(pinned_acquire(off));
            uint8_t* dev = nullptr;
            ck(cudaHostGetDevicePointer((void**)&dev, h->pin, 0), "mapped ptr");
            h->h_ctr = reinterpret_cast<Counters*>(h->pin + o_ctr);
            h->h_state = reinterpret_cast<DevState*>(h->pin + o_state);
            h->hx = reinterpret_cast<HostX*>(h->pin + o_hx);
            h->hx_dev = reinterpret_cast<HostX*>(dev + o_hx);
            h->hx_stats = reinterpret_cast<DevRoundStats*>(h->pin + o_stats);
            h->hx_stats_dev = reinterpret_cast<DevRoundStats*>(dev + o_stats);
            h->cap_hx_stats = kPinnedRounds;
            h->hx_lo = reinterpret_cast<double*>(h->pin + o_lo);
            h->hx_lo_dev = reinterpret_cast<double*>(dev + o_lo);
            h->hx_hi = reinterpret_cast<double*>(h->pin + o_hi);
            h->hx_hi_dev = reinterpret_cast<double*>(dev + o_hi);
            h->hx_c = h->pin + o_c;
            h->hx_c_dev = dev + o_c;
            h->hx_u = h->pin + o_u;
            h->hx_u_dev = dev + o_u;
        }
        const double tc4 = now_s();
        codegen_setup(h, sys);
        const double tc5 = now_s();
        dispatch_n<SetupK>(h->n, h);
        if (h->trace)
            std::fprintf(stderr, "[rb trace] create: streams/events %.2f ms, tables %.2f ms, buffers %.2f ms, pinned %.2f ms, "
                                 "codegen %.2f ms (%s), kernel setup %.2f ms\n", (tc1 - tc0) * 1e3, (tc2 - tc1) * 1e3,
                         (tc3 - tc2) * 1e3, (tc4 - tc3) * 1e3, (tc5 - tc4) * 1e3,
                         h->gen.ok ? "specialised kernels" : h->gen_err.c_str(), (now_s() - tc5) * 1e3);
        *out = h;
        return RB_OK;
    } catch (const CudaError& ce) {
        g_create_error = std::string(ce.what) + ": " + cudaGetErrorString(ce.e);
        cudaGetLastError();
    } catch (const ArgError& ae) {
        g_create_error = ae.msg;
        {
            PoolScope ps(h);
            release_all(h);
        }
        delete h;
        return ae.code;
    }
    {
        PoolScope ps(h);
        release_all(h);
    }
    delete h;
    return RB_ERR_CUDA;
}

int rb_solve(rb_handle* h, const rb_config* cfg, rb_result_info* info) {
    if (!h || !cfg) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
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
        codegen_poll(h);
        PoolScope ps(h);
        const int64_t N = h->r_n;
        if (N > 0 && h->r_on_host) {
            if (lo) std::memcpy(lo, h->hr_lo.data(), sizeof(double) * N * h->n);
            if (hi) std::memcpy(hi, h->hr_hi.data(), sizeof(double) * N * h->n);
            if (cert) std::memcpy(cert, h->hr_cert.data(), N);
            if (unsplit) std::memcpy(unsplit, h->hr_uns.data(), N);
        } else if (N > 0) {
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
        codegen_poll(h);
        PoolScope ps(h);
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
        codegen_poll(h);
        PoolScope ps(h);
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
        launch_hs_batches(h, M, M, prm, h->d_tags);
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

int rb_krawczyk(rb_handle* h, const double* lo, const double* hi, int64_t M, double* olo, double* ohi,
                uint8_t* ok) {
    if (!h || M < 0 || (M > 0 && (!lo || !hi || !olo || !ohi || !ok))) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    h->have_result = false;
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        const int n = h->n;
        if (M == 0) return RB_OK;
        for (int64_t k = 0; k < M * n; k++)  // hansen.py:154-155
            if (!std::isfinite(lo[k]) || !std::isfinite(hi[k])) throw ArgError{RB_ERR_ARG, "box must be bounded"};
        surv_reserve(h, M);
        Front sview{h->S.lo, h->S.hi, nullptr, nullptr, h->S.cap};
        DevFront tmp;
        tmp.f = sview;
        load_rows(h, tmp, 0, lo, hi, nullptr, nullptr, M);
        h->cur = 0;
        DevFront& out = h->F[1];
        front_reserve(h, out, M, 0);
        scratch_reserve(h, M);
        ck(cudaMemsetAsync(h->d_ctr, 0, sizeof(Counters), h->st), "ctr memset");
        for (int64_t b0 = 0; b0 < M; b0 += h->W.B)
            dispatch_n<KrawczykK>(n, h, b0, std::min<int64_t>(M, b0 + h->W.B), out.f, out.f.cert);
        std::vector<double> slo((size_t)M * n), shi((size_t)M * n);
        for (int j = 0; j < n; j++) {
            ck(cudaMemcpyAsync(slo.data() + (size_t)j * M, out.f.lo + (size_t)j * out.f.cap, sizeof(double) * M,
                               cudaMemcpyDeviceToHost, h->st), "d2h");
            ck(cudaMemcpyAsync(shi.data() + (size_t)j * M, out.f.hi + (size_t)j * out.f.cap, sizeof(double) * M,
                               cudaMemcpyDeviceToHost, h->st), "d2h");
        }
        ck(cudaMemcpyAsync(ok, out.f.cert, M, cudaMemcpyDeviceToHost, h->st), "d2h");
        ck(cudaStreamSynchronize(h->st), "sync");
        const double qnan = std::numeric_limits<double>::quiet_NaN();
        for (int64_t r = 0; r < M; r++)
            for (int j = 0; j < n; j++) {
                olo[r * n + j] = ok[r] ? slo[(size_t)j * M + r] : qnan;
                ohi[r * n + j] = ok[r] ? shi[(size_t)j * M + r] : qnan;
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
        PoolScope ps(h);
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
        codegen_poll(h);
        PoolScope ps(h);
        h->cur = 0;
        h->n_cur = 0;
        fronts_reserve(h, std::max<int64_t>(N, 1));
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
        codegen_poll(h);
        PoolScope ps(h);
        int64_t need_s, need_f;
        plan_capacity(h, need_s, need_f);
        for (;;) {
            fronts_reserve(h, need_f);
            surv_reserve(h, need_s);
            parents_reserve(h, std::max<int64_t>(h->n_cur, 1));
            launch_filter_phase(h, h->shard_target);
            sync_counters(h);
            if (h->h_ctr->n_surv > (unsigned long long)h->S.cap) {
                need_s = (int64_t)(h->h_ctr->n_surv + h->h_ctr->n_surv / 4);
                need_f = h->n_cur + 2 * need_s + 1;
                continue;
            }
            break;
        }
        h->shard_round = round_no;
        h->shard_need_f = need_f;
        update_order(h);
        const Counters& c = *h->h_ctr;
        if (carried) *carried = (int64_t)c.n_carried;
        if (survivors) *survivors = (int64_t)c.n_surv;
        if (child_width) *child_width = bits_to_double(c.child_wmax);
        if (children) *children = (int64_t)(c.n_par << h->n);
    })
}

int rb_round_hs(rb_handle* h, int32_t hs_on, int32_t hs_contract, int64_t* n_out, double* width, int64_t* hs_calls) {
    if (!h) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        HsParams prm{};
        prm.round_no = h->shard_round;
        prm.hs_mode = hs_on ? 1 : 2;
        prm.contract_output = hs_contract ? 1 : 0;
        for (;;) {
            launch_hs_phase(h, prm, false);  // exact dedup runs after the owner exchange (rb_shard_dedup)
            sync_counters(h);
            if (h->h_ctr->n_next > (unsigned long long)h->F[h->cur ^ 1].f.cap) {
                // redo the round with a larger frontier (the input rows are preserved)
                fronts_reserve(h, (int64_t)(h->h_ctr->n_next + h->h_ctr->n_next / 4));
                launch_filter_phase(h, h->shard_target);
                continue;
            }
            break;
        }
        RoundOut ro{};
        fill_round_out(h, ro);
        commit_round(h, ro);
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
        codegen_poll(h);
        PoolScope ps(h);
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
        dfree(dlo);
        dfree(dhi);
        dfree(dc);
        dfree(du);
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
        codegen_poll(h);
        PoolScope ps(h);
        h->n_cur = keep;
        fronts_reserve(h, keep + count);
        load_rows(h, h->F[h->cur], keep, lo, hi, cert, unsplit, count);
        h->n_cur = keep + count;
    })
}

int64_t rb_shard_size(rb_handle* h) { return h ? h->n_cur : -1; }

// kernels launched by this handle since its last rb_solve (the shard protocol's calls
// accumulate; rb_solve reports its own count in rb_result_info.kernel_launches)
int64_t rb_kernel_launches(rb_handle* h) { return h ? h->launches : -1; }

int rb_shard_partition(rb_handle* h, int32_t world, int64_t* counts) {
    if (!h || world < 1 || !counts) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        fronts_reserve(h, std::max<int64_t>(h->n_cur, 1));
        dispatch_n<PartitionK>(h->n, h, (int)world, counts);
    })
}

int rb_shard_dedup(rb_handle* h, int64_t* dups, double* width) {
    if (!h) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        fronts_reserve(h, std::max<int64_t>(h->n_cur, 1));
        // the dedup kernels read the row count from the counters (n_next) and skip
        // on overflow (n_surv <= S.cap is trivially true here)
        Counters c{};
        c.n_next = (unsigned long long)h->n_cur;
        ck(cudaMemcpyAsync(h->d_ctr, &c, sizeof(Counters), cudaMemcpyHostToDevice, h->st), "ctr h2d");
        if (h->n_cur >= 2) dispatch_n<DedupK>(h->n, h, h->F[h->cur].f, h->F[h->cur ^ 1].f);
        sync_counters(h);
        const int64_t d = (int64_t)h->h_ctr->dups;
        if (d > 0) h->cur ^= 1;  // compacted into the other buffer
        h->n_cur -= d;
        ck(cudaMemsetAsync(&h->d_ctr->wmax, 0, sizeof(unsigned long long), h->st), "memset");
        if (h->n_cur > 0) dispatch_n<WidthK>(h->n, h);
        sync_counters(h);
        if (dups) *dups = d;
        if (width) *width = h->n_cur ? bits_to_double(h->h_ctr->wmax) : 0.0;
    })
}

// row-major device buffers (e.g. torch CUDA tensors) <-> the shard; synchronous on the engine stream
int rb_shard_export_device(rb_handle* h, int64_t start, int64_t count, double* dlo, double* dhi, uint8_t* dcert,
                           uint8_t* duns) {
    if (!h || start < 0 || count < 0) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    if (start + count > h->n_cur) {
        h->err = "export range beyond the shard";
        return RB_ERR_ARG;
    }
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        if (count == 0) return RB_OK;
        Front f = h->F[h->cur].f, sub = f;
        sub.lo = f.lo + start;
        sub.hi = f.hi + start;
        sub.cert = f.cert + start;
        sub.unsplit = f.unsplit + start;
        h->launches++;
        k_gather_rows<<<grid_for(count, 256, h->sms * 8), 256, 0, h->st>>>(sub, h->n, count, nullptr, dlo, dhi,
                                                                            dcert, duns);
        ck(cudaGetLastError(), "export gather");
        ck(cudaStreamSynchronize(h->st), "export sync");
    })
}

int rb_shard_import_device(rb_handle* h, int64_t keep, const double* dlo, const double* dhi, const uint8_t* dcert,
                           const uint8_t* duns, int64_t count) {
    if (!h || keep < 0 || count < 0) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    if (keep > h->n_cur) {
        h->err = "keep beyond the shard";
        return RB_ERR_ARG;
    }
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        h->n_cur = keep;
        fronts_reserve(h, keep + count);
        if (count > 0) {
            h->launches++;
            k_rows_to_soa<<<grid_for(count, 256, h->sms * 8), 256, 0, h->st>>>(dlo, dhi, dcert, duns, h->n, count,
                                                                                h->F[h->cur].f, keep);
            ck(cudaGetLastError(), "import");
            ck(cudaStreamSynchronize(h->st), "import sync");
        }
        h->n_cur = keep + count;
    })
}

int rb_shard_route_count(rb_handle* h, int32_t world, int64_t* thin_counts, int64_t* nonthin) {
    if (!h || world < 1 || !thin_counts || !nonthin) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        fronts_reserve(h, std::max<int64_t>(h->n_cur, 1));
        dispatch_n<RouteCountK>(h->n, h, (int)world, thin_counts, nonthin);
    })
}

int rb_shard_route(rb_handle* h, int32_t world, int32_t rank, const int64_t* move, int64_t* send_counts) {
    if (!h || world < 1 || rank < 0 || rank >= world || !move || !send_counts) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->cap_route < h->n_cur || !h->d_route) {
        h->err = "rb_shard_route before rb_shard_route_count";
        return RB_ERR_STATE;
    }
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        fronts_reserve(h, std::max<int64_t>(h->n_cur, 1));
        dispatch_n<RouteK>(h->n, h, (int)world, (int)rank, move, send_counts);
    })
}

int rb_shard_finalize(rb_handle* h, int64_t* nboxes) {
    if (!h) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    RB_GUARD(h, {
        ck(cudaSetDevice(h->dev), "cudaSetDevice");
        codegen_poll(h);
        PoolScope ps(h);
        h->stats.clear();
        h->r_ready = false;
        finalize_sorted(h);
        h->have_result = true;
        if (nboxes) *nboxes = h->r_n;
    })
}

int rb_set_option(rb_handle* h, const char* key, int64_t value) {
    if (!h || !key) return RB_ERR_ARG;
    std::lock_guard<std::mutex> lk(h->mu);
    const std::string k(key);
    if (k == "filter_tab") {
        h->use_ftab = value != 0;
        return RB_OK;
    }
    if (k == "jconst") {  // 1 (default): constant J entries bypass the HS scratch (k_hs_lin_tps)
        h->jconst = value != 0;
        graph_release(h);
        return RB_OK;
    }
    if (k == "filter_wt") {  // warp-tabulated filter where it applies (5 <= n <= 16, tables fit); -1: auto
        h->use_fwt = value < 0 ? h->fwt_auto : value != 0;
        return RB_OK;
    }
    if (k == "hs_fused") {  // 0: eval/lin/sweep only, 1: by batch size, 2: fused only
        h->hs_fused = value != 0 && h->fused_smem <= (size_t)h->smem_optin;
        h->fused_rows = value == 2 ? INT64_MAX : (int64_t)h->sms * 80;
        return RB_OK;
    }
    if (k == "device_timing") {  // 0: return on the graph's completion flag, device_ms = -1
        h->device_timing = value != 0;
        return RB_OK;
    }
    if (k == "pdl") {
        h->pdl = value != 0;
        return RB_OK;
    }
    if (k == "small_rounds") {
        h->use_mk = value != 0;
        return RB_OK;
    }
    if (k == "mk_bps") {
        h->mk_bps = (int)std::max<int64_t>(1, value);
        return RB_OK;
    }
    if (k == "mk_cap") {
        h->mk_cap = value;
        return RB_OK;
    }
    if (k == "graph_fused_only") {  // round graph: k_hs_fused for every survivor count
        h->graph_fused_only = value != 0;
        return RB_OK;
    }
    if (k == "codegen") {  // 1: system-specialised kernels when compiled, 0: table kernels
        h->use_gen = value != 0;
        return RB_OK;
    }
    if (k == "codegen_wait") {  // block until a background compile has finished and take it over
        RB_GUARD(h, {
            ck(cudaSetDevice(h->dev), "cudaSetDevice");
            codegen_poll(h, true);
        })
    }
    if (k == "tail_blocks_x4") {  // round-tail grid = SMs * value / 4 blocks
        h->tail_blocks_per_sm = std::max<int64_t>(1, value) / 4.0;
        return RB_OK;
    }
    if (k == "graph_prologue") {  // ping-pong round graph: the first U rounds before the WHILE node
        h->graph_prologue = value != 0;
        return RB_OK;
    }
    if (k == "pingpong") {  // round graph: ping-pong frontiers, round end in the HS kernel
        h->pingpong = value != 0;
        return RB_OK;
    }
    if (k == "graph_cf") {  // round graph: classify + filter in one kernel
        h->graph_cf = value != 0;
        return RB_OK;
    }
    if (k == "append_dedup") {  // round graph: exact dedup at append time
        h->append_dedup = value != 0;
        return RB_OK;
    }
    if (k == "graph_unroll") {  // rounds per WHILE iteration of the round graph
        h->graph_unroll = (int)std::min<int64_t>(16, std::max<int64_t>(1, value));
        return RB_OK;
    }
    if (k == "hs_cond") {
        h->hs_cond = value != 0;
        return RB_OK;
    }
    if (k == "graph") {
        h->use_graph = value != 0;
        return RB_OK;
    }
    if (k == "stream_parents") {  // > 0: every host-driven round streams its parents in chunks of this size
        h->stream_parents = std::max<int64_t>(0, value);
        return RB_OK;
    }
    if (k == "mem_budget_mb") {  // engine memory budget (tests of the streamed rounds at small budgets)
        h->mem_budget = value > 0 ? (size_t)value << 20 : h->mem_budget_default;  // 0: the default
        return RB_OK;
    }
    if (k == "lin_tpb") {  // three-kernel HS: thread-per-box Gauss-Jordan in shared memory (2, n <= 12) or
                           // registers (1, n <= 8); 0 = G lanes per box (k_hs_lin)
        h->lin_tpb = (int)std::min<int64_t>(3, std::max<int64_t>(0, value));  // 3: two threads per box
        return RB_OK;
    }
    if (k == "hs_tile") {  // large HS batches: 1 = k_hs_tile (n <= 8), 0 = eval/lin/sweep
        h->hs_tile = value != 0 && h->n <= 8 && h->tile_tb > 0;
        return RB_OK;
    }
    if (k == "force_exact") {  // Exact policy everywhere (parity tests of interval.cuh's Exact)
        h->force_exact = value != 0;
        // poly_guard_ok fails for any coefficient exponent below -965 (kernels.cuh)
        h->meta.f_ecmin = h->force_exact ? -100000 : h->guard_f_ecmin;
        h->meta.j_ecmin = h->force_exact ? -100000 : h->guard_j_ecmin;
        return RB_OK;
    }
    h->err = "unknown option " + k;
    return RB_ERR_ARG;
}

// Independent chains of directed DMUL/DADD per thread; values stay in [1, 2).
__global__ void k_fp64_peak(double* sink, int iters) {
    double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 + 1e-10, a2 = a0 + 2e-10, a3 = a0 + 3e-10;
    double a4 = a0 + 4e-10, a5 = a0 + 5e-10, a6 = a0 + 6e-10, a7 = a0 + 7e-10;
    const double m = 1.0000000001, d = -1e-12;
    for (int i = 0; i < iters; i++) {
        a0 = __dmul_rd(a0, m); a1 = __dmul_ru(a1, m); a2 = __dadd_rd(a2, d); a3 = __dadd_ru(a3, d);
        a4 = __dmul_rd(a4, m); a5 = __dmul_ru(a5, m); a6 = __dadd_rd(a6, d); a7 = __dadd_ru(a7, d);
    }
    const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == 12345.0) sink[0] = r;  // never true; keeps the chains alive
}

int rb_fp64_peak(int device, double* ops_per_second) {
    if (!ops_per_second) return RB_ERR_ARG;
    try {
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "props");
        double* sink = nullptr;
        ck(cudaMalloc(&sink, 8), "malloc");
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "ev");
        ck(cudaEventCreate(&b), "ev");
        const int threads = 256, blocks = prop.multiProcessorCount * 8, iters = 1 << 14;
        k_fp64_peak<<<blocks, threads>>>(sink, 256);  // warm-up
        double best = 0.0;
        for (int rep = 0; rep < 5; rep++) {
            ck(cudaEventRecord(a), "ev");
            k_fp64_peak<<<blocks, threads>>>(sink, iters);
            ck(cudaEventRecord(b), "ev");
            ck(cudaEventSynchronize(b), "ev sync");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            const double ops = 8.0 * iters * (double)threads * blocks;
            best = std::max(best, ops / (ms * 1e-3));
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(sink);
        *ops_per_second = best;
        return RB_OK;
    } catch (const CudaError& ce) {
        g_create_error = std::string(ce.what) + ": " + cudaGetErrorString(ce.e);
        cudaGetLastError();
        return RB_ERR_CUDA;
    }
}

}  // extern "C"
