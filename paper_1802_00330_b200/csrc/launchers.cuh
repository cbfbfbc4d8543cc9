// launchers.cuh -- definitions of the per-dimension launchers declared in
// engine.cuh.  Included only by kinst.cu, which instantiates them explicitly.
#pragma once
#include "engine.cuh"

template <int N>
void SetupK<N>::run(rb_handle* h) {
    const int T = h->hs_threads;
    h->filter_smem = filter_off_xs(h->meta) + (size_t)2 * N * h->filter_threads * sizeof(double);
    h->eval_smem = stab_bytes(h->meta, false) + (size_t)3 * N * T * sizeof(double);
    h->lin_smem = (size_t)(T / 32) * LinLayout<N>::BPW * LinLayout<N>::doubles * sizeof(double);
    h->sweep_smem = (size_t)2 * N * T * sizeof(double);
    if (h->meta.ftab) {
        h->ftab_smem = ftab_smem_bytes<N>(h->meta);
        if (h->ftab_smem > 160 * 1024) h->meta.ftab = 0;  // tables too large: direct evaluation
    }
    h->fwt_bps = 0;
    if (N >= 5 && N <= 16 && h->meta.ftab) {
        h->fwt_smem = fwt_smem_bytes<N>(h->meta, 256);
        if ((int)h->fwt_smem <= h->smem_optin) {
            const void* kf = h->meta.fwt_direct ? (const void*)k_filter_wt<N, TabEval, true>
                                                : (const void*)k_filter_wt<N, TabEval, false>;
            set_max_dyn_smem(kf, h->smem_optin);
            int nbw = 0;
            ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbw, kf, 256, h->fwt_smem), "occ fwt");
            h->fwt_bps = nbw;
        }
    }
    // on by default when at most half of the equations have tables larger than a quarter of
    // a work unit's children (those are evaluated per child): katsura6 filter 6.1 -> 3.3 ms,
    // eco8 22.6 -> 10.0 ms, brown8 (one degree-8 product evaluated per child) 4.2 -> 3.8 ms
    h->fwt_auto = h->fwt_bps > 0 && 2 * __builtin_popcount((unsigned)h->meta.fwt_direct) <= N;
    h->use_fwt = h->fwt_auto;
    // the attribute is per kernel (shared by every handle of this n): set it to the opt-in maximum
    const size_t mx = std::max({h->filter_smem, h->eval_smem, h->lin_smem, h->sweep_smem});
    h->fused_smem = fused_off_tiles(h->meta) +
                    (size_t)(T / 32) * FusedLayout<N>::BPW * FusedLayout<N>::doubles * sizeof(double);
    if ((int)mx > h->smem_optin) throw ArgError{RB_ERR_LIMIT, "system tables exceed the shared-memory budget"};
    set_max_dyn_smem(k_filter<N>, h->smem_optin);
    set_max_dyn_smem(k_classify_filter<N>, h->smem_optin);
    set_max_dyn_smem(k_filter_tab<N>, h->smem_optin);
    set_max_dyn_smem(k_hs_eval<N>, h->smem_optin);
    set_max_dyn_smem(k_hs_lin<N>, h->smem_optin);
    set_max_dyn_smem(k_hs_sweep<N>, h->smem_optin);
    set_max_dyn_smem(k_hs_fused<N>, h->smem_optin);
    set_max_dyn_smem(k_hs_tile<N>, h->smem_optin);
    if constexpr (N <= 8) {  // thread-per-box Gauss-Jordan: registers (k_hs_lin_tpb) / shared (k_hs_lin_tps)
        int nb = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs_lin_tpb<N>, 128, 0), "occ lin tpb");
        h->lin_tpb_threads = 128;
        h->lin_tpb_smem = 0;
        h->lin_tpb_bps = std::max(1, nb);
    }
    if constexpr (N <= 12) {  // thread-per-box Gauss-Jordan with the tableau in shared memory
        int nb = 0;
        set_max_dyn_smem(k_hs_lin_tps<N>, h->smem_optin);
        h->lin_tps_smem = (size_t)N * N * TpsShape<N>::T * sizeof(double);
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs_lin_tps<N>, TpsShape<N>::T, h->lin_tps_smem),
           "occ lin tps");
        h->lin_tps_bps = std::max(1, nb);
        set_max_dyn_smem(k_hs_lin_tp2<N>, h->smem_optin);
        h->lin_tp2_smem = (size_t)N * N * 64 * sizeof(double);
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs_lin_tp2<N>, 128, h->lin_tp2_smem), "occ lin tp2");
        h->lin_tp2_bps = std::max(1, nb);
    }
    choose_tile(h, k_hs_tile<N>, N, stab_bytes(h->meta, false), h->tile_tb, h->tile_smem, h->tile_bps);
    if (N > 8 || h->tile_tb == 0) h->hs_tile = false;  // n > 8: one box per warp, the three kernels win
    if ((int)h->fused_smem > h->smem_optin) h->hs_fused = false;
    int nb = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_filter<N>, h->filter_threads, h->filter_smem), "occ");
    h->filter_blocks_per_sm = std::max(1, nb);
    if (h->meta.ftab) {
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_filter_tab<N>, 256, h->ftab_smem), "occ");
        h->ftab_blocks_per_sm = std::max(1, nb);
    }
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs_eval<N>, T, h->eval_smem), "occ");
    h->eval_blocks_per_sm = std::max(1, nb);
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs_lin<N>, T, h->lin_smem), "occ");
    h->lin_blocks_per_sm = std::max(1, nb);
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs_sweep<N>, T, h->sweep_smem), "occ");
    h->sweep_blocks_per_sm = std::max(1, nb);
    if (h->hs_fused) {
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hs_fused<N>, T, h->fused_smem), "occ");
        h->fused_blocks_per_sm = std::max(1, nb);
    }
    gen_configure(h);

}

template <int N>
void ClassifyK<N>::run(rb_handle* h, double target, const DevState* st, int64_t bound, DedupCtx dd) {
    Front cur = h->F[h->cur].f, next = h->F[h->cur ^ 1].f;
    const int blocks = grid_for(bound >= 0 ? bound : h->n_cur, 256, h->sms * 8);
    h->launches++;
    klaunch(h, k_classify<N>, blocks, 256, 0, h->meta, cur, h->n_cur, next, h->parents, h->d_ctr, target, st, dd);
    ck(cudaGetLastError(), "classify launch");
}

template <int N>
void ClassifyFilterK<N>::run(rb_handle* h, DedupCtx dd, int64_t bound) {
    Front cur = h->F[h->cur].f, next = h->F[h->cur ^ 1].f;
    h->launches++;
    unsigned long long* prof = h->trace ? h->d_trace + kTraceCfOff : (unsigned long long*)nullptr;
    if (gen_on(h)) {
        const int blocks = grid_for(bound, 256, h->sms * h->gen_cf_bps);
        klaunch_k(h, h->gen.cf, blocks, 256, h->filter_smem, h->meta, (const uint8_t*)h->d_tab, cur, next, h->d_ctr,
                  h->S, (const DevState*)h->d_state, (const int*)h->d_order, dd, prof);
    } else {
        const int blocks = grid_for(bound, 256, h->sms * h->filter_blocks_per_sm);
        klaunch(h, k_classify_filter<N>, blocks, 256, h->filter_smem, h->meta, h->d_tab, cur, next, h->d_ctr, h->S,
                (const DevState*)h->d_state, (const int*)h->d_order, dd, prof);
    }
    ck(cudaGetLastError(), "classify_filter launch");
}

template <int N>
void AllParentsK<N>::run(rb_handle* h) {
    const int blocks = grid_for(h->n_cur, 256, h->sms * 8);
    h->launches++;
    klaunch(h, k_all_parents<N>, blocks, 256, 0, h->meta, h->F[h->cur].f, h->n_cur, h->parents, h->d_ctr);
    ck(cudaGetLastError(), "parents launch");
}

template <int N>
void FilterK<N>::run(rb_handle* h, int64_t max_parents, int64_t* tags, int64_t p0, int64_t pcount) {
    // parents [p0, p0 + pcount) of the round's list (a streamed chunk), or all of them (pcount < 0)
    const uint32_t* par = h->parents + p0;
    // warp per parent; small rounds keep the direct filter (a table build is a serial
    // latency chain per warp: Broyden-tri-6 round 3, 2.4k boxes, 15.5 vs 9.6 us)
    if (h->use_fwt && h->fwt_bps > 0 && max_parents >= (int64_t)h->sms * 8) {
        const bool g = gen_on(h) && h->gen_fwt_bps > 0;
        const int64_t cap = (int64_t)h->sms * (g ? h->gen_fwt_bps : h->fwt_bps);
        const int64_t units = max_parents << (N > 10 ? N - 10 : 0);  // (parent, 1024-child chunk) above n = 10
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((units + 7) / 8, cap));
        h->launches++;
        if (g)
            klaunch_k(h, h->gen.filter_wt, blocks, 256, h->fwt_smem, h->meta, (const uint8_t*)h->d_tab, h->F[h->cur].f,
                      par, h->d_ctr, h->S, tags, (const int*)h->d_order, pcount);
        else if (h->meta.fwt_direct)
            klaunch(h, k_filter_wt<N, TabEval, true>, blocks, 256, h->fwt_smem, h->meta, h->d_tab, h->F[h->cur].f,
                    par, h->d_ctr, h->S, tags, h->d_order, pcount);
        else
            klaunch(h, k_filter_wt<N, TabEval, false>, blocks, 256, h->fwt_smem, h->meta, h->d_tab, h->F[h->cur].f,
                    par, h->d_ctr, h->S, tags, h->d_order, pcount);
        ck(cudaGetLastError(), "filter_wt launch");
        return;
    }
    if (h->meta.ftab && h->use_ftab) {
        using Sh = FtabShape<N>;
        const int64_t units = N >= 8 ? (max_parents << Sh::CHLOG) : ((max_parents + Sh::PPB - 1) >> Sh::LOGPPB);
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)h->sms * h->ftab_blocks_per_sm));
        h->launches++;
        if (gen_on(h))  // specialised sums of table entries (codegen.cpp fts*)
            klaunch_k(h, h->gen.filter_tab, (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)h->sms * h->gen_ftab_bps)),
                      256, h->ftab_smem, h->meta, (const uint8_t*)h->d_tab, h->F[h->cur].f, par, h->d_ctr, h->S, tags,
                      (const int*)h->d_order, pcount);
        else
            klaunch(h, k_filter_tab<N>, blocks, 256, h->ftab_smem, h->meta, h->d_tab, h->F[h->cur].f, par,
                    h->d_ctr, h->S, tags, h->d_order, pcount);
        ck(cudaGetLastError(), "filter_tab launch");
        return;
    }
    const int64_t work = max_parents << N;
    h->launches++;
    if (gen_on(h)) {
        const int blocks = grid_for(work, h->filter_threads, h->sms * h->gen_filter_bps);
        klaunch_k(h, h->gen.filter, blocks, h->filter_threads, h->filter_smem, h->meta, (const uint8_t*)h->d_tab,
                  h->F[h->cur].f, par, h->d_ctr, h->S, tags, (const int*)h->d_order, pcount);
        ck(cudaGetLastError(), "filter launch");
        return;
    }
    const int blocks = grid_for(work, h->filter_threads, h->sms * h->filter_blocks_per_sm);
    klaunch(h, k_filter<N>, blocks, h->filter_threads, h->filter_smem, h->meta, h->d_tab, h->F[h->cur].f,
                                                                     par, h->d_ctr, h->S, tags, h->d_order, pcount);
    ck(cudaGetLastError(), "filter launch");
}

template <int N>
void HsK<N>::run(rb_handle* h, int64_t b0, int64_t n_in, HsParams prm, int64_t* tags, int64_t batch_bound) {
    prm.force_exact = h->force_exact ? 1 : 0;
    const int T = h->hs_threads;
    const int64_t B = h->W.B;
    Front out = h->F[h->cur ^ 1].f;
    h->launches += 3;
    // the Gauss-Jordan variant first: with k_hs_lin_tps the constant J entries bypass the scratch
    int lin = 0;  // 0: G lanes per box (k_hs_lin), 1: registers (k_hs_lin_tpb), 2: shared (k_hs_lin_tps)
    if constexpr (N <= 8)
        if (h->lin_tpb == 1 && h->lin_tpb_threads > 0) lin = 1;
    if constexpr (N <= 12)
        if (lin == 0 && (h->lin_tpb == 2 || h->lin_tpb == 3)) lin = (h->lin_tpb == 2 && N > 8) ? 3 : h->lin_tpb;
    prm.jc = nullptr;
    if ((lin == 2 || lin == 3) && h->jconst && (h->jmask[0] | h->jmask[1] | h->jmask[2] | h->jmask[3])) {
        prm.jc = h->d_jc;
        for (int w = 0; w < 4; w++) prm.jm[w] = h->jmask[w];
    }
    // split each box's n^2 + n polynomials over R threads when the batch is small
    const int64_t bound = std::max<int64_t>(1, std::min<int64_t>(B, batch_bound));
    const int64_t target = (int64_t)h->sms * 1024;
    const int R = (int)std::max<int64_t>(1, std::min<int64_t>(N * N + N, (target + bound - 1) / bound));
    if (gen_on(h))  // specialised J(X) / F(x): one thread evaluates a whole box
        klaunch_k(h, h->gen.hs_eval, grid_for(bound, T, h->sms * h->gen_hse_bps), T, h->eval_smem, h->meta,
                  (const uint8_t*)h->d_tab, h->S, n_in, b0, prm, h->W, out, h->d_ctr, tags, 1);
    else
        klaunch(h, k_hs_eval<N>, grid_for(bound * R, T, h->sms * h->eval_blocks_per_sm), T, h->eval_smem,
            h->meta, h->d_tab, h->S, n_in, b0, prm, h->W, out, h->d_ctr, tags, R);
    if constexpr (N <= 8) {
        if (lin == 1) {
            const int tl = h->lin_tpb_threads;
            klaunch(h, k_hs_lin_tpb<N>, grid_for(bound, tl, h->sms * h->lin_tpb_bps), tl, h->lin_tpb_smem, h->S, n_in,
                    b0, prm, h->W, h->d_ctr);
        }
    }
    if constexpr (N <= 12) {
        if (lin == 2) {
            constexpr int TT = TpsShape<N>::T;
            klaunch(h, k_hs_lin_tps<N>, grid_for(bound, TT, h->sms * h->lin_tps_bps), TT, h->lin_tps_smem, h->S,
                    n_in, b0, prm, h->W, h->d_ctr);
        } else if (lin == 3) {  // two threads per box: 64 boxes per block
            klaunch(h, k_hs_lin_tp2<N>, grid_for(bound, 64, h->sms * h->lin_tp2_bps), 128, h->lin_tp2_smem, h->S,
                    n_in, b0, prm, h->W, h->d_ctr);
        }
    }
    if (lin == 0)
        klaunch(h, k_hs_lin<N>, grid_for(B, (T / 32) * LinLayout<N>::BPW, h->sms * h->lin_blocks_per_sm), T,
                h->lin_smem, h->S, n_in, b0, prm, h->W, h->d_ctr);
    klaunch(h, k_hs_sweep<N>, grid_for(B, T, h->sms * h->sweep_blocks_per_sm), T, h->sweep_smem,
        h->meta, h->S, n_in, b0, prm, h->W, out, h->d_ctr, tags);
    ck(cudaGetLastError(), "hs launch");
}

template <int N>
void HsTileK<N>::run(rb_handle* h, int64_t n_in, HsParams prm, int64_t* tags, int64_t bound) {
    prm.force_exact = h->force_exact ? 1 : 0;
    h->launches++;
    Front out = h->F[h->cur ^ 1].f;
    const int64_t rows = std::max<int64_t>(1, bound);
    if (gen_on(h) && h->gen_tile_tb > 0) {
        const int tb = h->gen_tile_tb;
        klaunch_k(h, h->gen.hs_tile, grid_for(rows, tb, h->sms * h->gen_tile_bps), tb, h->gen_tile_smem, h->meta,
                  (const uint8_t*)h->d_tab, h->S, n_in, prm, out, h->d_ctr, tags);
    } else {
        const int tb = h->tile_tb;
        klaunch(h, k_hs_tile<N>, grid_for(rows, tb, h->sms * h->tile_bps), tb, h->tile_smem, h->meta, h->d_tab,
                h->S, n_in, prm, out, h->d_ctr, tags);
    }
    ck(cudaGetLastError(), "hs tile launch");
}

template <int N>
void HsFusedK<N>::run(rb_handle* h, int64_t n_in, HsParams prm, int64_t* tags, int64_t bound) {
    prm.force_exact = h->force_exact ? 1 : 0;
    const int T = h->hs_threads;
    h->launches++;
    const int64_t lanes = std::max<int64_t>(1, bound) * FusedLayout<N>::G;
    if (h->trace) prm.prof = h->d_trace + (size_t)kTraceRounds * kTracePhases;
    if (gen_on(h) && !prm.has_cond)  // the specialised build never sets graph conditionals
        klaunch_k(h, h->gen.hs_fused, grid_for(lanes, T, h->sms * h->gen_hsf_bps), T, h->fused_smem, h->meta,
                  (const uint8_t*)h->d_tab, h->S, n_in, prm, h->F[h->cur ^ 1].f, h->d_ctr, tags);
    else
        klaunch(h, k_hs_fused<N>, grid_for(lanes, T, h->sms * h->fused_blocks_per_sm), T, h->fused_smem,
            h->meta, h->d_tab, h->S, n_in, prm, h->F[h->cur ^ 1].f, h->d_ctr, tags);
    ck(cudaGetLastError(), "hs fused launch");
}

template <int N>
void KrawczykK<N>::run(rb_handle* h, int64_t b0, int64_t b_end, Front out, uint8_t* ok) {
    const int T = h->hs_threads;
    const int64_t B = h->W.B;
    HsParams prm{};
    prm.hs_mode = 1;
    h->launches += 3;
    const int64_t bound = b_end - b0;
    const int64_t target = (int64_t)h->sms * 1024;
    const int R = (int)std::max<int64_t>(1, std::min<int64_t>(N * N + N, (target + bound - 1) / bound));
    klaunch(h, k_hs_eval<N>, grid_for(bound * R, T, h->sms * h->eval_blocks_per_sm), T, h->eval_smem,
        h->meta, h->d_tab, h->S, b_end, b0, prm, h->W, out, h->d_ctr, nullptr, R);
    klaunch(h, k_hs_lin<N>, grid_for(std::min(B, bound), (T / 32) * LinLayout<N>::BPW, h->sms * h->lin_blocks_per_sm), T, h->lin_smem, h->S, b_end, b0, prm, h->W, h->d_ctr);
    klaunch(h, k_krawczyk<N>, grid_for(bound, 128, h->sms * 16), 128, 0, h->S, b_end, b0, h->W, out, ok);
    ck(cudaGetLastError(), "krawczyk launch");
}

template <int N>
void SmallRoundsK<N>::run(rb_handle* h, const HsParams& prm, bool dedup, int64_t scap, cudaGraphConditionalHandle hw) {
    if (h->mk_blocks_per_sm == 0) {  // set up on first use: 256 threads, shared memory of its largest phase
        h->mk_smem = std::max<size_t>(filter_off_xs(h->meta) + (size_t)2 * N * 256 * sizeof(double),
                                      fused_off_tiles(h->meta) + (size_t)(256 / 32) * FusedLayout<N>::BPW *
                                                                     FusedLayout<N>::doubles * sizeof(double));
        h->mk_blocks_per_sm = -1;
        if ((int)h->mk_smem <= h->smem_optin) {
            set_max_dyn_smem(k_small_rounds<N>, h->smem_optin);
            int nb = 0;
            ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_small_rounds<N>, 256, h->mk_smem), "occ");
            if (nb > 0) h->mk_blocks_per_sm = nb;
        }
    }
    if (h->mk_blocks_per_sm < 1) return;  // not resident-capable: the WHILE loop runs every round
    SmallArgs a{};
    a.dedup = dedup ? 1 : 0;
    a.trace = h->trace ? h->d_trace : nullptr;
    a.meta = h->meta;
    a.gtab = h->d_tab;
    a.f0 = h->F[0].f;
    a.f1 = h->F[1].f;
    a.S = h->S;
    a.parents = h->parents;
    a.ctr = h->d_ctr;
    a.st = h->d_state;
    a.rstats = h->d_rstats;
    a.order = h->d_order;
    a.table = h->d_table;
    a.table_mask = (unsigned long long)(h->table_slots - 1);
    a.slot_of = h->d_slot;
    a.dead = h->d_dead;
    a.prm = prm;
    a.bar = h->d_bar;
    a.mk_cap = std::min<int64_t>(h->mk_cap, scap);
    a.graph_cap = scap;
    a.h_while = hw;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(h->sms * std::min(h->mk_blocks_per_sm, h->mk_bps)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = h->mk_smem;
    cfg.stream = h->st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    h->launches++;
    ck(cudaLaunchKernelEx(&cfg, k_small_rounds<N>, a), "small rounds launch");
}

template <int N>
void DedupInsertK<N>::run(rb_handle* h, Front next) {
    const int blocks = grid_for(next.cap, 256, h->sms * 8);
    h->launches++;
    klaunch(h, k_dedup_insert<N>, blocks, 256, 0, next, h->d_table, (unsigned long long)(h->table_slots - 1),
            h->d_slot, h->d_dead, h->d_ctr, h->S.cap);
}

template <int N>
void TailK<N>::run(rb_handle* h, bool dedup, int64_t bound, int64_t scap, cudaGraphConditionalHandle hw) {
    const int blocks = grid_for(bound, 256, std::max(1, (int)(h->sms * h->tail_blocks_per_sm)));
    h->launches++;
    klaunch(h, k_round_tail<N>, blocks, 256, 0, h->F[1].f, h->F[0].f, h->d_table, (const unsigned*)h->d_slot,
            (const uint8_t*)h->d_dead, dedup ? 1 : 0, h->d_state, h->d_ctr, h->d_rstats, scap, hw, h->d_order,
            h->meta);
}

template <int N>
void SettleK<N>::run(rb_handle* h, int64_t bound) {
    klaunch(h, k_settle<N>, grid_for(bound, 256, h->sms * 8), 256, 0, h->F[1].f, h->F[0].f, h->d_ctr);
    ck(cudaGetLastError(), "settle launch");
}

template <int N>
void DedupK<N>::run(rb_handle* h, Front next, Front other) {
    // persistent grids: the row count is read on the device
    const int blocks = grid_for(next.cap, 256, h->sms * 8);
    h->launches += 2;
    klaunch(h, k_dedup_insert<N>, blocks, 256, 0, next, h->d_table, (unsigned long long)(h->table_slots - 1),
                                                 h->d_slot, h->d_dead, h->d_ctr, h->S.cap);
    klaunch(h, k_dedup_finish<N>, blocks, 256, 0, next, other, h->d_table, h->d_slot, h->d_dead, h->d_ctr,
                                                 h->S.cap);
    ck(cudaGetLastError(), "dedup launch");
}

template <int N>
void PartitionK<N>::run(rb_handle* h, int world, int64_t* counts) {
    const int64_t n = h->n_cur;
    unsigned* owner = nullptr;
    unsigned long long* cnt = nullptr;
    dalloc(&owner, (size_t)std::max<int64_t>(n, 1));
    dalloc(&cnt, (size_t)2 * world);
    ck(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 2 * world, h->st), "memset");
    const int blocks = grid_for(n, 256, h->sms * 8);
    h->launches += 2;
    if (n > 0) k_owner_count<N><<<blocks, 256, 0, h->st>>>(h->F[h->cur].f, n, world, owner, cnt);
    std::vector<unsigned long long> hc(2 * world);
    ck(cudaMemcpyAsync(hc.data(), cnt, sizeof(unsigned long long) * world, cudaMemcpyDeviceToHost, h->st), "d2h");
    ck(cudaStreamSynchronize(h->st), "sync");
    unsigned long long off = 0;
    for (int r = 0; r < world; r++) {
        counts[r] = (int64_t)hc[r];
        hc[world + r] = off;
        off += hc[r];
    }
    ck(cudaMemcpyAsync(cnt + world, hc.data() + world, sizeof(unsigned long long) * world, cudaMemcpyHostToDevice,
                       h->st), "h2d");
    if (n > 0) k_owner_scatter<N><<<blocks, 256, 0, h->st>>>(h->F[h->cur].f, n, owner, cnt + world,
                                                            h->F[h->cur ^ 1].f);
    ck(cudaGetLastError(), "partition");
    h->cur ^= 1;
    dfree(owner);
    dfree(cnt);
    ck(cudaStreamSynchronize(h->st), "sync");
}

template <int N>
void RouteCountK<N>::run(rb_handle* h, int world, int64_t* thin_counts, int64_t* nonthin) {
    const int64_t n = h->n_cur;
    if (h->cap_route < std::max<int64_t>(n, 1) || !h->d_route) {
        dalloc(&h->d_route, (size_t)std::max<int64_t>(n, 1));
        h->cap_route = std::max<int64_t>(n, 1);
    }
    unsigned long long* cnt = nullptr;
    dalloc(&cnt, (size_t)world + 1);
    ck(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (world + 1), h->st), "memset");
    h->launches++;
    if (n > 0)
        k_route_count<N><<<grid_for(n, 256, h->sms * 8), 256, 0, h->st>>>(h->F[h->cur].f, n, world, h->d_route, cnt);
    ck(cudaGetLastError(), "route count");
    std::vector<unsigned long long> hc(world + 1);
    ck(cudaMemcpyAsync(hc.data(), cnt, sizeof(unsigned long long) * (world + 1), cudaMemcpyDeviceToHost, h->st),
       "d2h");
    ck(cudaStreamSynchronize(h->st), "sync");
    for (int r = 0; r < world; r++) thin_counts[r] = (int64_t)hc[r];
    *nonthin = (int64_t)hc[world];
    dfree(cnt);
}

template <int N>
void RouteK<N>::run(rb_handle* h, int world, int rank, const int64_t* move, int64_t* send_counts) {
    const int64_t n = h->n_cur;
    // device scratch: move offsets [world + 1], taken [1], counts [world], cursors [world]
    unsigned long long* buf = nullptr;
    dalloc(&buf, (size_t)3 * world + 2);
    std::vector<unsigned long long> hb(3 * world + 2, 0);
    unsigned long long off = 0;
    for (int d = 0; d < world; d++) {
        hb[d] = off;
        off += d == rank ? 0 : (unsigned long long)std::max<int64_t>(0, move[d]);
    }
    hb[world] = off;
    ck(cudaMemcpyAsync(buf, hb.data(), sizeof(unsigned long long) * hb.size(), cudaMemcpyHostToDevice, h->st), "h2d");
    unsigned long long* move_off = buf;
    unsigned long long* taken = buf + world + 1;
    unsigned long long* counts = buf + world + 2;
    unsigned long long* cursor = buf + 2 * world + 2;
    const int blocks = grid_for(n, 256, h->sms * 8);
    h->launches += 2;
    if (n > 0) k_route_assign<<<blocks, 256, 0, h->st>>>(n, world, rank, h->d_route, move_off, taken, counts);
    ck(cudaGetLastError(), "route assign");
    std::vector<unsigned long long> hc(world);
    ck(cudaMemcpyAsync(hc.data(), counts, sizeof(unsigned long long) * world, cudaMemcpyDeviceToHost, h->st), "d2h");
    ck(cudaStreamSynchronize(h->st), "sync");
    // own rows first, then the other ranks in rank order
    std::vector<unsigned long long> cur(world);
    unsigned long long o = hc[rank];
    cur[rank] = 0;
    for (int d = 0; d < world; d++) {
        send_counts[d] = (int64_t)hc[d];
        if (d == rank) continue;
        cur[d] = o;
        o += hc[d];
    }
    ck(cudaMemcpyAsync(cursor, cur.data(), sizeof(unsigned long long) * world, cudaMemcpyHostToDevice, h->st), "h2d");
    if (n > 0)
        k_owner_scatter<N><<<blocks, 256, 0, h->st>>>(h->F[h->cur].f, n, h->d_route, cursor, h->F[h->cur ^ 1].f);
    ck(cudaGetLastError(), "route scatter");
    h->cur ^= 1;
    dfree(buf);
    ck(cudaStreamSynchronize(h->st), "sync");
}

template <int N>
void WidthK<N>::run(rb_handle* h) {
    h->launches++;
    k_width<N><<<grid_for(h->n_cur, 256, h->sms * 8), 256, 0, h->st>>>(h->F[h->cur].f, h->n_cur, h->d_ctr);
    ck(cudaGetLastError(), "width");
}
