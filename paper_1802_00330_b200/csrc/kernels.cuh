// kernels.cuh -- the device side of the B200 engine (sm_100a, FP64 SIMT).
//
//   K3 k_classify   done / degenerate / active split of the frontier + compaction
//                   (bnb.py:249-269), parent exponent guards.
//   K1 k_filter     implicit 2^n bisection + inclusion-function filter + compaction
//                   (bnb.py:161-165, _batch.py:167-238), thread per child.
//   K2 k_hs         Hansen-Sengupta contraction (hansen.py:56-138, bnb.py:190-218),
//                   G lanes per box (G = 2n rounded up to a power of two).
//   k_dedup_*       exact duplicate removal with flag OR (_batch.py:253-266).
//   k_sort_*        canonical order keys + gather (_batch.py:244-250).
//
// Frontier layout in HBM: structure of arrays, component-major:
//   lo[j * cap + row], hi[j * cap + row] (float64), cert[row], unsplit[row] (u8).
// Consecutive threads touch consecutive rows -> fully coalesced 8-byte lanes.
#pragma once
#ifndef __CUDACC_RTC__
#include <climits>
#include <cstdint>
#endif
#include "interval.cuh"

// launch bounds of the round graph's kernels (0: block size only) -- dev knobs
#ifndef RB_CF_MINB
#define RB_CF_MINB 0
#endif
#if RB_CF_MINB > 0
#define RB_CF_BOUNDS __launch_bounds__(256, RB_CF_MINB)
#else
#define RB_CF_BOUNDS __launch_bounds__(256)
#endif
#ifndef RB_FUSED_MINB
#define RB_FUSED_MINB 0
#endif
#if RB_FUSED_MINB > 0
#define RB_FUSED_BOUNDS __launch_bounds__(128, RB_FUSED_MINB)
#else
#define RB_FUSED_BOUNDS __launch_bounds__(128)
#endif

#ifdef __CUDACC_RTC__
// system-specialised kernels (NVRTC) are never launched with graph conditionals
#define RB_SET_COND(h, v) ((void)(h), (void)(v))
#else
#define RB_SET_COND(h, v) cudaGraphSetConditional((h), (v))
#endif

namespace rb {

constexpr int MAX_N = 16;
constexpr int kTraceBlocks = 4096;  // RB_TRACE per-block timeline capacity
constexpr int kTraceBoxes = 8192;   // RB_TRACE per-box HS records (k_hs_fused)
// per-box records start this many words after HsParams::prof
constexpr int kTraceBoxOff = 48 + 7 * kTraceBlocks;  // after the HS and classify-filter block records

// ------------------------------------------------------------------ tables

// Device copy of the compiled system (rb_system), one contiguous global buffer:
//   double   coeff[T]
//   uint16_t poly_off[P + 1]       P = n + n*n
//   uint16_t fac_off[T + 1]
//   uint16_t fac[Fc]               var | exp << 8
struct TabMeta {
    int n, T, Fc, P;
    int TF, FcF;                    // F-only prefix sizes
    int off_poly, off_fac_off, off_fac, bytes;   // byte offsets in the global buffer
    int f_ecmin, f_ecmax, f_deg;    // guard constants: coefficient exponent range, max degree
    int j_ecmin, j_ecmax, j_deg;
    int ops_eq[MAX_N];              // algorithmic ops per equation
    int cost_eq[MAX_N];             // estimated instruction cost per equation (filter ordering)
    int ops_hs_pre;                 // ops of HS preconditioning per box
    int ops_hs_row;                 // ops of one sweep row
    // tabulated filter (k_filter_tab): per-parent term tables
    int ftab;                       // 1 when the tables fit the shared-memory budget
    int e_max;                      // max table entries of one equation (per parent)
    int ent_total;                  // total (term, combo) entries over the equations
    int off_tbase, off_ent_off, off_ent, bytes2;  // byte offsets (tbase u16[TF], ent_off u16[n+1], ent u32[])
    int off_termp, bytes3;          // packed F terms (TermP[TF]) for the direct filter
    // warp-tabulated filter (k_filter_wt): equations whose table would exceed a quarter of a
    // work unit's children are evaluated per child instead (bit e), the others' largest table
    int fwt_direct, fwt_emax;
};

// One F term packed for the direct filter: up to 4 factors of (var < 16,
// exponent 1..16) in one word, so a term costs a single 16-byte shared load.
struct __align__(16) TermP {
    double c;
    uint32_t fpack;   // factor f: bits 8f..8f+3 var, 8f+4..8f+7 exponent - 1
    uint16_t nf;      // number of factors
    uint16_t packed;  // 1: fpack holds every factor; 0: use the general tables
};

struct STab {
    const double* coeff;
    const uint16_t* poly_off;
    const uint16_t* fac_off;
    const uint16_t* fac;
};

__host__ __device__ inline int align8(int x) { return (x + 7) & ~7; }
__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

// bytes of the shared-memory copy (F only when f_only)
__host__ __device__ inline int stab_bytes(const TabMeta& m, bool f_only) {
    const int T = f_only ? m.TF : m.T;
    const int P = f_only ? m.n : m.P;
    const int Fc = f_only ? m.FcF : m.Fc;
    return align8(8 * T) + align8(2 * (P + 1)) + align8(2 * (T + 1)) + align8(2 * Fc);
}

// Asynchronous global -> shared copy (cp.async): every element copy of a table is
// in flight at once instead of each load waiting for the previous shared store
// (generic pointers may alias, so plain load/store loops serialise).  `bytes`
// is rounded up to whole `W`-byte words; both sides must be W-aligned and the
// destination region padded to the rounded size.  Completed by cp_async_wait().
template <int W>
__device__ __forceinline__ void copy_async(void* dst, const void* src, int bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const char* g = reinterpret_cast<const char*>(src);
    for (int i = threadIdx.x * W; i < bytes; i += blockDim.x * W) {
        if constexpr (W == 16)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + i), "l"(g + i) : "memory");
        else
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d + i), "l"(g + i), "n"(W) : "memory");
    }
}
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// issue the table copies (complete with cp_async_wait + a block barrier)
__device__ inline STab issue_stab(const TabMeta& m, const uint8_t* g, uint8_t* s, bool f_only);
__device__ inline STab load_stab(const TabMeta& m, const uint8_t* g, uint8_t* s, bool f_only) {
    const STab t = issue_stab(m, g, s, f_only);
    cp_async_wait();
    return t;
}
__device__ inline STab issue_stab(const TabMeta& m, const uint8_t* g, uint8_t* s, bool f_only) {
    const int T = f_only ? m.TF : m.T;
    const int P = f_only ? m.n : m.P;
    const int Fc = f_only ? m.FcF : m.Fc;
    STab t;
    double* c = reinterpret_cast<double*>(s);
    uint16_t* po = reinterpret_cast<uint16_t*>(s + align8(8 * T));
    uint16_t* fo = reinterpret_cast<uint16_t*>(s + align8(8 * T) + align8(2 * (P + 1)));
    uint16_t* fa = reinterpret_cast<uint16_t*>(s + align8(8 * T) + align8(2 * (P + 1)) + align8(2 * (T + 1)));
    // the global arrays are 8-aligned and zero-padded to 8 bytes, so whole 4-byte words stay in bounds
    copy_async<8>(c, g, 8 * T);
    copy_async<4>(po, g + m.off_poly, 2 * (P + 1));
    copy_async<4>(fo, g + m.off_fac_off, 2 * (T + 1));
    copy_async<4>(fa, g + m.off_fac, 2 * Fc);
    t.coeff = c;
    t.poly_off = po;
    t.fac_off = fo;
    t.fac = fa;
    return t;
}

// Polynomial.eval_interval (poly.py:187-203) / _batch.eval_poly (_batch.py:167-186):
// acc = [0,0]; per term in canonical order: t = [c,c] * x_j1^e1 * ... ; acc += t.
// x component j is at xlo[j*stride], xhi[j*stride].
template <class A>
__device__ __forceinline__ ival eval_poly(const STab& t, int p, const double* xlo, const double* xhi,
                                          int stride) {
    ival acc = mk(0.0, 0.0);
    const int t0 = t.poly_off[p], t1 = t.poly_off[p + 1];
    for (int q = t0; q < t1; ++q) {
        const double c = t.coeff[q];
        const int f0 = t.fac_off[q], f1 = t.fac_off[q + 1];
        ival term;
        if (f0 == f1) {
            term = mk(c, c);
        } else {
            uint32_t fv = t.fac[f0];
            int j = fv & 0xff, k = fv >> 8;
            term = A::mul_point(c, A::pow(mk(xlo[j * stride], xhi[j * stride]), k));
            for (int f = f0 + 1; f < f1; ++f) {
                fv = t.fac[f];
                j = fv & 0xff;
                k = fv >> 8;
                term = A::mul(term, A::pow(mk(xlo[j * stride], xhi[j * stride]), k));
            }
        }
        acc = A::add(acc, term);
    }
    return acc;
}

static __device__ __noinline__ ival eval_poly_exact(const STab& t, int p, const double* xlo, const double* xhi,
                                             int stride) {
    return eval_poly<Exact>(t, p, xlo, xhi, stride);
}

// Guard: every nonzero product of a polynomial evaluation over values with
// exponents in [emin, emax] stays inside the reference's trusted band with a
// 5-binade margin (so the Dekker error is exact and IEEE RD/RU == reference).
__device__ __forceinline__ bool poly_guard_ok(int ecmin, int ecmax, int deg, const ExpRange& r) {
    if (r.emin > r.emax) return true;  // all values zero
    const int lb = min(ecmin, 0) + deg * min(r.emin, 0);
    const int ub = max(ecmax + 1, 0) + deg * max(r.emax + 1, 0);
    return lb >= -965 && ub <= 990;
}

__device__ __forceinline__ bool prod_guard_ok(const ExpRange& a, const ExpRange& b) {
    if (a.emin > a.emax || b.emin > b.emax) return true;  // a side is all zero
    return a.emin + b.emin >= -965 && a.emax + b.emax + 2 <= 990 && a.emax < 990 && b.emax < 990;
}

__device__ __forceinline__ bool mul_guard_ok(ival x, ival y) {
    ExpRange a, b;
    a.init(); b.init();
    a.add(x.lo); a.add(x.hi);
    b.add(y.lo); b.add(y.hi);
    return prod_guard_ok(a, b);
}

// |v| <= 2^989 (operand side of the trusted band), a bit test on the high word
__device__ __forceinline__ bool op_small(double v) {
    return ((unsigned)__double2hiint(v) & 0x7fffffffu) < (2013u << 20);
}
// v == 0 or 2^-965 <= |v| <= 2^988 (result side of the trusted band)
__device__ __forceinline__ bool prod_in_band(double v) {
    const unsigned hi = (unsigned)__double2hiint(v) & 0x7fffffffu;
    return (hi - (58u << 20)) < ((2012u - 58u) << 20) || (hi | (unsigned)__double2loint(v)) == 0u;
}

// interval product, guarded per call (rarely taken slow path).  The guard is
// checked on the IEEE results themselves: every operand at most 2^989 and every
// directed product zero or in [2^-965, 2^988] -- then no product of nonzero
// operands reached the reference's untrusted band (a nonzero exact product below
// it has its away-from-zero rounding nonzero and below 2^-965), so the Dekker
// error is exact and IEEE RD/RU equal _mul_rd/_mul_ru (interval.py:98-136).
// force: always take the Exact product (rb_set_option "force_exact", parity tests of the Exact policy)
__device__ __forceinline__ ival gmul(ival x, ival y, bool force = false) {
    const double p0 = __dmul_rd(x.lo, y.lo), p1 = __dmul_rd(x.lo, y.hi);
    const double p2 = __dmul_rd(x.hi, y.lo), p3 = __dmul_rd(x.hi, y.hi);
    const double q0 = __dmul_ru(x.lo, y.lo), q1 = __dmul_ru(x.lo, y.hi);
    const double q2 = __dmul_ru(x.hi, y.lo), q3 = __dmul_ru(x.hi, y.hi);
    const bool ok = !force & op_small(x.lo) & op_small(x.hi) & op_small(y.lo) & op_small(y.hi) & prod_in_band(p0) &
                    prod_in_band(p1) & prod_in_band(p2) & prod_in_band(p3) & prod_in_band(q0) & prod_in_band(q1) &
                    prod_in_band(q2) & prod_in_band(q3);
    if (ok) return mk(py_min(py_min(p0, p1), py_min(p2, p3)), py_max(py_max(q0, q1), py_max(q2, q3)));
    return Exact::mul(x, y);
}

enum { DIV_EMPTY = 0, DIV_SINGLE = 1, DIV_SPLIT = 2, DIV_WHOLE = 3 };

// interval.py:394-432 (div_extended), Hanson/Kahan case table.
static __device__ __noinline__ int div_extended(ival x, ival y, ival& p0, ival& p1, bool force = false) {
    if (!contains_zero(y)) {
        ival r = mk(div_rd(1.0, y.hi), div_ru(1.0, y.lo));  // recip, interval.py:347-351
        p0 = gmul(x, r, force);  // guarded product: Fast when provably trusted
        return DIV_SINGLE;
    }
    if (y.lo == 0.0 && y.hi == 0.0) {
        if (contains_zero(x)) { p0 = mk(-CUDART_INF, CUDART_INF); return DIV_WHOLE; }
        return DIV_EMPTY;
    }
    if (x.lo < 0.0 && 0.0 < x.hi) { p0 = mk(-CUDART_INF, CUDART_INF); return DIV_WHOLE; }
    if (x.lo == 0.0 && x.hi == 0.0) { p0 = mk(0.0, 0.0); return DIV_SINGLE; }
    if (x.hi <= 0.0) {
        if (y.lo == 0.0) { p0 = mk(-CUDART_INF, div_ru(x.hi, y.hi)); return DIV_SINGLE; }
        if (y.hi == 0.0) { p0 = mk(div_rd(x.hi, y.lo), CUDART_INF); return DIV_SINGLE; }
        double a = div_ru(x.hi, y.hi);
        double b = div_rd(x.hi, y.lo);
        if (a >= b) { p0 = mk(-CUDART_INF, CUDART_INF); return DIV_WHOLE; }
        p0 = mk(-CUDART_INF, a);
        p1 = mk(b, CUDART_INF);
        return DIV_SPLIT;
    }
    if (y.lo == 0.0) { p0 = mk(div_rd(x.lo, y.hi), CUDART_INF); return DIV_SINGLE; }
    if (y.hi == 0.0) { p0 = mk(-CUDART_INF, div_ru(x.lo, y.lo)); return DIV_SINGLE; }
    double a = div_ru(x.lo, y.lo);
    double b = div_rd(x.lo, y.hi);
    if (a >= b) { p0 = mk(-CUDART_INF, CUDART_INF); return DIV_WHOLE; }
    p0 = mk(-CUDART_INF, a);
    p1 = mk(b, CUDART_INF);
    return DIV_SPLIT;
}


// ------------------------------------------------------------------ frontier views

struct Front {
    double* lo;
    double* hi;
    uint8_t* cert;
    uint8_t* unsplit;
    int64_t cap;
};

// The counters every block of a round updates.  The latency-critical ones (the slot
// reservations of the appenders, the block-done counter of the round end) sit on
// their own 128-byte lines, so their atomics do not queue behind each other at L2.
struct Counters {
    alignas(128) unsigned long long n_next;  // rows appended to the next frontier
    alignas(128) unsigned long long n_surv;  // filter survivors (may exceed S capacity)
    alignas(128) unsigned long long tail_done;  // blocks finished (the last one runs the round end)
    alignas(128) unsigned long long wmax;    // bits of max width over the next frontier
    unsigned long long child_wmax;           // bits of max child width over survivors
    alignas(128) unsigned long long n_carried;  // of n_next, carried (done / degenerate)
    unsigned long long n_par;                // active parents
    unsigned long long filter_ops;
    unsigned long long hs_ops;
    unsigned long long hs_calls;
    unsigned long long exact_boxes;
    unsigned long long dups;
    unsigned long long hs_on;
    unsigned long long n_compact;
    // per-equation filter statistics (evaluations, rejections): the next round
    // evaluates the equations in descending rejections-per-op order.  Any order
    // gives the same survivor set -- a child is kept iff every equation encloses 0.
    alignas(128) unsigned long long f_eval[16];
    unsigned long long f_rej[16];
};

// Programmatic dependent launch: round-path kernels are launched with programmatic
// stream serialization, so a kernel's blocks may start while its predecessor drains.
// Every such kernel releases its successor at once and then waits for the full
// completion (and memory visibility) of its predecessor before touching global
// data; because every kernel of the chain waits, completion stays transitive.
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// no-op unless the kernel was launched with a programmatic dependency
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
    pdl_launch();
    pdl_wait();
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ double canon0(double v) { return __dadd_rn(v, 0.0); }  // -0 -> +0

__device__ __forceinline__ void atomic_or_u8_(uint8_t* p, uint8_t v) {
    if (!v) return;
    const size_t a = reinterpret_cast<size_t>(p);
    unsigned* w = reinterpret_cast<unsigned*>(a & ~size_t(3));
    atomicOr(w, (unsigned)v << (8 * (a & 3)));
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// warp-aggregated append: returns the slot of this lane (valid if pred)
__device__ __forceinline__ unsigned long long warp_append(bool pred, unsigned long long* counter,
                                                          unsigned long long mult = 1) {
    const unsigned b = __ballot_sync(0xffffffffu, pred);
    unsigned long long base = 0;
    const int lane = threadIdx.x & 31;
    if (b) {
        const int leader = __ffs(b) - 1;
        if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(b) * mult);
        base = __shfl_sync(0xffffffffu, base, leader);
    }
    return base + (unsigned long long)__popc(b & lanemask_lt()) * mult;
}

// ------------------------------------------------------------------ dedup at append time

// Exact dedup (dedup_sorted, _batch.py:253-266) done by the thread that appends a
// row, instead of a separate pass over the next frontier: the row is stored, made
// visible (fence), then inserted into the open-addressing table; a thread that finds
// an equal row already inserted marks its own row dead and ORs its flags into the
// keeper.  The table, slot_of and dead have the layout k_dedup_insert uses, so the
// round tail cleans up and compacts the same way.
struct DevState;
struct DedupCtx {
    unsigned* table;            // nullptr (and etable nullptr): no dedup at append time
    unsigned long long mask;
    unsigned* slot_of;
    uint8_t* dead;
    // epoch table (ping-pong round graph): entries (epoch << 32 | row + 1); an entry of an
    // older epoch is empty, so the table needs no cleanup pass between rounds
    unsigned long long* etable;
    const DevState* st;         // epoch = st->epoch
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long x);

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned cas_acq_rel(unsigned* p, unsigned cmp, unsigned val) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
    return old;
}

// Which rows can be duplicates.  Frontier rows descend from bisection cells with
// disjoint interiors (children [lo, m], [m, hi]); HS outputs are subsets of their
// input (intersections with it), kept / skipped rows are their input, carried rows
// are unchanged.  The only overlap between lineages comes from an HS fork, whose two
// pieces in the split component are [cur.lo, RU(x + a)] and [RD(x + b), cur.hi] with
// a < b: they can share at most ~2 ulps.  So two equal rows from different entries
// lie in a set with empty interior or a few ulps thick in some component, and a row
// none of whose components is that thin has no duplicate.  Such rows skip the table
// (dead = 0); `kThinUlps` leaves a wide margin over the 2-ulp bound.
constexpr long long kThinUlps = 64;

__device__ __forceinline__ long long ordkey(double x) {  // monotone in x, +0 == -0
    const long long b = __double_as_longlong(x);
    return b >= 0 ? b : (long long)0x8000000000000000ull - b;
}
__device__ __forceinline__ bool thin_comp(double lo, double hi) { return ordkey(hi) - ordkey(lo) <= kThinUlps; }

// row `i` of f holds (lo[j], hi[j]) and the flags, already stored by this thread or
// its lane group and fenced; one thread inserts it.
__device__ __forceinline__ unsigned long long cas_acq_rel64(unsigned long long* p, unsigned long long cmp,
                                                            unsigned long long val) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(val) : "memory");
    return old;
}
__device__ __forceinline__ unsigned state_epoch(const DevState* st);
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int N>
__device__ __forceinline__ void dedup_insert_regs(const Front& f, int64_t i, const double* lo, const double* hi,
                                                  uint8_t cert, uint8_t uns, const DedupCtx& d, Counters* ctr) {
    bool thin = false;
#pragma unroll
    for (int j = 0; j < N; j++) thin |= thin_comp(lo[j], hi[j]);
    if (!thin) {  // cannot have a duplicate (see kThinUlps)
        d.dead[i] = 0;
        d.slot_of[i] = 0xffffffffu;
        return;
    }
    unsigned long long h = 0x9e3779b97f4a7c15ull;  // = row_hash over the stored (canonical) values
#pragma unroll
    for (int j = 0; j < N; j++) {
        h = mix64(h ^ (unsigned long long)__double_as_longlong(__dadd_rn(lo[j], 0.0)));
        h = mix64(h ^ (unsigned long long)__double_as_longlong(__dadd_rn(hi[j], 0.0)));
    }
    unsigned long long slot = h & d.mask;
    bool dup = false;
    const unsigned long long ep = d.etable ? (unsigned long long)state_epoch(d.st) << 32 : 0ull;
    unsigned long long seen = d.etable ? ld_acquire64(&d.etable[slot]) : 0ull;
    while (true) {
        // release: this row's stores (and the group's, ordered by __syncwarp) before the slot is
        // published; acquire: the keeper's row is visible once its slot is seen
        int64_t k;
        if (d.etable) {
            if ((seen >> 32) != (ep >> 32)) {  // empty in this epoch: claim it
                const unsigned long long prev = cas_acq_rel64(&d.etable[slot], seen, ep | (unsigned long long)(i + 1));
                if (prev == seen) break;
                seen = prev;  // lost the race: look at the winner
                continue;
            }
            k = (int64_t)(seen & 0xffffffffull) - 1;
        } else {
            const unsigned prev = cas_acq_rel(&d.table[slot], 0u, (unsigned)(i + 1));
            if (prev == 0u) break;
            k = (int64_t)prev - 1;
        }
        bool eq = true;
#pragma unroll
        for (int j = 0; j < N; j++)
            eq = eq && (ld_cg(&f.lo[j * f.cap + k]) == lo[j]) && (ld_cg(&f.hi[j * f.cap + k]) == hi[j]);
        if (eq) {
            dup = true;
            atomic_or_u8_(&f.cert[k], cert);
            atomic_or_u8_(&f.unsplit[k], uns);
            break;
        }
        slot = (slot + 1) & d.mask;
        if (d.etable) seen = ld_acquire64(&d.etable[slot]);
    }
    d.dead[i] = dup ? 1 : 0;
    d.slot_of[i] = dup ? 0xffffffffu : (unsigned)slot;
    if (dup) atomicAdd(&ctr->dups, 1ull);
}

// ------------------------------------------------------------------ device-resident round loop state

// State of a solve whose round loop runs on the device (a CUDA graph WHILE node,
// engine.cu): the kernels read the frontier size, target and round number here
// instead of from launch parameters, and k_round_end advances it.
struct DevState {
    unsigned long long n_cur;   // rows of the current frontier (always in F[0] in graph mode)
    double target;
    long long max_boxes;
    int round_no;               // round being executed (1-based)
    int max_rounds;
    int done, bail, status, nrounds;
    int n_small_log2;           // bail when n_cur << n exceeds S capacity
    unsigned long long t_round_ns;
    int cur;                    // frontier in F[cur] (ping-pong round graph; k_small_rounds)
    unsigned epoch;             // dedup table epoch of the round (ping-pong round graph)
    int round0;                 // round the graph launch started from (k_solve_start)
    unsigned finish_blocks;     // k_solve_finish blocks done (host sets 0 in the start state)
    unsigned long long seq;     // solve sequence number, echoed to HostX::done_seq at the end
};

__device__ __forceinline__ unsigned state_epoch(const DevState* st) { return *(volatile const unsigned*)&st->epoch; }

struct DevRoundStats {
    long long round, boxes_in, after_filter, after_hs, children, hs_calls, filter_ops, hs_ops, dups, exact, hs_on;
    double width, elapsed;
};

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ K3 classify

// bnb.py:249-269.  Carried rows (done: width <= target or unsplittable; or
// degenerate: some midpoint equals an endpoint) are appended to `next` with
// their flags (degenerate -> cert 0, unsplit 1); the rest become parents.
// Parent entries carry the filter guard verdict in bit 31 (1 = exact path).
template <int N>
__device__ __forceinline__ void k_classify_body(TabMeta meta, Front cur, int64_t n_cur_arg, Front next,
                                                  uint32_t* parents, Counters* ctr, double target_arg,
                                                  const DevState* st, DedupCtx dd = DedupCtx{}) {
    if (st && (st->done || st->bail)) return;  // unrolled round after the end of the device loop
    const int64_t n_cur = st ? (int64_t)st->n_cur : n_cur_arg;
    const double target = st ? st->target : target_arg;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_cur; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < n_cur;
        double lo[N], hi[N];
        double w = 0.0;
        bool carried = false, deg = false, exact = false;
        uint8_t cert = 0, uns = 0;
        if (valid) {
            ExpRange r;
            r.init();
#pragma unroll
            for (int j = 0; j < N; j++) {
                lo[j] = cur.lo[j * cur.cap + i];
                hi[j] = cur.hi[j * cur.cap + i];
                const double d = __dsub_rn(hi[j], lo[j]);
                w = j == 0 ? d : (d > w ? d : w);
            }
            cert = cur.cert[i];
            uns = cur.unsplit[i];
            const bool done = (w <= target) || uns;
            if (!done) {
#pragma unroll
                for (int j = 0; j < N; j++) {
                    const double m = mid_of(lo[j], hi[j]);
                    deg |= (m == lo[j]) || (m == hi[j]);
                    r.add(lo[j]);
                    r.add(hi[j]);
                    r.add(m);
                }
                exact = !poly_guard_ok(meta.f_ecmin, meta.f_ecmax, meta.f_deg, r);
            }
            carried = done || deg;
            if (deg && !done) {
                cert = 0;
                uns = 1;
            }
        }
        // carried rows -> next frontier
        const unsigned long long slot = warp_append(valid && carried, &ctr->n_next);
        if (valid && carried && slot < (unsigned long long)next.cap) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                next.lo[j * next.cap + slot] = lo[j];
                next.hi[j * next.cap + slot] = hi[j];
            }
            next.cert[slot] = cert;
            next.unsplit[slot] = uns;
            if (dd.table || dd.etable) dedup_insert_regs<N>(next, (int64_t)slot, lo, hi, cert, uns, dd, ctr);
        }
        const unsigned long long ps = warp_append(valid && !carried, &ctr->n_par);
        if (valid && !carried) parents[ps] = (uint32_t)i | (exact ? 0x80000000u : 0u);
        // widths of carried rows feed width_now (bnb.py:329)
        unsigned long long wb = (valid && carried) ? (unsigned long long)__double_as_longlong(w) : 0ull;
        wb = warp_max(wb);
        const unsigned long long nc = __popc(__ballot_sync(0xffffffffu, valid && carried));
        if ((threadIdx.x & 31) == 0) {
            if (wb) atomicMax(&ctr->wmax, wb);
            if (nc) atomicAdd(&ctr->n_carried, nc);
        }
    }
}

template <int N>
__global__ void __launch_bounds__(256) k_classify(TabMeta meta, Front cur, int64_t n_cur_arg, Front next,
                                                  uint32_t* parents, Counters* ctr, double target_arg,
                                                  const DevState* st, DedupCtx dd) {
    pdl_enter();
    k_classify_body<N>(meta, cur, n_cur_arg, next, parents, ctr, target_arg, st, dd);
}

// Parents for the rb_filter test hook: every row is a parent (no degeneracy split).
template <int N>
__global__ void k_all_parents(TabMeta meta, Front cur, int64_t n_cur, uint32_t* parents, Counters* ctr) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_cur;
         i += (int64_t)gridDim.x * blockDim.x) {
        ExpRange r;
        r.init();
#pragma unroll
        for (int j = 0; j < N; j++) {
            const double lo = cur.lo[j * cur.cap + i], hi = cur.hi[j * cur.cap + i];
            r.add(lo);
            r.add(hi);
            r.add(mid_of(lo, hi));
        }
        const bool exact = !poly_guard_ok(meta.f_ecmin, meta.f_ecmax, meta.f_deg, r);
        parents[i] = (uint32_t)i | (exact ? 0x80000000u : 0u);
        if (i == 0) ctr->n_par = (unsigned long long)n_cur;
    }
}

// ------------------------------------------------------------------ K1 filter

struct SBuf {  // survivor buffer (HS input), SoA
    double* lo;
    double* hi;
    int64_t cap;
};

// Polynomial.eval_interval (poly.py:187-203) over packed terms; x component j is
// xs2[j * stride] = (lo, hi).  Same operation order as eval_poly.
template <class A>
__device__ __forceinline__ ival eval_poly_packed(const TermP* tp, const STab& t, int p, const double2* xs2,
                                                 int stride) {
    ival acc = mk(0.0, 0.0);
    const int t0 = t.poly_off[p], t1 = t.poly_off[p + 1];
    for (int q = t0; q < t1; ++q) {
        const TermP T = tp[q];
        ival term;
        if (T.nf == 0) {
            term = mk(T.c, T.c);
        } else if (T.packed) {
            uint32_t f = T.fpack;
            double2 x = xs2[(f & 15u) * stride];
            term = A::mul_point(T.c, A::pow(mk(x.x, x.y), (int)((f >> 4) & 15u) + 1));
            for (int k = 1; k < T.nf; k++) {
                f >>= 8;
                x = xs2[(f & 15u) * stride];
                term = A::mul(term, A::pow(mk(x.x, x.y), (int)((f >> 4) & 15u) + 1));
            }
        } else {
            const int f0 = t.fac_off[q], f1 = t.fac_off[q + 1];
            term = mk(T.c, T.c);
            for (int f = f0; f < f1; ++f) {
                const uint32_t fv = t.fac[f];
                const double2 x = xs2[(fv & 0xff) * stride];
                const ival pw = A::pow(mk(x.x, x.y), (int)(fv >> 8));
                term = (f == f0) ? A::mul_point(T.c, pw) : A::mul(term, pw);
            }
        }
        acc = A::add(acc, term);
    }
    return acc;
}

static __device__ __noinline__ ival eval_poly_packed_exact(const TermP* tp, const STab& t, int p, const double2* xs2,
                                                    int stride) {
    return eval_poly_packed<Exact>(tp, t, p, xs2, stride);
}

// Polynomial evaluators.  TabEval interprets the flat tables copied to shared
// memory; a system-specialised evaluator (codegen.cpp, compiled by NVRTC) has the
// same interface with every polynomial as straight-line code and needs no tables.
// Both perform the same operations in the same order, so results are bit-identical.
struct TabEval {
    static constexpr bool tables = true;
    static constexpr bool whole_box = false;  // HS evaluates J(X) and F(x) polynomial by polynomial
    // F equation e over x = xs2[j * stride] = (lo, hi)
    template <class A>
    __device__ __forceinline__ static ival feq(const TermP* tp, const STab& t, int e, const double2* xs2, int stride) {
        return A::exact ? eval_poly_packed_exact(tp, t, e, xs2, stride) : eval_poly_packed<A>(tp, t, e, xs2, stride);
    }
    // k_filter_wt's per-child equations (the specialised evaluator compiles only those)
    template <class A>
    __device__ __forceinline__ static ival feq_direct(const TermP* tp, const STab& t, int e, const double2* xs2,
                                                      int stride) {
        return feq<A>(tp, t, e, xs2, stride);
    }
    // k_filter_wt: f(sum) with sum(c, tb) = tsum of equation e (selected once)
    template <int N, class A, class F>
    __device__ __forceinline__ static void with_tsum(const STab& t, const uint16_t* tbase, int e, F&& f) {
        f([&](uint32_t c, const double2* tb) { return tsum<N, A>(t, tbase, e, c, tb); });
    }
    // k_filter_tab: equation e of child c as the canonical-order sum of its terms' table
    // entries tb[tbase[q] + combo], combo = the child's half bits of the term's factors
    template <int N, class A>
    __device__ __forceinline__ static ival tsum(const STab& t, const uint16_t* tbase, int e, uint32_t c,
                                                const double2* tb) {
        ival acc = mk(0.0, 0.0);
        const int t0 = t.poly_off[e], t1 = t.poly_off[e + 1];
        for (int q = t0; q < t1; q++) {
            int combo = 0;
            for (int f = t.fac_off[q]; f < t.fac_off[q + 1]; f++) {
                const int v = t.fac[f] & 0xff;
                combo = (combo << 1) | (int)((c >> (N - 1 - v)) & 1u);
            }
            const double2 tv = tb[tbase[q] + combo];
            acc = A::add(acc, mk(tv.x, tv.y));
        }
        return acc;
    }
};

// Filter policy.  A sign-selected 2-product multiply (branch on "no operand straddles
// zero", warp-uniform for bisection cells) measured slower than the branch-free 8-product
// tree: katsura6 filter 6.7 -> 11.1 ms, eco8 26.2 -> 33.6 ms (tools/hs_bench.py).
#ifndef RB_FILTER_FAST
#define RB_FILTER_FAST Fast
#endif
#ifndef RB_FILTER_WARPSTAGE
#define RB_FILTER_WARPSTAGE 1  // k_filter: parents staged per warp, no block barrier per iteration
                               // (filter katsura6 6.7 -> 6.2 ms, brown8 5.1 -> 4.3, eco8 23.5 -> 22.7)
#endif
template <int N, class A, class EV = TabEval>
__device__ __forceinline__ bool feasible(const TabMeta& meta, const TermP* tp, const STab& t, const double2* xs2,
                                         int stride, const int* order, unsigned* s_eval, unsigned* s_rej,
                                         bool sample, unsigned& ops) {
    if (!sample) {  // plain short-circuit (bnb.py:149-154) in the adaptive order
#pragma unroll 1
        for (int k = 0; k < N; k++) {
            const int e = order[k];
            const ival v = EV::template feq<A>(tp, t, e, xs2, stride);
            ops += meta.ops_eq[e];
            if (!(v.lo <= 0.0 && 0.0 <= v.hi)) return false;
        }
        return true;
    }
    // sampled blocks also count evaluations / rejections per equation
    const unsigned m = __activemask();
    const int leader = __ffs(m) - 1;
    const int lane = threadIdx.x & 31;
    bool alive = true;
#pragma unroll 1
    for (int k = 0; k < N; k++) {
        const unsigned live = __ballot_sync(m, alive);
        if (live == 0) break;
        const int e = order[k];
        bool rej = false;
        if (alive) {
            const ival v = EV::template feq<A>(tp, t, e, xs2, stride);
            ops += meta.ops_eq[e];
            rej = !(v.lo <= 0.0 && 0.0 <= v.hi);
        }
        const unsigned rm = __ballot_sync(m, rej);
        if (lane == leader) {
            atomicAdd(&s_eval[e], (unsigned)__popc(live));
            if (rm) atomicAdd(&s_rej[e], (unsigned)__popc(rm));
        }
        if (rej) alive = false;
    }
    return alive;
}

__host__ __device__ inline int filter_off_termp(const TabMeta& m) { return align16(stab_bytes(m, true)); }
__host__ __device__ inline int filter_off_xs(const TabMeta& m) { return filter_off_termp(m) + 16 * m.TF; }

// One thread per child.  Child c of parent p takes the low half of component j
// iff bit (n-1-j) of c is 0 (_batch.py:226-238).  Survivors are compacted by
// warp ballot + one atomic per warp into S.  `tags` (test hook) receives the
// child's global index p*2^n + c so the host can restore reference order.
template <int N, class EV = TabEval>
__device__ __forceinline__ void k_filter_body(TabMeta meta, const uint8_t* __restrict__ gtab, Front cur,
                                                const uint32_t* __restrict__ parents, Counters* ctr, SBuf S,
                                                int64_t* tags, const int* __restrict__ eq_order,
                                                int64_t pcount = -1) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int s_order[16];
    __shared__ unsigned s_eval[16], s_rej[16];
    // the system tables are constant: copied before waiting on the previous kernel (PDL)
    TermP* tp = reinterpret_cast<TermP*>(smem + filter_off_termp(meta));
    STab tab{};
    if constexpr (EV::tables) {
        copy_async<16>(tp, gtab + meta.off_termp, 16 * meta.TF);
        tab = issue_stab(meta, gtab, smem, true);
    }
    pdl_wait();
    if (threadIdx.x < 16) {
        s_order[threadIdx.x] = (eq_order && threadIdx.x < N) ? eq_order[threadIdx.x] : (int)threadIdx.x;
        s_eval[threadIdx.x] = 0;
        s_rej[threadIdx.x] = 0;
    }
    const int stride = blockDim.x;
    double2* xs2 = reinterpret_cast<double2*>(smem + filter_off_xs(meta)) + threadIdx.x;
    // parents[0, pcount) (a chunk of a streamed round), else all ctr->n_par of the round;
    // read while the table copies are in flight
    const unsigned long long total = (pcount >= 0 ? (unsigned long long)pcount : ctr->n_par) << N;
    cp_async_wait();
    __syncthreads();
    const unsigned long long gstride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long ops_acc = 0, exact_acc = 0;
    // the block's parents of an iteration (blockDim / 2^N of them, or one parent's slice of
    // children for 2^N >= blockDim): (lo, mid, hi) per component staged once in shared
    // memory, so a child picks its halves with one 16-byte load per component instead of
    // every child re-reading the parent and recomputing the midpoints
    __shared__ double s_par[384];  // max over N of (256 >> N) * N * 3 (N = 1, 2), and 3N for N >= 8
    __shared__ uint8_t s_pex[128];
#if RB_FILTER_WARPSTAGE
    // per warp: its 32 children belong to one parent (n >= 5) or to 32 / 2^n parents,
    // whose (lo, mid, hi) lanes 0 .. np*n-1 stage in the warp's own slice (no block barrier)
    constexpr int np = N >= 5 ? 1 : (32 >> N);
    double* par = s_par + (threadIdx.x >> 5) * 48;
    uint8_t* pex = s_pex + (threadIdx.x >> 5) * 16;
    const int lane_f = threadIdx.x & 31;
#else
    const int log_bd = 31 - __clz((int)blockDim.x);
    const int np = N >= log_bd ? 1 : (int)(blockDim.x >> N);
    double* par = s_par;
    uint8_t* pex = s_pex;
#endif
    for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < total; base += gstride) {
        const unsigned long long idx = base + threadIdx.x;
        const bool valid = idx < total;
#if RB_FILTER_WARPSTAGE
        const unsigned long long p_first = (base + (threadIdx.x & ~31u)) >> N;
        __syncwarp();  // the warp's previous children are done with its slice
        if (lane_f < np * N) {
            const int lp = lane_f / N, j = lane_f - lp * N;
            if (((p_first + lp) << N) < total) {
#else
        const unsigned long long p_first = base >> N;
        __syncthreads();  // the previous iteration's children are done with s_par
        for (int k = threadIdx.x; k < np * N; k += blockDim.x) {
            const int lp = k / N, j = k - lp * N;
            if (((p_first + lp) << N) < total) {
#endif
                const uint32_t pe = parents[p_first + lp];
                const uint32_t p = pe & 0x7fffffffu;
                const double lo = cur.lo[j * cur.cap + p], hi = cur.hi[j * cur.cap + p];
                double* q = par + 3 * (lp * N + j);
                q[0] = lo;
                q[1] = mid_of(lo, hi);
                q[2] = hi;
                if (j == 0) pex[lp] = (uint8_t)(pe >> 31);
            }
        }
#if RB_FILTER_WARPSTAGE
        __syncwarp();
#else
        __syncthreads();
#endif
        bool keep = false;
        double w = 0.0;
        unsigned ops = 0;
        if (valid) {
            const int lp = (int)((idx >> N) - p_first);
            const bool exact = pex[lp] != 0;
            const uint32_t c = (uint32_t)(idx & ((1ull << N) - 1));
#pragma unroll
            for (int j = 0; j < N; j++) {
                const bool up = (c >> (N - 1 - j)) & 1u;
                const double* q = par + 3 * (lp * N + j) + (up ? 1 : 0);
                xs2[j * stride] = make_double2(q[0], q[1]);
            }
            const bool sample = (blockIdx.x & 3) == 0;  // statistics from a quarter of the blocks
            if (!exact) keep = feasible<N, RB_FILTER_FAST, EV>(meta, tp, tab, xs2, stride, s_order, s_eval, s_rej, sample, ops);
            else {
                keep = feasible<N, Exact, EV>(meta, tp, tab, xs2, stride, s_order, s_eval, s_rej, sample, ops);
                exact_acc++;
            }
            ops_acc += ops;
            if (keep) {  // child width (bnb.py:290) only for survivors
#pragma unroll
                for (int j = 0; j < N; j++) {
                    const double2 x = xs2[j * stride];
                    const double d = __dsub_rn(x.y, x.x);
                    w = j == 0 ? d : (d > w ? d : w);
                }
            }
        }
        const unsigned long long slot = warp_append(keep, &ctr->n_surv);
        if (keep && slot < (unsigned long long)S.cap) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                const double2 x = xs2[j * stride];
                S.lo[j * S.cap + slot] = x.x;
                S.hi[j * S.cap + slot] = x.y;
            }
            if (tags) tags[slot] = (int64_t)idx;
        }
        unsigned long long wb = keep ? (unsigned long long)__double_as_longlong(w) : 0ull;
        wb = warp_max(wb);
        if ((threadIdx.x & 31) == 0 && wb) atomicMax(&ctr->child_wmax, wb);
    }
    ops_acc = warp_sum(ops_acc);
    exact_acc = warp_sum(exact_acc);
    if ((threadIdx.x & 31) == 0) {
        if (ops_acc) atomicAdd(&ctr->filter_ops, ops_acc);
        if (exact_acc) atomicAdd(&ctr->exact_boxes, exact_acc);
    }
    __syncthreads();
    if (threadIdx.x < N) {
        if (s_eval[threadIdx.x]) atomicAdd(&ctr->f_eval[threadIdx.x], (unsigned long long)s_eval[threadIdx.x]);
        if (s_rej[threadIdx.x]) atomicAdd(&ctr->f_rej[threadIdx.x], (unsigned long long)s_rej[threadIdx.x]);
    }
}

template <int N, class EV = TabEval>
__global__ void __launch_bounds__(256) k_filter(TabMeta meta, const uint8_t* __restrict__ gtab, Front cur,
                                                const uint32_t* __restrict__ parents, Counters* ctr, SBuf S,
                                                int64_t* tags, const int* __restrict__ eq_order, int64_t pcount) {
    pdl_launch();
    k_filter_body<N, EV>(meta, gtab, cur, parents, ctr, S, tags, eq_order, pcount);  // waits after the table copies
}

// K3 + K1 in one launch for the device round loop: thread per (frontier row, child).
// Each thread classifies its row (the k_classify rules, bnb.py:249-269): a carried
// row is appended to `next` by its child-0 thread (and inserted for exact dedup);
// a parent's children are built and filtered as in k_filter_body.  Saves the
// classify kernel and the parents list round trip; costs 2^n - 1 idle threads per
// carried row, which is why only the small rounds of the round graph use it.
template <int N, class EV = TabEval>
__global__ void RB_CF_BOUNDS k_classify_filter(TabMeta meta, const uint8_t* __restrict__ gtab, Front cur,
                                                         Front next, Counters* ctr, SBuf S, const DevState* st,
                                                         const int* __restrict__ eq_order, DedupCtx dd,
                                                         unsigned long long* prof) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int s_order[16];
    __shared__ unsigned s_eval[16], s_rej[16];
    // RB_TRACE: (start, tables ready, loop done, end) of each block
    unsigned long long* btr = (prof && threadIdx.x == 0 && blockIdx.x < kTraceBlocks) ? prof + 4 * blockIdx.x : nullptr;
    const unsigned long long t_start = btr ? gtimer() : 0ull;
    TermP* tp = reinterpret_cast<TermP*>(smem + filter_off_termp(meta));
    STab tab{};
    if constexpr (EV::tables) {
        copy_async<16>(tp, gtab + meta.off_termp, 16 * meta.TF);
        tab = issue_stab(meta, gtab, smem, true);
    }
    pdl_enter();
    if (threadIdx.x < 16) {
        s_order[threadIdx.x] = threadIdx.x < N ? eq_order[threadIdx.x] : (int)threadIdx.x;
        s_eval[threadIdx.x] = 0;
        s_rej[threadIdx.x] = 0;
    }
    const bool skip = st->done || st->bail;  // unrolled round after the end of the device loop
    if (skip) btr = nullptr;
    if (btr) btr[0] = t_start;
    const int64_t n_cur = skip ? 0 : (int64_t)st->n_cur;
    const double target = st->target;
    const int stride = blockDim.x;
    double2* xs2 = reinterpret_cast<double2*>(smem + filter_off_xs(meta)) + threadIdx.x;
    cp_async_wait();
    __syncthreads();
    if (btr) btr[1] = gtimer();
    const unsigned long long total = (unsigned long long)n_cur << N;
    const unsigned long long gstride = (unsigned long long)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    unsigned long long ops_acc = 0, exact_acc = 0;
    for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < total; base += gstride) {
        const unsigned long long idx = base + threadIdx.x;
        const bool valid = idx < total;
        const int64_t p = (int64_t)(idx >> N);
        const uint32_t c = (uint32_t)(idx & ((1ull << N) - 1));
        bool keep = false, carried = false, parent = false;
        double w = 0.0, wrow = 0.0;
        double lo[N], hi[N];
        uint8_t cert = 0, uns = 0;
        unsigned ops = 0;
        if (valid) {
            ExpRange r;
            r.init();
            bool deg = false;
#pragma unroll
            for (int j = 0; j < N; j++) {
                lo[j] = cur.lo[j * cur.cap + p];
                hi[j] = cur.hi[j * cur.cap + p];
                const double d = __dsub_rn(hi[j], lo[j]);
                wrow = j == 0 ? d : (d > wrow ? d : wrow);
            }
            cert = cur.cert[p];
            uns = cur.unsplit[p];
            const bool done = (wrow <= target) || uns;
            if (!done) {
#pragma unroll
                for (int j = 0; j < N; j++) {
                    const double m = mid_of(lo[j], hi[j]);
                    deg |= (m == lo[j]) || (m == hi[j]);
                    r.add(lo[j]);
                    r.add(hi[j]);
                    r.add(m);
                    const bool up = (c >> (N - 1 - j)) & 1u;
                    const double cl = up ? m : lo[j], ch = up ? hi[j] : m;
                    xs2[j * stride] = make_double2(cl, ch);
                    const double d = __dsub_rn(ch, cl);
                    w = j == 0 ? d : (d > w ? d : w);
                }
            }
            carried = done || deg;
            if (deg && !done) {
                cert = 0;
                uns = 1;
            }
            parent = !carried;
            if (parent) {
                const bool exact = !poly_guard_ok(meta.f_ecmin, meta.f_ecmax, meta.f_deg, r);
                const bool sample = (blockIdx.x & 3) == 0;  // statistics from a quarter of the blocks
                if (!exact) keep = feasible<N, RB_FILTER_FAST, EV>(meta, tp, tab, xs2, stride, s_order, s_eval, s_rej, sample, ops);
                else {
                    keep = feasible<N, Exact, EV>(meta, tp, tab, xs2, stride, s_order, s_eval, s_rej, sample, ops);
                    exact_acc++;
                }
                ops_acc += ops;
            }
        }
        // carried rows -> next frontier (child-0 thread of the row)
        const bool app = valid && carried && c == 0;
        const unsigned long long cs = warp_append(app, &ctr->n_next);
        if (app && cs < (unsigned long long)next.cap) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                next.lo[j * next.cap + cs] = lo[j];
                next.hi[j * next.cap + cs] = hi[j];
            }
            next.cert[cs] = cert;
            next.unsplit[cs] = uns;
            if (dd.table || dd.etable) {
                dedup_insert_regs<N>(next, (int64_t)cs, lo, hi, cert, uns, dd, ctr);
            }
        }
        // survivors -> S
        const unsigned long long slot = warp_append(keep, &ctr->n_surv);
        if (keep && slot < (unsigned long long)S.cap) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                const double2 x = xs2[j * stride];
                S.lo[j * S.cap + slot] = x.x;
                S.hi[j * S.cap + slot] = x.y;
            }
        }
        unsigned long long wb = keep ? (unsigned long long)__double_as_longlong(w) : 0ull;
        unsigned long long wc = app ? (unsigned long long)__double_as_longlong(wrow) : 0ull;
        wb = warp_max(wb);
        wc = warp_max(wc);
        const unsigned nc = __popc(__ballot_sync(0xffffffffu, app));
        const unsigned np = __popc(__ballot_sync(0xffffffffu, valid && parent && c == 0));
        if (lane == 0) {
            if (wb) atomicMax(&ctr->child_wmax, wb);
            if (wc) atomicMax(&ctr->wmax, wc);
            if (nc) atomicAdd(&ctr->n_carried, (unsigned long long)nc);
            if (np) atomicAdd(&ctr->n_par, (unsigned long long)np);
        }
    }
    if (btr) btr[2] = gtimer();
    ops_acc = warp_sum(ops_acc);
    exact_acc = warp_sum(exact_acc);
    if (lane == 0) {
        if (ops_acc) atomicAdd(&ctr->filter_ops, ops_acc);
        if (exact_acc) atomicAdd(&ctr->exact_boxes, exact_acc);
    }
    __syncthreads();
    if (threadIdx.x < N) {
        if (s_eval[threadIdx.x]) atomicAdd(&ctr->f_eval[threadIdx.x], (unsigned long long)s_eval[threadIdx.x]);
        if (s_rej[threadIdx.x]) atomicAdd(&ctr->f_rej[threadIdx.x], (unsigned long long)s_rej[threadIdx.x]);
    }
    if (btr) btr[3] = gtimer();
}

// Next round's equation order: descending rejections per algorithmic op, from
// this round's counts (equations not evaluated keep their relative position).
__host__ __device__ inline void filter_order(const unsigned long long* ev, const unsigned long long* rj,
                                             const int* ops_eq, int n, int* order) {
    double key[16];
    for (int e = 0; e < n; e++)
        key[e] = ev[e] ? ((double)rj[e] / (double)ev[e]) / (double)(ops_eq[e] > 0 ? ops_eq[e] : 1) : -1.0;
    int cur[16];
    for (int k = 0; k < n; k++) cur[k] = order[k];
    // stable insertion sort of the current order by key (unknown keys stay in place relative to each other)
    for (int a = 1; a < n; a++) {
        const int e = cur[a];
        int b = a - 1;
        while (b >= 0 && key[cur[b]] < key[e] && key[e] >= 0.0) {
            cur[b + 1] = cur[b];
            b--;
        }
        cur[b + 1] = e;
    }
    for (int k = 0; k < n; k++) order[k] = cur[k];
}

// ------------------------------------------------------------------ K1' tabulated filter
//
// Every child of a parent is a product of half intervals of the parent:
// component j is [lo_j, m_j] or [m_j, hi_j].  A term c * x_v1^e1 * ... * x_vd^ed
// therefore takes at most 2^d distinct values over the 2^n children.  The block
// computes those values once per parent (same operands, same operation order as
// the per-child evaluation, so the bits are identical), and each child thread
// evaluates an equation as the canonical-order sum of table lookups.  Tables are
// built lazily per equation, only while some child of the block is still alive
// (the reference's short-circuit, bnb.py:149-154).

template <int N>
struct FtabShape {
    static constexpr int LOGPPB = N >= 8 ? 0 : 8 - N;   // parents per 256-thread work unit (log2)
    static constexpr int PPB = 1 << LOGPPB;
    static constexpr int CHLOG = N > 8 ? N - 8 : 0;     // 256-child chunks per parent (log2)
};

__host__ __device__ inline int ftab_meta_bytes(const TabMeta& m) {
    return align8(2 * m.TF) + align8(2 * (m.n + 1)) + align8(4 * m.ent_total);
}

// dynamic shared memory layout of k_filter_tab
template <int N>
__host__ __device__ inline int ftab_off_sp(const TabMeta& m) {
    return align16(stab_bytes(m, true) + ftab_meta_bytes(m));
}
template <int N>
__host__ __device__ inline int ftab_off_table(const TabMeta& m) {
    return align16(ftab_off_sp<N>(m) + FtabShape<N>::PPB * (3 * N + 1) * 8);
}
template <int N>
__host__ __device__ inline int ftab_smem_bytes(const TabMeta& m) {
    return ftab_off_table<N>(m) + FtabShape<N>::PPB * m.e_max * 16;
}

template <class A>
__device__ __forceinline__ ival term_value(const STab& t, int q, int combo, const double* plo, const double* phi,
                                           const double* pmid) {
    const double c = t.coeff[q];
    const int f0 = t.fac_off[q], f1 = t.fac_off[q + 1];
    if (f0 == f1) return mk(c, c);
    const int d = f1 - f0;
    ival term = mk(c, c);
    for (int f = f0; f < f1; f++) {
        const uint32_t fv = t.fac[f];
        const int v = fv & 0xff, k = fv >> 8;
        const bool up = (combo >> (d - 1 - (f - f0))) & 1;
        const ival half = up ? mk(pmid[v], phi[v]) : mk(plo[v], pmid[v]);
        const ival pw = A::pow(half, k);
        term = (f == f0) ? A::mul_point(c, pw) : A::mul(term, pw);
    }
    return term;
}

static __device__ __noinline__ ival term_value_exact(const STab& t, int q, int combo, const double* plo, const double* phi,
                                              const double* pmid) {
    return term_value<Exact>(t, q, combo, plo, phi, pmid);
}

template <int N, class EV = TabEval>
__global__ void __launch_bounds__(256) k_filter_tab(TabMeta meta, const uint8_t* __restrict__ gtab, Front cur,
                                                    const uint32_t* __restrict__ parents, Counters* ctr, SBuf S,
                                                    int64_t* tags, const int* __restrict__ eq_order, int64_t pcount) {
    pdl_enter();
    using Sh = FtabShape<N>;
    __shared__ int s_order[16];
    __shared__ unsigned s_eval[16], s_rej[16];
    if (threadIdx.x < 16) {
        s_order[threadIdx.x] = (eq_order && threadIdx.x < N) ? eq_order[threadIdx.x] : (int)threadIdx.x;
        s_eval[threadIdx.x] = 0;
        s_rej[threadIdx.x] = 0;
    }
    extern __shared__ __align__(16) uint8_t smem[];
    const STab tab = load_stab(meta, gtab, smem, true);
    uint8_t* p8 = smem + stab_bytes(meta, true);
    uint16_t* tbase = reinterpret_cast<uint16_t*>(p8);
    uint16_t* ent_off = reinterpret_cast<uint16_t*>(p8 + align8(2 * meta.TF));
    uint32_t* ent = reinterpret_cast<uint32_t*>(p8 + align8(2 * meta.TF) + align8(2 * (N + 1)));
    double* sp = reinterpret_cast<double*>(smem + ftab_off_sp<N>(meta));  // [PPB][3N + 1]: lo, hi, mid, exact
    double2* table = reinterpret_cast<double2*>(smem + ftab_off_table<N>(meta));
    copy_async<4>(tbase, gtab + meta.off_tbase, 2 * meta.TF);
    copy_async<4>(ent_off, gtab + meta.off_ent_off, 2 * (N + 1));
    copy_async<4>(ent, gtab + meta.off_ent, 4 * meta.ent_total);
    cp_async_wait();
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const unsigned long long n_par = pcount >= 0 ? (unsigned long long)pcount : ctr->n_par;
    const unsigned long long units =
        N >= 8 ? (n_par << Sh::CHLOG) : ((n_par + Sh::PPB - 1) >> Sh::LOGPPB);
    unsigned long long ops_acc = 0, exact_acc = 0;
    for (unsigned long long u = blockIdx.x; u < units; u += gridDim.x) {
        int lp;
        unsigned long long pidx, pbase;
        uint32_t c;
        if (N >= 8) {
            lp = 0;
            pbase = pidx = u >> Sh::CHLOG;
            c = (uint32_t)(((u & ((1ull << Sh::CHLOG) - 1)) << 8) | (unsigned)tid);
        } else {
            lp = tid >> N;
            pbase = u << Sh::LOGPPB;
            pidx = pbase + lp;
            c = (uint32_t)(tid & ((1 << N) - 1));
        }
        const bool valid = pidx < n_par;
        __syncthreads();  // the previous unit is done with sp / table
        for (int k = tid; k < Sh::PPB * N; k += blockDim.x) {
            const int l2 = k / N, j = k % N;
            const unsigned long long p = pbase + l2;
            double* q = sp + l2 * (3 * N + 1);
            if (p < n_par) {
                const uint32_t pe = parents[p];
                const uint32_t row = pe & 0x7fffffffu;
                const double lo = cur.lo[j * cur.cap + row], hi = cur.hi[j * cur.cap + row];
                q[j] = lo;
                q[N + j] = hi;
                q[2 * N + j] = mid_of(lo, hi);
                if (j == 0) q[3 * N] = (pe >> 31) ? 1.0 : 0.0;
            }
        }
        __syncthreads();
        const double* my = sp + lp * (3 * N + 1);
        const bool exact = valid && my[3 * N] != 0.0;
        bool alive = valid;
        unsigned ops = 0;
#pragma unroll 1
        for (int k = 0; k < N; k++) {
            const int e = s_order[k];
            const int n_alive = __syncthreads_count(alive);  // also: everyone is done with the previous tables
            if (n_alive == 0) break;
            if (tid == 0) atomicAdd(&s_eval[e], (unsigned)n_alive);
            const int e0 = ent_off[e], E = ent_off[e + 1] - e0;
            for (int k = tid; k < Sh::PPB * E; k += blockDim.x) {
                const int l2 = k / E, i = k % E;
                if (pbase + l2 >= n_par) continue;
                const uint32_t en = ent[e0 + i];
                const double* q = sp + l2 * (3 * N + 1);
                const ival v = (q[3 * N] != 0.0) ? term_value_exact(tab, en & 0xffff, en >> 16, q, q + N, q + 2 * N)
                                                 : term_value<RB_FILTER_FAST>(tab, en & 0xffff, en >> 16, q, q + N, q + 2 * N);
                table[l2 * meta.e_max + i] = make_double2(v.lo, v.hi);
            }
            __syncthreads();
            if (alive) {
                const double2* tb = table + lp * meta.e_max;
                const ival acc = exact ? EV::template tsum<N, Exact>(tab, tbase, e, c, tb)
                                       : EV::template tsum<N, Fast>(tab, tbase, e, c, tb);
                ops += meta.ops_eq[e];
                alive = acc.lo <= 0.0 && 0.0 <= acc.hi;
                if (!alive) atomicAdd(&s_rej[e], 1u);
            }
        }
        ops_acc += ops;
        exact_acc += exact ? 1 : 0;
        // survivors -> S (warp ballot + one atomic per warp)
        const bool keep = alive;
        const unsigned long long slot = warp_append(keep, &ctr->n_surv);
        double w = 0.0;
        if (keep) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                const bool up = (c >> (N - 1 - j)) & 1u;
                const double cl = up ? my[2 * N + j] : my[j];
                const double ch = up ? my[N + j] : my[2 * N + j];
                const double d = __dsub_rn(ch, cl);
                w = j == 0 ? d : (d > w ? d : w);
                if (slot < (unsigned long long)S.cap) {
                    S.lo[j * S.cap + slot] = cl;
                    S.hi[j * S.cap + slot] = ch;
                }
            }
            if (tags && slot < (unsigned long long)S.cap) tags[slot] = (int64_t)((pidx << N) | c);
        }
        unsigned long long wb = keep ? (unsigned long long)__double_as_longlong(w) : 0ull;
        wb = warp_max(wb);
        if (lane == 0 && wb) atomicMax(&ctr->child_wmax, wb);
    }
    ops_acc = warp_sum(ops_acc);
    exact_acc = warp_sum(exact_acc);
    if (lane == 0) {
        if (ops_acc) atomicAdd(&ctr->filter_ops, ops_acc);
        if (exact_acc) atomicAdd(&ctr->exact_boxes, exact_acc);
    }
    __syncthreads();
    if (threadIdx.x < N) {
        if (s_eval[threadIdx.x]) atomicAdd(&ctr->f_eval[threadIdx.x], (unsigned long long)s_eval[threadIdx.x]);
        if (s_rej[threadIdx.x]) atomicAdd(&ctr->f_rej[threadIdx.x], (unsigned long long)s_rej[threadIdx.x]);
    }
}

// K1'' warp-tabulated filter: the tables of k_filter_tab, one warp per parent (n >= 5:
// 2^n / 32 children per lane).  The warp stages its parent, builds equation e's table
// (entries over the 32 lanes) only while one of its children is alive, and sums the
// table entries for its live children: no block barrier, and the 8 warps of a block
// work on 8 parents independently.  Same term values and summation order as
// k_filter / k_filter_tab (bit-identical); survivors compacted per child bit.
template <int N>
__host__ __device__ inline int fwt_warp_doubles(const TabMeta& m) {
    return ((3 * N + 1 + 1) & ~1) + 2 * m.fwt_emax;  // parent (lo, hi, mid, exact) + table (double2)
}
// per-child evaluation of the direct equations: packed terms, then a child box per thread
template <int N>
__host__ __device__ inline int fwt_off_termp(const TabMeta& m, int threads) {
    return align16(ftab_off_sp<N>(m) + (threads / 32) * fwt_warp_doubles<N>(m) * 8);
}
template <int N>
__host__ __device__ inline int fwt_off_xs(const TabMeta& m, int threads) {
    return align16(fwt_off_termp<N>(m, threads) + 16 * m.TF);
}
template <int N>
__host__ __device__ inline int fwt_smem_bytes(const TabMeta& m, int threads) {
    if (!m.fwt_direct) return ftab_off_sp<N>(m) + (threads / 32) * fwt_warp_doubles<N>(m) * 8;
    return fwt_off_xs<N>(m, threads) + 16 * N * threads;
}

#ifndef RB_FWT_UNROLL
#define RB_FWT_UNROLL 2
#endif
// k_filter_wt's minimum blocks per SM (0: block size only).  ptxas settles on 80
// registers with ~100 B of spills either way; 3 measured best (brown8 filter 3.65 ->
// 3.48 ms, eco8 5.57 -> 5.40; 2 blocks: slower), a compacted evaluation of the live
// children after the first equation slower still (eco8 5.6 -> 6.3 ms)
#ifndef RB_FWT_MINB
#define RB_FWT_MINB 3
#endif
#if RB_FWT_MINB > 0
#define RB_FWT_BOUNDS __launch_bounds__(256, RB_FWT_MINB)
#else
#define RB_FWT_BOUNDS __launch_bounds__(256)
#endif
constexpr int kFwtUnroll = RB_FWT_UNROLL;
// HYB: some equations evaluated per child (meta.fwt_direct); a separate instantiation, as
// that path's code in the loop cost the all-table systems ~15 % (instruction fetch)
template <int N, class EV = TabEval, bool HYB = false>
__global__ void RB_FWT_BOUNDS k_filter_wt(TabMeta meta, const uint8_t* __restrict__ gtab, Front cur,
                                                   const uint32_t* __restrict__ parents, Counters* ctr, SBuf S,
                                                   int64_t* tags, const int* __restrict__ eq_order, int64_t pcount) {
    pdl_enter();
    if constexpr (N >= 5 && N <= 16) {
        // a work unit = one parent's 32 K children: K = 2^n / 32 up to n = 10, above that
        // a parent is CH units of 1024 children (each unit builds the tables it needs)
        constexpr int K = N <= 10 ? (1 << N) / 32 : 32;  // children per lane: c = c0 + 32 i + lane
        constexpr int CHLOG = N <= 10 ? 0 : N - 10;
        __shared__ int s_order[16];
        __shared__ unsigned s_eval[16], s_rej[16];
        if (threadIdx.x < 16) {
            s_order[threadIdx.x] = (eq_order && threadIdx.x < N) ? eq_order[threadIdx.x] : (int)threadIdx.x;
            s_eval[threadIdx.x] = 0;
            s_rej[threadIdx.x] = 0;
        }
        extern __shared__ __align__(16) uint8_t smem[];
        const STab tab = issue_stab(meta, gtab, smem, true);
        uint8_t* p8 = smem + stab_bytes(meta, true);
        uint16_t* tbase = reinterpret_cast<uint16_t*>(p8);
        uint16_t* ent_off = reinterpret_cast<uint16_t*>(p8 + align8(2 * meta.TF));
        uint32_t* ent = reinterpret_cast<uint32_t*>(p8 + align8(2 * meta.TF) + align8(2 * (N + 1)));
        copy_async<4>(tbase, gtab + meta.off_tbase, 2 * meta.TF);
        copy_async<4>(ent_off, gtab + meta.off_ent_off, 2 * (N + 1));
        copy_async<4>(ent, gtab + meta.off_ent, 4 * meta.ent_total);
        TermP* tp = reinterpret_cast<TermP*>(smem + fwt_off_termp<N>(meta, blockDim.x));
        double2* xs2 = reinterpret_cast<double2*>(smem + fwt_off_xs<N>(meta, blockDim.x)) + threadIdx.x;
        if (HYB) copy_async<16>(tp, gtab + meta.off_termp, 16 * meta.TF);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        double* sp = reinterpret_cast<double*>(smem + ftab_off_sp<N>(meta)) + wid * fwt_warp_doubles<N>(meta);
        double2* table = reinterpret_cast<double2*>(sp + ((3 * N + 1 + 1) & ~1));
        const unsigned long long n_par = pcount >= 0 ? (unsigned long long)pcount : ctr->n_par;
        cp_async_wait();
        __syncthreads();
        unsigned long long ops_acc = 0, exact_acc = 0;
        const unsigned long long units = n_par << CHLOG;
        for (unsigned long long unit = (unsigned long long)blockIdx.x * nw + wid; unit < units;
             unit += (unsigned long long)gridDim.x * nw) {
            const unsigned long long pidx = unit >> CHLOG;
            const uint32_t c0 = (uint32_t)(unit & ((1ull << CHLOG) - 1)) << 10;
            __syncwarp();  // the previous unit's children are done with sp / table
            if (lane < N) {
                const uint32_t pe = parents[pidx];
                const uint32_t row = pe & 0x7fffffffu;
                const double lo = cur.lo[lane * cur.cap + row], hi = cur.hi[lane * cur.cap + row];
                sp[lane] = lo;
                sp[N + lane] = hi;
                sp[2 * N + lane] = mid_of(lo, hi);
                if (lane == 0) sp[3 * N] = (pe >> 31) ? 1.0 : 0.0;
            }
            __syncwarp();
            const bool exact = sp[3 * N] != 0.0;
            uint32_t alive = K >= 32 ? 0xffffffffu : ((1u << K) - 1u);
            unsigned ops = 0;
#pragma unroll 1
            for (int k = 0; k < N; k++) {
                if (__ballot_sync(0xffffffffu, alive != 0) == 0) break;
                const int e = s_order[k];
                if (HYB && ((meta.fwt_direct >> e) & 1)) {  // per child, as k_filter (same operations)
                    const uint32_t before = alive;
#pragma unroll 1
                    for (int i = 0; i < K; i++) {
                        if (!((alive >> i) & 1u)) continue;
                        const uint32_t c = c0 + (uint32_t)(32 * i + lane);
#pragma unroll
                        for (int j = 0; j < N; j++) {
                            const bool up = (c >> (N - 1 - j)) & 1u;
                            xs2[j * blockDim.x] = up ? make_double2(sp[2 * N + j], sp[N + j])
                                                     : make_double2(sp[j], sp[2 * N + j]);
                        }
                        const ival v = exact ? EV::template feq_direct<Exact>(tp, tab, e, xs2, blockDim.x)
                                             : EV::template feq_direct<RB_FILTER_FAST>(tp, tab, e, xs2, blockDim.x);
                        if (!(v.lo <= 0.0 && 0.0 <= v.hi)) alive &= ~(1u << i);
                    }
                    const unsigned ne = (unsigned)__popc(before), nr = ne - (unsigned)__popc(alive);
                    ops += ne * (unsigned)meta.ops_eq[e];
                    if ((blockIdx.x & 3) == 0) {
                        const unsigned se = __reduce_add_sync(0xffffffffu, ne), sr = __reduce_add_sync(0xffffffffu, nr);
                        if (lane == 0) {
                            atomicAdd(&s_eval[e], se);
                            if (sr) atomicAdd(&s_rej[e], sr);
                        }
                    }
                    continue;
                }
                const int e0 = ent_off[e], E = ent_off[e + 1] - e0;
                for (int i = lane; i < E; i += 32) {
                    const uint32_t en = ent[e0 + i];
                    const ival v = exact ? term_value_exact(tab, en & 0xffff, en >> 16, sp, sp + N, sp + 2 * N)
                                         : term_value<RB_FILTER_FAST>(tab, en & 0xffff, en >> 16, sp, sp + N, sp + 2 * N);
                    table[i] = make_double2(v.lo, v.hi);
                }
                __syncwarp();
                const uint32_t before = alive;
                // the equation's sum is selected once (not per child); with every child of the
                // lane alive the K sums are independent chains, evaluated without branches
                auto sweep = [&](auto fts) {
                    if (alive == (K >= 32 ? 0xffffffffu : ((1u << K) - 1u))) {
                        uint32_t keep = 0;
#pragma unroll kFwtUnroll  // bounded: the loop is instantiated once per equation (instruction cache)
                        for (int i = 0; i < K; i++) {
                            const ival acc = fts(c0 + (uint32_t)(32 * i + lane), table);
                            keep |= (uint32_t)(acc.lo <= 0.0 && 0.0 <= acc.hi) << i;
                        }
                        alive = keep;
                    } else {
#pragma unroll 1
                        for (int i = 0; i < K; i++) {
                            if ((alive >> i) & 1u) {
                                const ival acc = fts(c0 + (uint32_t)(32 * i + lane), table);
                                if (!(acc.lo <= 0.0 && 0.0 <= acc.hi)) alive &= ~(1u << i);
                            }
                        }
                    }
                };
                if (exact) EV::template with_tsum<N, Exact>(tab, tbase, e, sweep);
                else EV::template with_tsum<N, Fast>(tab, tbase, e, sweep);
                const unsigned ne = (unsigned)__popc(before), nr = ne - (unsigned)__popc(alive);
                ops += ne * (unsigned)meta.ops_eq[e];
                if ((blockIdx.x & 3) == 0) {  // statistics from a quarter of the blocks (as k_filter)
                    const unsigned se = __reduce_add_sync(0xffffffffu, ne), sr = __reduce_add_sync(0xffffffffu, nr);
                    if (lane == 0) {
                        atomicAdd(&s_eval[e], se);
                        if (sr) atomicAdd(&s_rej[e], sr);
                    }
                }
                __syncwarp();  // the table is rebuilt for the next equation
            }
            ops_acc += ops;
            if (lane == 0 && exact) exact_acc += 32u * K;
            // survivors -> S, one child bit at a time (ballot + one atomic per non-empty bit)
            double w = 0.0;
#pragma unroll 1
            for (int i = 0; i < K; i++) {
                if (__ballot_sync(0xffffffffu, alive != 0) == 0) break;
                const bool keep = (alive >> i) & 1u;
                const unsigned long long slot = warp_append(keep, &ctr->n_surv);
                if (keep) {
                    const uint32_t c = c0 + (uint32_t)(32 * i + lane);
#pragma unroll
                    for (int j = 0; j < N; j++) {
                        const bool up = (c >> (N - 1 - j)) & 1u;
                        const double cl = up ? sp[2 * N + j] : sp[j];
                        const double ch = up ? sp[N + j] : sp[2 * N + j];
                        const double d = __dsub_rn(ch, cl);
                        w = (d > w) ? d : w;
                        if (slot < (unsigned long long)S.cap) {
                            S.lo[j * S.cap + slot] = cl;
                            S.hi[j * S.cap + slot] = ch;
                        }
                    }
                    if (tags && slot < (unsigned long long)S.cap) tags[slot] = (int64_t)((pidx << N) | c);
                }
                alive &= ~(1u << i);
            }
            unsigned long long wb = (unsigned long long)__double_as_longlong(w);
            wb = warp_max(wb);
            if (lane == 0 && wb) atomicMax(&ctr->child_wmax, wb);
        }
        ops_acc = warp_sum(ops_acc);
        if (lane == 0) {
            if (ops_acc) atomicAdd(&ctr->filter_ops, ops_acc);
            if (exact_acc) atomicAdd(&ctr->exact_boxes, exact_acc);
        }
        __syncthreads();
        if (threadIdx.x < N) {
            if (s_eval[threadIdx.x]) atomicAdd(&ctr->f_eval[threadIdx.x], (unsigned long long)s_eval[threadIdx.x]);
            if (s_rej[threadIdx.x]) atomicAdd(&ctr->f_rej[threadIdx.x], (unsigned long long)s_rej[threadIdx.x]);
        }
    }
}

// ------------------------------------------------------------------ K2 Hansen-Sengupta
//
// hansen.contract (hansen.py:56-138) over a batch of boxes as a three-kernel
// pipeline with an HBM scratch of J/M, F(x)/g and x per box (SoA, stride B):
//
//   K2a k_hs_eval   thread per box: x = mid(X), J(X) (n^2 interval polynomials),
//                   F(x) (n point polynomials) -- the same uniform interpreter as K1
//   K2b k_hs_lin    G lanes per box: mid(J), Gauss-Jordan inverse A (lane = column,
//                   registers), M = A J and g = A F(x), written back over J / F(x)
//   K2c k_hs_sweep  thread per box: Gauss-Seidel sweep with extended division,
//                   fork / certification, compaction of 0-2 outputs into F_next
//
// The scratch costs ~2 x (2n^2 + 3n) x 8 B of HBM traffic per box (written by K2a, read
// and rewritten by K2b, read by K2c): ~2.8 KB per box at n = 8 against 0.3 KB of frontier
// I/O (ncu, brown8 round 6: 8.2 GB for 2.96M boxes in k_hs_lin_tps).  It is not what
// bounds these kernels (k_hs_lin_tps runs at 1.6 TB/s, ~25 % of HBM): keeping the
// operands on chip (k_hs_tile) cost more residency than the traffic it saved.

struct HsParams {
    int round_no;
    int hs_mode;           // 0: decide on device (bnb.py:289-296), 1: force on, 2: force off
    int hs_enable_round;   // < 0: None
    int hs_possible;
    double hs_enable_width;// NaN: None
    int contract_output;   // SolverConfig.hs_contract
    int count_from_ctr;    // n_in = ctr->n_surv instead of n_in arg
    const DevState* st;    // graph mode: the round number comes from the device state
    long long fused_max;   // k_hs_fused takes n_in <= fused_max rows, eval/lin/sweep take larger counts
    int has_cond;          // graph mode: k_hs_fused selects the eval/lin/sweep branch (IF node)
    cudaGraphConditionalHandle big_cond;
    unsigned long long* prof;  // RB_TRACE: k_hs_fused phase clocks of block 0's first box (dev aid)
    DedupCtx dd;           // k_hs_fused / pass-through: dedup at append time (table null: off)
    // ping-pong round graph: the last k_hs_fused block ends the round (statistics,
    // termination, dedup compaction) instead of a separate round-tail kernel
    int round_end;
    DevRoundStats* rstats;
    int* eq_order;
    int64_t s_cap;
    int force_exact;       // every guard fails: the Exact policy everywhere (parity tests)
    // constant entries of J (polynomials without variables: [c, c] for every box): with jc
    // set, k_hs_eval does not store them and k_hs_lin_tps takes c instead of loading
    const double* jc;      // [n^2] values (null: every entry through the scratch)
    unsigned long long jm[4];  // bit q: entry q constant
};

// bit q of the constant-J mask, words held in registers (q may be a runtime index)
struct JMask {
    unsigned long long w0, w1, w2, w3;
    __device__ __forceinline__ explicit JMask(const HsParams& p)
        : w0(p.jc ? p.jm[0] : 0), w1(p.jc ? p.jm[1] : 0), w2(p.jc ? p.jm[2] : 0), w3(p.jc ? p.jm[3] : 0) {}
    __device__ __forceinline__ bool operator()(int q) const {
        const unsigned long long w = q < 64 ? w0 : (q < 128 ? w1 : (q < 192 ? w2 : w3));
        return (w >> (q & 63)) & 1ull;
    }
};

struct HsScratch {         // SoA with stride B (batch capacity)
    double* x;             // [n][B] midpoints
    double* jl;            // [n*n][B] J(X), then M = A J
    double* jh;
    double* fl;            // [n][B] F(x), then g = A F(x)
    double* fh;
    uint8_t* flags;        // [B] bit0: exact J/F, bit1: exact M/g, bit2: singular
    int64_t B;
};

enum { HS_EMPTY = 0, HS_ONE = 1, HS_TWO = 2, HS_SKIP = 3 };
enum { HSF_EXACT_EVAL = 1, HSF_EXACT_LIN = 2, HSF_SINGULAR = 4 };

// number of HS boxes this launch may process; also decides the HS trigger
__device__ __forceinline__ int64_t hs_count(const HsParams& prm, const Counters* ctr, int64_t n_in_arg,
                                            int64_t s_cap, bool& hs_on) {
    int64_t n_in = n_in_arg;
    if (prm.count_from_ctr) {
        const unsigned long long ns = ctr->n_surv;
        if (ns > (unsigned long long)s_cap) {  // overflowed: the host grows S and redoes the round
            hs_on = false;
            return -1;
        }
        n_in = (int64_t)ns;
    }
    if (prm.hs_mode == 1) hs_on = true;
    else if (prm.hs_mode == 2) hs_on = false;
    else {  // bnb.py:289-296 on the max width of the filter survivors
        const double cw = __longlong_as_double((long long)ctr->child_wmax);
        const int round_no = prm.st ? prm.st->round_no : prm.round_no;
        hs_on = false;
        if (n_in > 0 && prm.hs_possible) {
            if (prm.hs_enable_round >= 0 && round_no >= prm.hs_enable_round) hs_on = true;
            if (!isnan(prm.hs_enable_width) && cw <= prm.hs_enable_width) hs_on = true;
        }
    }
    return n_in;
}

// HS off for this round: survivors join the frontier uncertified (bnb.py:580-581)
template <int N>
__device__ void hs_passthrough(const SBuf& S, int64_t n_in, const Front& out, Counters* ctr, int64_t* tags,
                               const DedupCtx& dd = DedupCtx{}) {
    const int lane = threadIdx.x & 31;
    // pass-through: survivors join the frontier uncertified
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x < n_in;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool valid = i < n_in;
        double w = 0.0;
        const unsigned long long slot = warp_append(valid, &ctr->n_next);
        if (valid) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                const double lo = S.lo[j * S.cap + i], hi = S.hi[j * S.cap + i];
                const double d = __dsub_rn(hi, lo);
                w = j == 0 ? d : (d > w ? d : w);
                if (slot < (unsigned long long)out.cap) {
                    out.lo[j * out.cap + slot] = lo;
                    out.hi[j * out.cap + slot] = hi;
                }
            }
            if (slot < (unsigned long long)out.cap) {
                out.cert[slot] = 0;
                out.unsplit[slot] = 0;
                if (tags) tags[slot] = 2 * i;
                if (dd.table || dd.etable) {
                    double lo[N], hi[N];
#pragma unroll
                    for (int j = 0; j < N; j++) lo[j] = S.lo[j * S.cap + i], hi[j] = S.hi[j * S.cap + i];
                    dedup_insert_regs<N>(out, (int64_t)slot, lo, hi, 0, 0, dd, ctr);
                }
            }
        }
        unsigned long long wb = valid ? (unsigned long long)__double_as_longlong(w) : 0ull;
        wb = warp_max(wb);
        if (lane == 0 && wb) atomicMax(&ctr->wmax, wb);
    }
}

// K2a: thread per box.  Rows [b0, b0 + B) of S.  When HS is off for this round the
// first batch launch copies S into F_next instead (bnb.py:580-581).
#ifndef RB_EVAL_PREFETCH
#define RB_EVAL_PREFETCH 1
#endif
#ifndef RB_EVAL_MINB
#define RB_EVAL_MINB 1  // k_hs_eval min blocks per SM (register cap)
#endif
template <int N, class EV = TabEval>
__global__ void __launch_bounds__(128, RB_EVAL_MINB) k_hs_eval(TabMeta meta, const uint8_t* __restrict__ gtab, SBuf S,
                                                 int64_t n_in_arg, int64_t b0, HsParams prm, HsScratch W,
                                                 Front out, Counters* ctr, int64_t* tags, int R) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t smem[];
    bool hs_on;
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S.cap, hs_on);
    if (n_in < 0 || n_in <= prm.fused_max) return;  // small counts: k_hs_fused
    if (blockIdx.x == 0 && threadIdx.x == 0 && b0 == 0) ctr->hs_on = hs_on ? 1ull : 0ull;
    const int lane = threadIdx.x & 31;
    if (!hs_on) {
        if (b0 == 0) hs_passthrough<N>(S, n_in, out, ctr, tags);
        return;
    }
    const int64_t b_end = min(n_in, b0 + W.B);
    if (b0 >= b_end) return;
    STab tab{};
    if constexpr (EV::tables) tab = load_stab(meta, gtab, smem, false);
    double* xs = reinterpret_cast<double*>(smem + stab_bytes(meta, false));
    const int stride = blockDim.x;
    double* xlo = xs + threadIdx.x;
    double* xhi = xs + N * stride + threadIdx.x;
    double* xmid = xs + 2 * N * stride + threadIdx.x;
    __syncthreads();
    // work item = (poly group r, box t): the n^2 + n polynomials of a box are split
    // into R groups so small batches still fill the GPU (R = 1 for large batches)
    constexpr int P = N * N + N;
    const int64_t nb = b_end - b0;
    const int64_t items = nb * R;
    unsigned long long exact_acc = 0;
    // stage box b (components at xlo / xhi / xmid [j * stride]); guards of J(X) and F(x)
    auto stage_regs = [&](const double (&blo)[N], const double (&bhi)[N], int64_t t, bool write_x, bool& fastJ,
                          bool& fastF) {
        ExpRange rx, rm;
        rx.init();
        rm.init();
#pragma unroll
        for (int j = 0; j < N; j++) {
            const double lo = blo[j], hi = bhi[j];
            const double m = mid_of(lo, hi);  // Box.midpoint, poly.py:114-115
            xlo[j * stride] = lo;
            xhi[j * stride] = hi;
            xmid[j * stride] = m;
            if (write_x) W.x[j * W.B + t] = m;
            rx.add(lo);
            rx.add(hi);
            rm.add(m);
        }
        fastJ = poly_guard_ok(meta.j_ecmin, meta.j_ecmax, meta.j_deg, rx);
        fastF = poly_guard_ok(meta.f_ecmin, meta.f_ecmax, meta.f_deg, rm);
    };
    auto stage = [&](int64_t b, int64_t t, bool write_x, bool& fastJ, bool& fastF) {
        double blo[N], bhi[N];
#pragma unroll
        for (int j = 0; j < N; j++) blo[j] = S.lo[j * S.cap + b], bhi[j] = S.hi[j * S.cap + b];
        stage_regs(blo, bhi, t, write_x, fastJ, fastF);
    };
    // the next box's rows are loaded while this one is evaluated (the loads' latency was
    // the kernel's main stall: long scoreboard ~10 per issue at 12 % occupancy)
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    double nlo[N], nhi[N];
    auto fetch = [&](int64_t it2) {
        if (it2 < items) {
            const int64_t b2 = b0 + it2 % nb;
#pragma unroll
            for (int j = 0; j < N; j++) nlo[j] = S.lo[j * S.cap + b2], nhi[j] = S.hi[j * S.cap + b2];
        }
    };
    if (RB_EVAL_PREFETCH) fetch((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    bool deferred = false;
    // constant J entries are not stored when k_hs_lin_tps takes them from prm.jc (the
    // specialised evaluator skips exactly the entries the engine's mask holds)
    const JMask jskip(prm);
    const bool skipc = prm.jc != nullptr;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items; it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = it % nb;
        const int r = (int)(it / nb);
        const int64_t b = b0 + t;
        bool fastJ, fastF;
        if (RB_EVAL_PREFETCH) {
            double blo[N], bhi[N];
#pragma unroll
            for (int j = 0; j < N; j++) blo[j] = nlo[j], bhi[j] = nhi[j];
            fetch(it + gs);
            stage_regs(blo, bhi, t, r == 0, fastJ, fastF);
        } else {
            stage(b, t, r == 0, fastJ, fastF);
        }
        if constexpr (EV::whole_box) {  // specialised evaluator: all of J(X) and F(x) by this thread (R = 1)
            // a box needing the Exact policy is evaluated after the loop: no out-of-line call
            // in the hot loop (its calling convention spilled the loop state to the stack)
            if (fastJ && fastF) {
                EV::template J<Fast>(xlo, xhi, stride, W.jl + t, W.jh + t, W.B, skipc);
                EV::template F<Fast>(xmid, xmid, stride, W.fl + t, W.fh + t, W.B);
            } else {
                deferred = true;
            }
        }
        const int p0 = EV::whole_box ? P : (int)((int64_t)r * P / R), p1 = (int)((int64_t)(r + 1) * P / R);
#pragma unroll 1
        for (int q = p0; q < p1; q++) {
            if (q < N * N) {
                if (jskip(q)) continue;  // constant entry: k_hs_lin_tps takes it from prm.jc
                // J(X) (hansen.py:61-63); zero polynomials evaluate to [0,0]
                const ival v = fastJ ? eval_poly<Fast>(tab, N + q, xlo, xhi, stride)
                                     : eval_poly_exact(tab, N + q, xlo, xhi, stride);
                W.jl[q * W.B + t] = v.lo;
                W.jh[q * W.B + t] = v.hi;
            } else {
                // F(x) = eval_point (poly.py:205-207): interval arithmetic on the point box
                const int i = q - N * N;
                const ival v = fastF ? eval_poly<Fast>(tab, i, xmid, xmid, stride)
                                     : eval_poly_exact(tab, i, xmid, xmid, stride);
                W.fl[i * W.B + t] = v.lo;
                W.fh[i * W.B + t] = v.hi;
            }
        }
        if (r == 0) {
            const bool ex = !(fastJ && fastF);
            W.flags[t] = ex ? HSF_EXACT_EVAL : 0;
            exact_acc += ex;
        }
    }
    if constexpr (EV::whole_box) {
        if (__syncthreads_or(deferred)) {  // rare: this block's Exact-policy boxes (R = 1: t = it)
            for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += (int64_t)gridDim.x * blockDim.x) {
                if (!(W.flags[t] & HSF_EXACT_EVAL)) continue;
                bool fastJ, fastF;
                stage(b0 + t, t, false, fastJ, fastF);
                if (fastJ) EV::template J<Fast>(xlo, xhi, stride, W.jl + t, W.jh + t, W.B, skipc);
                else EV::template J<Exact>(xlo, xhi, stride, W.jl + t, W.jh + t, W.B, skipc);
                if (fastF) EV::template F<Fast>(xmid, xmid, stride, W.fl + t, W.fh + t, W.B);
                else EV::template F<Exact>(xmid, xmid, stride, W.fl + t, W.fh + t, W.B);
            }
        }
    }
    exact_acc = warp_sum(exact_acc);
    if (lane == 0 && exact_acc) atomicAdd(&ctr->exact_boxes, exact_acc);
}

template <int G>
__device__ __forceinline__ double gshfl(unsigned mask, double v, int src) {
    return __shfl_sync(mask, v, src, G);
}
template <int G>
__device__ __forceinline__ int gshfl(unsigned mask, int v, int src) {
    return __shfl_sync(mask, v, src, G);
}

#ifndef RB_REDUX
#define RB_REDUX 1
#endif
template <int G>
__device__ __forceinline__ void group_reduce(unsigned mask, ExpRange& r) {
#if RB_REDUX
    // one redux.sync per bound (the group's lanes are exactly the mask's)
    r.emin = __reduce_min_sync(mask, r.emin);
    r.emax = __reduce_max_sync(mask, r.emax);
#else
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        r.emin = min(r.emin, __shfl_xor_sync(mask, r.emin, o, G));
        r.emax = max(r.emax, __shfl_xor_sync(mask, r.emax, o, G));
    }
#endif
}

template <int G>
__device__ __forceinline__ double group_max(unsigned mask, double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(mask, v, o, G);
        v = w > v ? w : v;
    }
    return v;
}

template <int N>
struct LinLayout {
    static constexpr int G = N <= 2 ? 4 : (N <= 4 ? 8 : (N <= 8 ? 16 : 32));
    static constexpr int BPW = 32 / G;
    static constexpr int oA = 0;           // A[N*N]
    static constexpr int oCol = N * N;     // pivot column[N] + pivot row
    static constexpr int doubles = N * N + N + 1;
};

// [a,a] * [l,h] as min/max of both directed products (no sign selects): for a >= 0
// the minimum is RD(a l), for a < 0 it is RD(a h) -- the 4-product min/max of
// interval.py:322-326 for a point left operand.
__device__ __forceinline__ ival pmul_minmax(double a, ival y) {
    return mk(py_min(__dmul_rd(a, y.lo), __dmul_rd(a, y.hi)), py_max(__dmul_ru(a, y.lo), __dmul_ru(a, y.hi)));
}
// The same two products chosen by a's sign bit (integer pipe: no FP64 compare, half
// the DMULs of pmul_minmax).  a = -0.0 takes the a < 0 operands: both products are
// then zeros, equal in value to pmul_minmax's (zero signs are canonicalised on output).
__device__ __forceinline__ ival pmul_sign(double a, ival y) {
    const bool neg = __double_as_longlong(a) < 0;
    const double p = neg ? y.hi : y.lo, q = neg ? y.lo : y.hi;
    return mk(__dmul_rd(a, p), __dmul_ru(a, q));
}
// Measured (bench other_configs, full solves): sign-bit products cut banded12's HS time
// 6.29 -> 5.84 ms (N = 12, 32 lanes per box) but cost katsura6 (N = 7) 3%.
#ifndef RB_PMUL_SIGN_MIN_N
#define RB_PMUL_SIGN_MIN_N 9  // sign-bit point products from this n up (A/B: tools/hs_bench.py)
#endif
// The thread-per-box products (lin_products_acc: k_hs_lin_tps / tpb, n <= 8) take the
// sign-bit form at every n (brown8 HS 23.8 -> 21.9 ms, katsura6 10.6 -> 10.3 ms); an L1
// prefetch of the next J column there measured slower (brown8 HS 24.4 ms).
template <class A>
__device__ __forceinline__ ival pmul_tpb(double a, ival y) {
    if constexpr (A::exact) return A::mul_point(a, y);
    else return pmul_sign(a, y);
}
template <class A, int N>
__device__ __forceinline__ ival pmul(double a, ival y) {
    if constexpr (A::exact) return A::mul_point(a, y);
    else if constexpr (N >= RB_PMUL_SIGN_MIN_N) return pmul_sign(a, y);
    else return pmul_minmax(a, y);
}

// Where one box's HS operands live: J / M at jl, jh[(i*N + j) * ws], F(x) / g at
// fl, fh[i * ws] -- the HBM scratch (ws = batch stride) or a shared-memory tile (ws = 1).
struct LinSink {
    double* jl;
    double* jh;
    double* fl;
    double* fh;
    int64_t ws;
};

// M = A J and g = A F(x) (linalg.py:102-129): acc = [0,0]; acc += [a,a] * B[u][j], u ascending.
// Lane (col, half) holds J[:, col] in registers and produces rows of its half.
template <int N, class A>
__device__ __forceinline__ void lin_products(const double* Am, const ival* jcol, int l, const LinSink& K,
                                             unsigned gmask) {
    constexpr int H = (N + 1) / 2;
    if (l < 2 * N) {
        const int col = l % N, half = l / N;
#pragma unroll
        for (int r = 0; r < H; r++) {
            const int i = half * H + r;
            if (i < N) {
                ival acc = mk(0.0, 0.0);
#pragma unroll
                for (int u = 0; u < N; u++) acc = A::add(acc, pmul<A, N>(Am[i * N + u], jcol[u]));
                K.jl[(i * N + col) * K.ws] = acc.lo;
                K.jh[(i * N + col) * K.ws] = acc.hi;
            }
        }
    }
    ival acc = mk(0.0, 0.0);
    if (l < N) {
#pragma unroll
        for (int u = 0; u < N; u++) acc = A::add(acc, pmul<A, N>(Am[l * N + u], mk(K.fl[u * K.ws], K.fh[u * K.ws])));
    }
    __syncwarp(gmask);  // every lane has read F(x) before g overwrites it
    if (l < N) {
        K.fl[l * K.ws] = acc.lo;
        K.fh[l * K.ws] = acc.hi;
    }
}

template <int N>
static __device__ __noinline__ void lin_products_exact(const double* Am, const ival* jcol, int l, const LinSink& K,
                                                unsigned gmask) {
    lin_products<N, Exact>(Am, jcol, l, K, gmask);
}

// K2b on one box by the G lanes of a group: mid(J), Gauss-Jordan inverse A (lane =
// column of [mid J | I], registers; pivot column broadcast through sCol), then
// M = A J and g = A F(x) over J / F(x) in place.  Returns true when singular.
template <int N, int G>
__device__ __forceinline__ bool lin_group(const LinSink& K, double* Am, double* sCol, int l, unsigned gmask,
                                          bool& exact_lin, bool force, unsigned long long* pr = nullptr) {
    // J column (l % N), kept in registers for M
    ival jcol[N];
    double c[N];
    double colmax = 0.0;
    ExpRange rj;
    rj.init();
    if (l < 2 * N) {
        const int col = l % N;
#pragma unroll
        for (int i = 0; i < N; i++) {
            jcol[i] = mk(K.jl[(i * N + col) * K.ws], K.jh[(i * N + col) * K.ws]);
            rj.add(jcol[i].lo);
            rj.add(jcol[i].hi);
        }
    }
    if (l < N) {
#pragma unroll
        for (int i = 0; i < N; i++) {
            c[i] = mid_of(jcol[i].lo, jcol[i].hi);  // mid_matrix, linalg.py:132-134
            colmax = fmax(colmax, fabs(c[i]));
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; i++) c[i] = (l - N == i) ? 1.0 : 0.0;
    }
    if (pr) pr[0] = clock64() + (unsigned long long)(c[0] + colmax) * 0ull;
    // Gauss-Jordan inverse (linalg.py:137-172), lane = column of [jc | I]
    const double scale = group_max<G>(gmask, l < N ? colmax : 0.0);
    if (pr) pr[1] = clock64() + (unsigned long long)scale * 0ull;
    bool singular = scale == 0.0;
    const double threshold = __dmul_rn(1e-12, scale);
#ifndef RB_GJ_SHFL_MAX_N
#define RB_GJ_SHFL_MAX_N 8  // pivot column broadcast by shuffles up to this n, through shared memory above
#endif
    if constexpr (N <= RB_GJ_SHFL_MAX_N) {
        // column k broadcast by shuffles; every lane repeats the pivot search on it
#pragma unroll
        for (int k = 0; k < N; k++) {
            if (singular) break;  // group-uniform
            double col[N];
#pragma unroll
            for (int i = 0; i < N; i++) col[i] = gshfl<G>(gmask, c[i], k);
            int pr = k;  // first row r >= k with max |c[r][k]|
            double best = fabs(col[k]), pivot = col[k];
#pragma unroll
            for (int r = k + 1; r < N; r++)
                if (fabs(col[r]) > best) {
                    best = fabs(col[r]);
                    pr = r;
                    pivot = col[r];
                }
            if (fabs(pivot) < threshold) {
                singular = true;
            } else {
#pragma unroll
                for (int r = k + 1; r < N; r++)
                    if (r == pr) {
                        const double tmp = c[k];
                        c[k] = c[r];
                        c[r] = tmp;
                    }
                const double inv = __drcp_rn(pivot);  // RN(1/pivot) == 1.0 / pivot (linalg.py:160)
                if (l >= k && l < 2 * N) {
                    c[k] = __dmul_rn(c[k], inv);
#pragma unroll
                    for (int i = 0; i < N; i++) {
                        if (i == k) continue;
                        const double f = i == pr ? col[k] : col[i];  // column k after the row swap
                        c[i] = __dsub_rn(c[i], __dmul_rn(f, c[k]));
                    }
                }
            }
        }
    } else {
    #pragma unroll
        for (int k = 0; k < N; k++) {
            if (singular) break;  // group-uniform
            if (l == k) {
                int pr = k;  // first row r >= k with max |c[r][k]|
                double best = fabs(c[k]);
    #pragma unroll
                for (int r = k + 1; r < N; r++)
                    if (fabs(c[r]) > best) {
                        best = fabs(c[r]);
                        pr = r;
                    }
    #pragma unroll
                for (int i = 0; i < N; i++) sCol[i] = c[i];
                sCol[N] = (double)pr;
            }
            __syncwarp(gmask);
            const int pr = (int)sCol[N];
            const double pivot = sCol[pr];
            if (fabs(pivot) < threshold) {
                singular = true;
            } else {
    #pragma unroll
                for (int r = k + 1; r < N; r++)
                    if (r == pr) {
                        const double tmp = c[k];
                        c[k] = c[r];
                        c[r] = tmp;
                    }
                const double inv = __drcp_rn(pivot);  // RN(1/pivot) == 1.0 / pivot (linalg.py:160)
                if (l >= k && l < 2 * N) {
                    c[k] = __dmul_rn(c[k], inv);
    #pragma unroll
                    for (int i = 0; i < N; i++) {
                        if (i == k) continue;
                        const double f = sCol[i == pr ? k : i];  // column k after the row swap
                        // the reference skips f == 0 (linalg.py:168); c - 0*c[k] == c for the finite
                        // values here (only a zero's sign could differ), so no test is needed
                        c[i] = __dsub_rn(c[i], __dmul_rn(f, c[k]));
                    }
                }
            }
            __syncwarp(gmask);
        }
    }
    if (pr) pr[2] = clock64() + (unsigned long long)c[N - 1] * 0ull;
    exact_lin = false;
    if (singular) return true;
    ExpRange ra, rf;
    ra.init();
    rf.init();
    if (l >= N && l < 2 * N) {
#pragma unroll
        for (int i = 0; i < N; i++) {
            Am[i * N + (l - N)] = c[i];
            ra.add(c[i]);
        }
    }
    if (l < N) {
        rf.add(K.fl[l * K.ws]);
        rf.add(K.fh[l * K.ws]);
    }
    group_reduce<G>(gmask, ra);
    group_reduce<G>(gmask, rj);
    group_reduce<G>(gmask, rf);
    rj.emin = min(rj.emin, rf.emin);
    rj.emax = max(rj.emax, rf.emax);
    const bool fastM = !force && prod_guard_ok(ra, rj);
    if (pr) pr[3] = clock64() + (unsigned long long)fastM * 0ull;
    __syncwarp(gmask);
    if (fastM) lin_products<N, Fast>(Am, jcol, l, K, gmask);
    else lin_products_exact<N>(Am, jcol, l, K, gmask);
    exact_lin = !fastM;
    return false;
}

// K2b: G lanes per box; boxes assigned warp-uniformly.
template <int N>
#ifndef RB_LIN_MINB
#define RB_LIN_MINB 1  // __launch_bounds__ min blocks per SM of k_hs_lin (register cap)
#endif
__global__ void __launch_bounds__(128, RB_LIN_MINB) k_hs_lin(SBuf S, int64_t n_in_arg, int64_t b0, HsParams prm, HsScratch W,
                                                Counters* ctr) {
    pdl_enter();
    using L = LinLayout<N>;
    constexpr int G = L::G;
    extern __shared__ __align__(16) uint8_t smem[];
    bool hs_on;
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S.cap, hs_on);
    if (n_in < 0 || !hs_on || n_in <= prm.fused_max) return;
    const int64_t b_end = min(n_in, b0 + W.B);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane / G, l = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gi * G));
    double* s = reinterpret_cast<double*>(smem) + (size_t)(warp * L::BPW + gi) * L::doubles;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t wglob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    for (int64_t wb0 = b0 + wglob * L::BPW; wb0 < b_end; wb0 += warps_total * L::BPW) {
        const int64_t b = wb0 + gi;
        if (b < b_end) {
            const int64_t t = b - b0;
            const LinSink K{W.jl + t, W.jh + t, W.fl + t, W.fh + t, W.B};
            bool exact_lin;
            const bool singular = lin_group<N, G>(K, s + L::oA, s + L::oCol, l, gmask, exact_lin, prm.force_exact);
            if (l == 0) W.flags[t] |= singular ? HSF_SINGULAR : (exact_lin ? HSF_EXACT_LIN : 0);
            __syncwarp(gmask);
        }
        __syncwarp();
    }
}

// K2b, thread per box (n <= 8): the Gauss-Jordan inverse of lin_group with the same
// operations in the same order, run by one thread in registers -- with G lanes per
// box (k_hs_lin) every group re-executes the pivot search, row-swap selects and
// pivot-column shuffles on all of its lanes (ncu, katsura6 round 5: ~1,080 warp
// instructions per box for k_hs_lin<7>); here they are one thread's scalar work, and
// the J / F(x) scratch is read and M / g written with coalesced thread-per-box
// accesses.  The tableau is kept in place (n x n instead of [mid J | I], n x 2n):
//   slot s < k holds the column of the right half that became non-trivial at step s
//   (label e_s = original row of the step-s pivot row), slot s >= k the left column s.
// Every non-trivial operation of linalg.py:137-172 is performed with the same operands;
// the skipped ones act on exact zeros / ones of the identity half (x - f*0 = x,
// 1 * inv = inv, 0 - f*inv = -(f*inv)), so the inverse is bit-identical (zero signs
// aside, which no later operation can observe).  Row swaps are predicated selects.
#ifndef RB_LIN_COLS
#define RB_LIN_COLS 2  // lin_products_acc: columns of J per pass
#endif
struct JLoad {  // J entry q of box t from the scratch
    const HsScratch& W;
    int64_t t;
    __device__ __forceinline__ ival operator()(int q) const { return mk(W.jl[q * W.B + t], W.jh[q * W.B + t]); }
};
template <int N, class A, class AM, int IU = N, class JG = JLoad>
__device__ __forceinline__ void lin_products_acc(const AM& am, HsScratch& W, int64_t t, const JG* jg = nullptr);

template <int N, class A>
__device__ __forceinline__ void lin_products_reg(const double (&a)[N][N], HsScratch& W, int64_t t) {
    lin_products_acc<N, A>([&](int i, int u) { return a[i][u]; }, W, t);
}

// M = A J and g = A F(x) with A given by an accessor am(i, u); IU = unrolling of the row
// loop (N for A in registers; small for A in shared memory, bounding the loads in flight)
template <int N, class A, class AM, int IU, class JG>
__device__ __forceinline__ void lin_products_acc(const AM& am, HsScratch& W, int64_t t, const JG* jg) {
    // M = A J (linalg.py:102-114) and g = A F(x) (linalg.py:117-129), u ascending: the n
    // columns of J and F(x) as n + 1 columns v, RB_LIN_COLS of them per pass so each A
    // element read serves several columns; column v of M is written over column v of J
    constexpr int CP = RB_LIN_COLS;
    auto ld = [&](int v, int u) -> ival {
        if (v == N) return mk(W.fl[u * W.B + t], W.fh[u * W.B + t]);
        return jg ? (*jg)(u * N + v) : mk(W.jl[(u * N + v) * W.B + t], W.jh[(u * N + v) * W.B + t]);
    };
    auto st = [&](int v, int i, const ival& r) {
        if (v == N) {
            W.fl[i * W.B + t] = r.lo;
            W.fh[i * W.B + t] = r.hi;
        } else {
            W.jl[(i * N + v) * W.B + t] = r.lo;
            W.jh[(i * N + v) * W.B + t] = r.hi;
        }
    };
#pragma unroll 1
    for (int v0 = 0; v0 <= N; v0 += CP) {
        ival jc[CP][N];
#pragma unroll
        for (int c = 0; c < CP; c++)
#pragma unroll
            for (int u = 0; u < N; u++) jc[c][u] = v0 + c <= N ? ld(v0 + c, u) : mk(0.0, 0.0);
#pragma unroll IU
        for (int i = 0; i < N; i++) {
            ival acc[CP];
#pragma unroll
            for (int c = 0; c < CP; c++) acc[c] = mk(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < N; u++) {
                const double a = am(i, u);
#pragma unroll
                for (int c = 0; c < CP; c++) acc[c] = A::add(acc[c], pmul_tpb<A>(a, jc[c][u]));
            }
#pragma unroll
            for (int c = 0; c < CP; c++)
                if (v0 + c <= N) st(v0 + c, i, acc[c]);
        }
    }
}

template <int N>
static __device__ __noinline__ void lin_products_reg_exact(const double (&a)[N][N], HsScratch& W, int64_t t) {
    lin_products_reg<N, Exact>(a, W, t);
}

#ifndef RB_LIN_REG_MINB
#define RB_LIN_REG_MINB 2
#endif
template <int N>
__global__ void __launch_bounds__(128, RB_LIN_REG_MINB) k_hs_lin_tpb(SBuf S, int64_t n_in_arg, int64_t b0,
                                                                     HsParams prm, HsScratch W, Counters* ctr) {
    pdl_enter();
    static_assert(N <= 8, "k_hs_lin_tpb: one thread holds a box's n x n Gauss-Jordan tableau in registers");
    bool hs_on;
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S.cap, hs_on);
    if (n_in < 0 || !hs_on || n_in <= prm.fused_max) return;
    const int64_t b_end = min(n_in, b0 + W.B);
    for (int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < b_end;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = b - b0;
        // mid(J) (mid_matrix, linalg.py:132-134) with the exponent range of J
        ExpRange rj, ra, rf;
        rj.init();
        ra.init();
        rf.init();
        double c[N][N];
        double scale = 0.0;
#pragma unroll
        for (int i = 0; i < N; i++)
#pragma unroll
            for (int j = 0; j < N; j++) {
                const double lo = W.jl[(i * N + j) * W.B + t], hi = W.jh[(i * N + j) * W.B + t];
                rj.add(lo);
                rj.add(hi);
                c[i][j] = mid_of(lo, hi);
                scale = fmax(scale, fabs(c[i][j]));
            }
        // Gauss-Jordan (linalg.py:137-172): threshold 1e-12 scale, first-max pivot,
        // inv = RN(1/pivot), pivot row scaled, other rows eliminated, no FMA
        bool singular = scale == 0.0;
        const double threshold = __dmul_rn(1e-12, scale);
        uint32_t orig = 0, label = 0;  // 4-bit fields: original row at each position; e_s per slot
#pragma unroll
        for (int r = 0; r < N; r++) orig |= (uint32_t)r << (4 * r);
#pragma unroll
        for (int k = 0; k < N; k++) {
            // no early exit (a break would keep the compiler from unrolling the steps, and
            // with them every register index of c): a singular tableau skips its steps
            int pr = k;
            double best = fabs(c[k][k]), pv = c[k][k];
#pragma unroll
            for (int r = k + 1; r < N; r++)
                if (fabs(c[r][k]) > best) {
                    best = fabs(c[r][k]);
                    pv = c[r][k];
                    pr = r;
                }
            singular = singular || fabs(pv) < threshold;
            if (!singular) {
                // swap rows k and pr (every slot: left columns >= k and the stored right columns)
#pragma unroll
                for (int r = k + 1; r < N; r++)
                    if (r == pr) {
#pragma unroll
                        for (int s2 = 0; s2 < N; s2++) {
                            const double tmp = c[k][s2];
                            c[k][s2] = c[r][s2];
                            c[r][s2] = tmp;
                        }
                    }
                const uint32_t ok = (orig >> (4 * k)) & 15u, op = (orig >> (4 * pr)) & 15u;
                orig = (orig & ~((15u << (4 * k)) | (15u << (4 * pr)))) | (op << (4 * k)) | (ok << (4 * pr));
                label |= op << (4 * k);  // e_k: original row of the pivot row
                const double inv = __drcp_rn(pv);  // RN(1/pivot) == 1.0 / pivot (linalg.py:162)
                // c[k][j] *= inv (linalg.py:163-164): left j > k and the stored right columns;
                // the right column e_k becomes 1 * inv = inv (slot k; left column k is dead)
#pragma unroll
                for (int s2 = 0; s2 < N; s2++) c[k][s2] = s2 == k ? inv : __dmul_rn(c[k][s2], inv);
#pragma unroll
                for (int i = 0; i < N; i++) {
                    if (i == k) continue;
                    const double f = c[i][k];
                    if (f != 0.0) {  // linalg.py:168
#pragma unroll
                        for (int s2 = 0; s2 < N; s2++)
                            c[i][s2] = s2 == k ? __dsub_rn(0.0, __dmul_rn(f, inv))  // 0 - f * inv
                                               : __dsub_rn(c[i][s2], __dmul_rn(f, c[k][s2]));
                    }
                }
            }
        }
        uint8_t fl = 0;
        if (singular) {
            fl = HSF_SINGULAR;
        } else {
            // unscramble in place, row by row: A[i][e_s] = slot s (predicated selects)
            double (&a)[N][N] = c;
#pragma unroll
            for (int i = 0; i < N; i++) {
                double row[N];
#pragma unroll
                for (int u = 0; u < N; u++) {
                    row[u] = c[i][0];
#pragma unroll
                    for (int s2 = 1; s2 < N; s2++)
                        if (((label >> (4 * s2)) & 15u) == (uint32_t)u) row[u] = c[i][s2];
                }
#pragma unroll
                for (int u = 0; u < N; u++) c[i][u] = row[u];
            }
#pragma unroll
            for (int i = 0; i < N; i++)
#pragma unroll
                for (int u = 0; u < N; u++) ra.add(a[i][u]);
#pragma unroll
            for (int u = 0; u < N; u++) {
                rf.add(W.fl[u * W.B + t]);
                rf.add(W.fh[u * W.B + t]);
            }
            rj.emin = min(rj.emin, rf.emin);
            rj.emax = max(rj.emax, rf.emax);
            if (!prm.force_exact && prod_guard_ok(ra, rj)) {
                lin_products_reg<N, Fast>(a, W, t);
            } else {  // rare: the Exact policy on a memory copy (keeps `a` itself in registers)
                double ax[N][N];
#pragma unroll
                for (int i = 0; i < N; i++)
#pragma unroll
                    for (int u = 0; u < N; u++) ax[i][u] = a[i][u];
                lin_products_reg_exact<N>(ax, W, t);
                fl = HSF_EXACT_LIN;
            }
        }
        W.flags[t] |= fl;
    }
}

__device__ __forceinline__ double lds_volatile(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}

template <bool B, class T, class F>
struct pick_t {
    using type = T;
};
template <class T, class F>
struct pick_t<false, T, F> {
    using type = F;
};
#ifndef RB_TPS_MINB7
#define RB_TPS_MINB7 4
#endif
#ifndef RB_TPS_MINB12
#define RB_TPS_MINB12 3
#endif
#ifndef RB_TPS_MINB8
#define RB_TPS_MINB8 3
#endif
// k_hs_lin_tps shape: n^2 doubles of shared memory per thread; 128 threads per block up to
// n = 8, 64 above (n = 12: 72 KB per block, 3 blocks per SM)
template <int N>
struct TpsShape {
    static constexpr int T = N <= 8 ? 128 : 64;
    static constexpr int MINB = N <= 7 ? RB_TPS_MINB7 : (N <= 8 ? RB_TPS_MINB8 : RB_TPS_MINB12);
    using Lbl = typename pick_t<(N > 8), unsigned long long, uint32_t>::type;
};
// J entry q: the constant [c, c] where the mask says so, else the scratch
struct JConst {
    const HsScratch& W;
    int64_t t;
    JMask jm;
    const double* jc;
    __device__ __forceinline__ ival operator()(int q) const {
        if (jm(q)) {
            const double c = jc[q];
            return mk(c, c);
        }
        return mk(W.jl[q * W.B + t], W.jh[q * W.B + t]);
    }
};
template <int N>
static __device__ __noinline__ void lin_products_tps_exact(const double* C, HsScratch W, int64_t t, HsParams prm) {
    const JConst jg{W, t, JMask(prm), prm.jc};
    auto am = [&](int i, int u) { return C[(i * N + u) * TpsShape<N>::T]; };
    lin_products_acc<N, Exact, decltype(am), N, JConst>(am, W, t, &jg);
}

// k_hs_lin_tpb with the in-place tableau in shared memory (this thread's column:
// element (i, s) at C[(i * n + s) * T], conflict-free) instead of registers: n^2 doubles
// per thread, so more threads stay resident and no register limit is reached at n = 8.
// Same operations in the same order; the row swap and the unscrambling index memory.
#ifndef RB_TPS_MID_UNROLL
#define RB_TPS_MID_UNROLL 1
#endif
constexpr int kTpsMidUnroll = RB_TPS_MID_UNROLL;
#ifndef RB_TPS_ROW_UNROLL
#define RB_TPS_ROW_UNROLL 1
#endif
constexpr int kTpsRowUnroll = RB_TPS_ROW_UNROLL;
template <int N>
__global__ void __launch_bounds__(TpsShape<N>::T, TpsShape<N>::MINB) k_hs_lin_tps(SBuf S, int64_t n_in_arg, int64_t b0, HsParams prm, HsScratch W,
                                                    Counters* ctr) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t smem[];
    bool hs_on;
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S.cap, hs_on);
    if (n_in < 0 || !hs_on || n_in <= prm.fused_max) return;
    const int64_t b_end = min(n_in, b0 + W.B);
    constexpr int T = TpsShape<N>::T;  // the launch's block size: tableau offsets are immediates
    double* C = reinterpret_cast<double*>(smem) + threadIdx.x;
    auto c = [&](int i, int s2) -> double& { return C[(i * N + s2) * T]; };
    const JMask jmask(prm);
    for (int64_t b = b0 + (int64_t)blockIdx.x * T + threadIdx.x; b < b_end; b += (int64_t)gridDim.x * T) {
        const int64_t t = b - b0;
        const JConst jg{W, t, jmask, prm.jc};
        ExpRange rj, ra, rf;
        rj.init();
        ra.init();
        rf.init();
        double scale = 0.0;
#pragma unroll kTpsMidUnroll  // a row of J per step: full unrolling hoisted every load and spilled
        for (int i = 0; i < N; i++)
#pragma unroll
            for (int j = 0; j < N; j++) {
                const ival v = jg(i * N + j);
                const double lo = v.lo, hi = v.hi;
                rj.add(lo);
                rj.add(hi);
                const double m = mid_of(lo, hi);
                c(i, j) = m;
                scale = fmax(scale, fabs(m));
            }
        bool singular = scale == 0.0;
        const double threshold = __dmul_rn(1e-12, scale);
        using Lbl = typename TpsShape<N>::Lbl;  // 4-bit fields: n <= 8 in 32 bits, else 64
        Lbl orig = 0, label = 0;
#pragma unroll
        for (int r = 0; r < N; r++) orig |= (Lbl)r << (4 * r);
#pragma unroll(N <= 8 ? N : 1)  // n > 8: the unrolled steps overflowed the instruction cache
        for (int k = 0; k < N; k++) {
            int pr = k;
            double best = fabs(c(k, k)), pv = c(k, k);
#pragma unroll
            for (int r = k + 1; r < N; r++) {
                const double v = c(r, k);
                if (fabs(v) > best) {
                    best = fabs(v);
                    pv = v;
                    pr = r;
                }
            }
            singular = singular || fabs(pv) < threshold;
            if (!singular) {
                const Lbl ok = (orig >> (4 * k)) & 15u, op = (orig >> (4 * pr)) & 15u;
                orig = (orig & ~(((Lbl)15 << (4 * k)) | ((Lbl)15 << (4 * pr)))) | (op << (4 * k)) | (ok << (4 * pr));
                label |= op << (4 * k);
                const double inv = __drcp_rn(pv);  // RN(1/pivot) == 1.0 / pivot (linalg.py:162)
                double rowk[N];
#pragma unroll
                for (int s2 = 0; s2 < N; s2++) {  // swap (row pr <- old row k) and scale row k
                    const double vk = c(k, s2), vp = c(pr, s2);
                    c(pr, s2) = vk;
                    rowk[s2] = s2 == k ? inv : __dmul_rn(vp, inv);
                    c(k, s2) = rowk[s2];
                }
#pragma unroll
                for (int i = 0; i < N; i++) {
                    if (i == k) continue;
                    const double f = c(i, k);
                    if (f != 0.0) {  // linalg.py:168
#pragma unroll
                        for (int s2 = 0; s2 < N; s2++)
                            c(i, s2) = s2 == k ? __dsub_rn(0.0, __dmul_rn(f, inv))
                                               : __dsub_rn(c(i, s2), __dmul_rn(f, rowk[s2]));
                    }
                }
            }
        }
        uint8_t fl = 0;
        if (singular) {
            fl = HSF_SINGULAR;
        } else {
            // unscramble in place, row by row: slot s holds A[i][e_s] (a permutation), so the
            // products read A at fixed offsets
#pragma unroll 1
            for (int i = 0; i < N; i++) {
                double row[N];
#pragma unroll
                for (int s2 = 0; s2 < N; s2++) row[s2] = c(i, s2);
#pragma unroll
                for (int s2 = 0; s2 < N; s2++) {
                    c(i, (int)((label >> (4 * s2)) & 15u)) = row[s2];
                    ra.add(row[s2]);
                }
            }
#pragma unroll
            for (int u = 0; u < N; u++) {
                rf.add(W.fl[u * W.B + t]);
                rf.add(W.fh[u * W.B + t]);
            }
            rj.emin = min(rj.emin, rf.emin);
            rj.emax = max(rj.emax, rf.emax);
            if (!prm.force_exact && prod_guard_ok(ra, rj)) {
                auto am_tps = [&](int i, int u) { return lds_volatile(&c(i, u)); };
                // volatile shared loads: kept inside the column loop (hoisting all n^2 of A out
                // of it is what spilled)
                lin_products_acc<N, Fast, decltype(am_tps), kTpsRowUnroll, JConst>(am_tps, W, t, &jg);
            } else {  // rare: out of line, A read from the tableau (no local copy in this frame)
                lin_products_tps_exact<N>(C, W, t, prm);
                fl = HSF_EXACT_LIN;
            }
        }
        W.flags[t] |= fl;
    }
}

// k_hs_lin_tps with two threads per box (lin_tpb = 3): the pair shares the box's
// tableau in shared memory and splits its columns by parity -- each thread swaps, scales
// and eliminates its own columns (the pivot search and the bookkeeping are repeated by
// both, identically), and computes the M / g columns of its parity.  Per element the
// same operations in the same order as k_hs_lin_tps; twice the threads for the same
// shared memory per box, so more warps hide the latencies.
// measured (tools/hs_bench.py): slower than k_hs_lin_tps up to n = 8 (brown8 15.8 -> 18.4 ms
// per solve), faster above (banded12 3.89 -> 3.61 ms at 4 blocks per SM): the default for
// 8 < n <= 12
#ifndef RB_TP2_MINB
#define RB_TP2_MINB 5
#endif
#ifndef RB_TP2_MINB_WIDE
#define RB_TP2_MINB_WIDE 4
#endif
template <int N>
static __device__ __noinline__ void lin_products_pair_exact(const double* C, int S, HsScratch W, int64_t t, HsParams prm) {
    const JConst jg{W, t, JMask(prm), prm.jc};
    auto am = [&](int i, int u) { return C[(i * N + u) * S]; };
    lin_products_acc<N, Exact, decltype(am), N, JConst>(am, W, t, &jg);
}
template <int N>
__global__ void __launch_bounds__(128, (N > 8 ? RB_TP2_MINB_WIDE : RB_TP2_MINB)) k_hs_lin_tp2(SBuf S_, int64_t n_in_arg, int64_t b0, HsParams prm, HsScratch W,
                                                    Counters* ctr) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t smem[];
    bool hs_on;
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S_.cap, hs_on);
    if (n_in < 0 || !hs_on || n_in <= prm.fused_max) return;
    const int64_t b_end = min(n_in, b0 + W.B);
    constexpr int T = 128, SL = T / 2;  // 64 boxes per block, slot = tid / 2
    const int slot = threadIdx.x >> 1, h = threadIdx.x & 1;
    const unsigned pm = 3u << ((threadIdx.x & 31) & ~1);  // the pair's lanes
    double* C = reinterpret_cast<double*>(smem) + slot;
    auto c = [&](int i, int s2) -> double& { return C[(i * N + s2) * SL]; };
    const JMask jmask(prm);
    for (int64_t b = b0 + (int64_t)blockIdx.x * SL + slot; b < b_end; b += (int64_t)gridDim.x * SL) {
        const int64_t t = b - b0;
        const JConst jg{W, t, jmask, prm.jc};
        ExpRange rj, ra, rf;
        rj.init();
        ra.init();
        rf.init();
        double scale = 0.0;
        // mid(J): this thread's columns (j = h, h + 2, ...)
#pragma unroll 1
        for (int i = 0; i < N; i++)
#pragma unroll
            for (int q = 0; q < (N + 1) / 2; q++) {
                const int j = 2 * q + h;
                if (j >= N) break;
                const ival v = jg(i * N + j);
                rj.add(v.lo);
                rj.add(v.hi);
                const double m = mid_of(v.lo, v.hi);
                c(i, j) = m;
                scale = fmax(scale, fabs(m));
            }
        scale = fmax(scale, __shfl_xor_sync(pm, scale, 1));
        rj.emin = min(rj.emin, __shfl_xor_sync(pm, rj.emin, 1));
        rj.emax = max(rj.emax, __shfl_xor_sync(pm, rj.emax, 1));
        __syncwarp(pm);
        bool singular = scale == 0.0;
        const double threshold = __dmul_rn(1e-12, scale);
        using Lbl = typename TpsShape<N>::Lbl;
        Lbl orig = 0, label = 0;
#pragma unroll
        for (int r = 0; r < N; r++) orig |= (Lbl)r << (4 * r);
#pragma unroll 1
        for (int k = 0; k < N; k++) {
            int pr = k;
            double best = fabs(c(k, k)), pv = c(k, k);
#pragma unroll
            for (int r = k + 1; r < N; r++) {
                const double v = c(r, k);
                if (fabs(v) > best) {
                    best = fabs(v);
                    pv = v;
                    pr = r;
                }
            }
            singular = singular || fabs(pv) < threshold;
            if (!singular) {  // pair-uniform (same reads, same decisions)
                const Lbl ok = (orig >> (4 * k)) & 15u, op = (orig >> (4 * pr)) & 15u;
                orig = (orig & ~(((Lbl)15 << (4 * k)) | ((Lbl)15 << (4 * pr)))) | (op << (4 * k)) | (ok << (4 * pr));
                label |= op << (4 * k);
                const double inv = __drcp_rn(pv);  // RN(1/pivot) == 1.0 / pivot (linalg.py:162)
                __syncwarp(pm);  // both searched column k before anything is swapped
                double rowk[(N + 1) / 2];
#pragma unroll
                for (int q = 0; q < (N + 1) / 2; q++) {  // swap and scale row k, own columns
                    const int s2 = 2 * q + h;
                    if (s2 >= N) break;
                    const double vk = c(k, s2), vp = c(pr, s2);
                    c(pr, s2) = vk;
                    rowk[q] = s2 == k ? inv : __dmul_rn(vp, inv);
                    c(k, s2) = rowk[q];
                }
                __syncwarp(pm);  // column k swapped (by its owner)
                double fcol[N];
#pragma unroll
                for (int i = 0; i < N; i++) fcol[i] = c(i, k);
                __syncwarp(pm);  // both hold column k before its owner rewrites it
#pragma unroll
                for (int i = 0; i < N; i++) {
                    if (i == k) continue;
                    const double f = fcol[i];
                    if (f != 0.0) {  // linalg.py:168
#pragma unroll
                        for (int q = 0; q < (N + 1) / 2; q++) {
                            const int s2 = 2 * q + h;
                            if (s2 >= N) break;
                            c(i, s2) = s2 == k ? __dsub_rn(0.0, __dmul_rn(f, inv))
                                               : __dsub_rn(c(i, s2), __dmul_rn(f, rowk[q]));
                        }
                    }
                }
                __syncwarp(pm);
            }
        }
        uint8_t fl = 0;
        if (singular) {
            fl = HSF_SINGULAR;
        } else {
            // unscramble, row by row: slot s holds A[i][e_s]; a thread writes its
            // destination columns after both read the row
#pragma unroll 1
            for (int i = 0; i < N; i++) {
                double row[N];
#pragma unroll
                for (int s2 = 0; s2 < N; s2++) row[s2] = c(i, s2);
                __syncwarp(pm);
#pragma unroll
                for (int s2 = 0; s2 < N; s2++) {
                    const int u = (int)((label >> (4 * s2)) & 15u);
                    if ((u & 1) == h) c(i, u) = row[s2];
                    ra.add(row[s2]);
                }
                __syncwarp(pm);
            }
#pragma unroll
            for (int u = 0; u < N; u++) {
                rf.add(W.fl[u * W.B + t]);
                rf.add(W.fh[u * W.B + t]);
            }
            rj.emin = min(rj.emin, rf.emin);
            rj.emax = max(rj.emax, rf.emax);
            __syncwarp(pm);  // both read F(x) before its owner overwrites it with g
            if (!prm.force_exact && prod_guard_ok(ra, rj)) {
                // own columns v = h, h + 2, ... of [J | F(x)] (v = N: F(x) -> g), two per pass
#pragma unroll 1
                for (int v0 = h; v0 <= N; v0 += 4) {
                    const bool two = v0 + 2 <= N;
                    ival j0[N], j1[N];
#pragma unroll
                    for (int u = 0; u < N; u++) {
                        j0[u] = v0 == N ? mk(W.fl[u * W.B + t], W.fh[u * W.B + t]) : jg(u * N + v0);
                        j1[u] = !two ? mk(0.0, 0.0)
                                     : (v0 + 2 == N ? mk(W.fl[u * W.B + t], W.fh[u * W.B + t]) : jg(u * N + v0 + 2));
                    }
#pragma unroll 1
                    for (int i = 0; i < N; i++) {
                        ival a0 = mk(0.0, 0.0), a1 = mk(0.0, 0.0);
#pragma unroll
                        for (int u = 0; u < N; u++) {
                            const double a = lds_volatile(&c(i, u));
                            a0 = Fast::add(a0, pmul_tpb<Fast>(a, j0[u]));
                            a1 = Fast::add(a1, pmul_tpb<Fast>(a, j1[u]));
                        }
                        if (v0 == N) {
                            W.fl[i * W.B + t] = a0.lo;
                            W.fh[i * W.B + t] = a0.hi;
                        } else {
                            W.jl[(i * N + v0) * W.B + t] = a0.lo;
                            W.jh[(i * N + v0) * W.B + t] = a0.hi;
                        }
                        if (two) {
                            if (v0 + 2 == N) {
                                W.fl[i * W.B + t] = a1.lo;
                                W.fh[i * W.B + t] = a1.hi;
                            } else {
                                W.jl[(i * N + v0 + 2) * W.B + t] = a1.lo;
                                W.jh[(i * N + v0 + 2) * W.B + t] = a1.hi;
                            }
                        }
                    }
                }
            } else {  // rare: one thread, out of line
                if (h == 0) lin_products_pair_exact<N>(C, SL, W, t, prm);
                fl = HSF_EXACT_LIN;
            }
        }
        if (h == 0) W.flags[t] |= fl;
        __syncwarp(pm);  // the tableau is reused for the next box
    }
}

// K2k: the Krawczyk operator (hansen.py:141-170) on the K2a/K2b scratch (x, M, g),
// thread per box.  Row i: acc = [x_i,x_i] - g_i + sum_{j, (I - M)_ij != [0,0]}
// (I - M)_ij (X_j - [x_j,x_j]), left to right, then acc intersected with X_i.
// ok[b] = 0 for None (singular midpoint Jacobian or an empty intersection).
template <int N>
__global__ void __launch_bounds__(128) k_krawczyk(SBuf S, int64_t b_end, int64_t b0, HsScratch W, Front out,
                                                  uint8_t* ok) {
    pdl_enter();
    for (int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < b_end;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = b - b0;
        bool good = !(W.flags[t] & HSF_SINGULAR);
        double xl[N], xh[N], xv[N];
#pragma unroll
        for (int j = 0; j < N; j++) {
            xl[j] = S.lo[j * S.cap + b];
            xh[j] = S.hi[j * S.cap + b];
            xv[j] = W.x[j * W.B + t];
        }
        ival d[N];
#pragma unroll
        for (int j = 0; j < N; j++) d[j] = Fast::sub(mk(xl[j], xh[j]), mk(xv[j], xv[j]));
#pragma unroll 1
        for (int i = 0; i < N && good; i++) {
            ival acc = Fast::sub(mk(xv[i], xv[i]), mk(W.fl[i * W.B + t], W.fh[i * W.B + t]));
#pragma unroll
            for (int j = 0; j < N; j++) {
                const ival m = mk(W.jl[(i * N + j) * W.B + t], W.jh[(i * N + j) * W.B + t]);
                const double e = (i == j) ? 1.0 : 0.0;
                const ival c = Fast::sub(mk(e, e), m);
                if (c.lo == 0.0 && c.hi == 0.0) continue;
                acc = Fast::add(acc, gmul(c, d[j]));
            }
            double xi_lo = xl[0], xi_hi = xh[0];
#pragma unroll
            for (int j = 1; j < N; j++)
                if (j == i) {
                    xi_lo = xl[j];
                    xi_hi = xh[j];
                }
            const double lo = py_max(acc.lo, xi_lo), hi = py_min(acc.hi, xi_hi);  // Interval.intersect
            if (lo > hi) {
                good = false;
                break;
            }
            out.lo[i * out.cap + b] = canon0(lo);
            out.hi[i * out.cap + b] = canon0(hi);
        }
        ok[b] = good ? 1 : 0;
    }
}

// 1/y rounded down or up (up != 0) for a normal y whose reciprocal is normal: one
// round-to-nearest reciprocal r, whose FMA residual 1 - y r is exact; the residual's
// sign times y's tells on which side of 1/y r lies (the directed-rounding division
// sequences are ~3x longer on sm_100).
__device__ __forceinline__ double recip_dir(double y, bool up) {
    const double r = __drcp_rn(y);
    const double e = __fma_rn(-y, r, 1.0);
    if (e == 0.0) return r;
    const bool r_below = (e > 0.0) == (y > 0.0);  // r < 1/y
    const long long b = __double_as_longlong(r);
    // one ulp toward +inf (up, r below) or -inf (down, r above); r != 0
    if (up == r_below) return __longlong_as_double(b + (((r > 0.0) == up) ? 1 : -1));
    return r;
}

// fast reciprocal-based single case of div_extended; exact emulation elsewhere
__device__ __forceinline__ int div_extended_fast(ival p, ival y, ival& q0, ival& q1, bool force = false) {
    if (!force && !contains_zero(y)) {
        // magnitudes, not endpoints: for y < 0 the larger magnitude is |y.lo| (a y with
        // |y.lo| >= 2^990 or |y.hi| <= 2^-990 must take the reference's untrusted-band
        // division; found by tests/test_gpu_exact.py on kat_interval.npz)
        const double al = fmin(fabs(y.lo), fabs(y.hi)), ah = fmax(fabs(y.lo), fabs(y.hi));
        if (al > 0x1p-990 && ah < 0x1p990) {
            // _div_rd/_div_ru (interval.py:157-190) == IEEE directed division inside the trusted band
            const ival r = mk(recip_dir(y.hi, false), recip_dir(y.lo, true));
            q0 = gmul(p, r);
            return DIV_SINGLE;
        }
    }
    return div_extended(p, y, q0, q1, force);
}

// K2c: thread per box: the Gauss-Seidel sweep (hansen.py:91-138) and the
// _hs_pass output rules (bnb.py:197-210), compacted into `out` after the carried rows.
#ifndef RB_SWEEP_MINB
#define RB_SWEEP_MINB 4  // k_hs_sweep min blocks per SM: 120 registers at n = 8, no spills (4 vs 1: katsura6 / brown8 / eco8 solves -3 %)
#endif
template <int N>
__global__ void __launch_bounds__(128, (N <= 10 ? RB_SWEEP_MINB : 1)) k_hs_sweep(TabMeta meta, SBuf S, int64_t n_in_arg, int64_t b0, HsParams prm,
                                                  HsScratch W, Front out, Counters* ctr, int64_t* tags) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t smem[];
    bool hs_on;
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S.cap, hs_on);
    if (n_in < 0 || !hs_on || n_in <= prm.fused_max) return;
    const int64_t b_end = min(n_in, b0 + W.B);
    const int lane = threadIdx.x & 31;
    const int stride = blockDim.x;
    double* cl = reinterpret_cast<double*>(smem) + threadIdx.x;  // current[j].lo at cl[j*stride]
    double* ch = cl + N * stride;
    unsigned long long ops_acc = 0, calls_acc = 0;
    for (int64_t base = b0 + (int64_t)blockIdx.x * blockDim.x; base < b_end; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = base + threadIdx.x;
        const bool valid = b < b_end;
        const int64_t t = b - b0;
        int kind = HS_EMPTY;
        bool cert = false;
        int fork_i = -1;
        ival fp0 = mk(0.0, 0.0), fp1 = mk(0.0, 0.0);
        int rows = 0;
        if (valid) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                cl[j * stride] = S.lo[j * S.cap + b];
                ch[j * stride] = S.hi[j * S.cap + b];
            }
            if (W.flags[t] & HSF_SINGULAR) {
                kind = HS_SKIP;
            } else {
                kind = HS_ONE;
                double xv[N];
#pragma unroll
                for (int j = 0; j < N; j++) xv[j] = W.x[j * W.B + t];
#pragma unroll 1
                for (int i = 0; i < N; i++) {
                    rows = i + 1;
                    // row i of M, loaded together (independent loads, one latency)
                    ival mrow[N];
#pragma unroll
                    for (int j = 0; j < N; j++)
                        mrow[j] = mk(W.jl[(i * N + j) * W.B + t], W.jh[(i * N + j) * W.B + t]);
                    // p = -g_i - sum_{j != i, M_ij != [0,0]} M_ij (current_j - [x_j, x_j]), left to right
                    ival p = mk(-W.fh[i * W.B + t], -W.fl[i * W.B + t]);
#pragma unroll
                    for (int j = 0; j < N; j++) {
                        if (j == i) continue;
                        if (mrow[j].lo == 0.0 && mrow[j].hi == 0.0) continue;
                        const ival d = Fast::sub(mk(cl[j * stride], ch[j * stride]), mk(xv[j], xv[j]));
                        p = Fast::sub(p, gmul(mrow[j], d, prm.force_exact));
                    }
                    ival mii = mrow[0];
                    double xi = xv[0];
#pragma unroll
                    for (int j = 1; j < N; j++)
                        if (j == i) {
                            mii = mrow[j];
                            xi = xv[j];
                        }
                    ival q0 = mk(0.0, 0.0), q1 = mk(0.0, 0.0);
                    const int dk = div_extended_fast(p, mii, q0, q1, prm.force_exact);
                    if (dk == DIV_EMPTY) {
                        kind = HS_EMPTY;
                        break;
                    }
                    if (dk == DIV_WHOLE) continue;
                    const ival cur_i = mk(cl[i * stride], ch[i * stride]);
                    ival pieces[2];
                    int npieces = 0;
                    const int np = dk == DIV_SPLIT ? 2 : 1;
#pragma unroll
                    for (int q = 0; q < 2; q++) {
                        if (q < np) {
                            const ival y = Fast::add(mk(xi, xi), q == 0 ? q0 : q1);
                            const double lo = py_max(y.lo, cur_i.lo);  // Interval.intersect
                            const double hi = py_min(y.hi, cur_i.hi);
                            if (!(lo > hi)) pieces[npieces++] = mk(lo, hi);
                        }
                    }
                    if (npieces == 0) {
                        kind = HS_EMPTY;
                        break;
                    }
                    ival nc = pieces[0];
                    if (npieces == 2) {
                        nc = mk(py_min(pieces[0].lo, pieces[1].lo), py_max(pieces[0].hi, pieces[1].hi));  // hull
                        if (fork_i < 0) {
                            fork_i = i;
                            fp0 = pieces[0];
                            fp1 = pieces[1];
                        }
                    }
                    cl[i * stride] = nc.lo;
                    ch[i * stride] = nc.hi;
                }
                if (kind == HS_ONE && fork_i >= 0) kind = HS_TWO;
                if (kind == HS_ONE) {  // certified iff strictly inside the input (hansen.py:129-132)
                    cert = true;
#pragma unroll
                    for (int j = 0; j < N; j++)
                        cert = cert && (S.lo[j * S.cap + b] < cl[j * stride]) && (ch[j * stride] < S.hi[j * S.cap + b]);
                }
            }
            calls_acc++;
            ops_acc += meta.ops_hs_pre + (unsigned long long)meta.ops_hs_row * rows;
        }
        // outputs (bnb.py:197-210)
        int cnt = 0;
        bool use_input = false;
        if (valid) {
            if (kind == HS_SKIP) {
                cnt = 1;
                use_input = true;
                cert = false;
            } else if (kind == HS_EMPTY) {
                cnt = 0;
            } else if (!prm.contract_output) {
                cnt = 1;
                use_input = true;
            } else {
                cnt = kind == HS_TWO ? 2 : 1;
            }
        }
        const unsigned b1 = __ballot_sync(0xffffffffu, cnt == 1);
        const unsigned b2 = __ballot_sync(0xffffffffu, cnt == 2);
        const unsigned lt = lanemask_lt();
        const unsigned off = __popc(b1 & lt) + 2 * __popc(b2 & lt);
        const unsigned total = __popc(b1) + 2 * __popc(b2);
        unsigned long long wbase = 0;
        if (lane == 0 && total) wbase = atomicAdd(&ctr->n_next, (unsigned long long)total);
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        double wmax = 0.0;
        for (int q = 0; q < cnt; q++) {
            const unsigned long long slot = wbase + off + q;
            double w = 0.0;
#pragma unroll
            for (int j = 0; j < N; j++) {
                double lo, hi;
                if (use_input) {
                    lo = S.lo[j * S.cap + b];
                    hi = S.hi[j * S.cap + b];
                } else if (j == fork_i) {
                    lo = q == 0 ? fp0.lo : fp1.lo;
                    hi = q == 0 ? fp0.hi : fp1.hi;
                } else {
                    lo = cl[j * stride];
                    hi = ch[j * stride];
                }
                const double d = __dsub_rn(hi, lo);
                w = j == 0 ? d : (d > w ? d : w);
                if (slot < (unsigned long long)out.cap) {
                    out.lo[j * out.cap + slot] = canon0(lo);
                    out.hi[j * out.cap + slot] = canon0(hi);
                }
            }
            wmax = fmax(wmax, w);
            if (slot < (unsigned long long)out.cap) {
                out.cert[slot] = cert ? 1 : 0;
                out.unsplit[slot] = 0;
                if (tags) tags[slot] = 2 * b + q;
            }
        }
        unsigned long long wbits = (unsigned long long)__double_as_longlong(wmax);
        wbits = warp_max(wbits);
        if (lane == 0 && wbits) atomicMax(&ctr->wmax, wbits);
    }
    ops_acc = warp_sum(ops_acc);
    calls_acc = warp_sum(calls_acc);
    if (lane == 0) {
        if (ops_acc) atomicAdd(&ctr->hs_ops, ops_acc);
        if (calls_acc) atomicAdd(&ctr->hs_calls, calls_acc);
    }
}


// ------------------------------------------------------------------ K2 tiled (throughput HS)
//
// k_hs_tile: the whole HS pass over tiles of TB boxes per block (TB = blockDim.x),
// every operand of a tile in shared memory -- the throughput replacement of
// k_hs_eval -> k_hs_lin -> k_hs_sweep, whose J / M / g round trip through an HBM
// scratch (uncoalesced column reads in k_hs_lin) cost ~4.5 KB of DRAM traffic per
// box against ~0.3 KB algorithmic (ncu, katsura6 round 5).  Per tile:
//   load   thread per box: X -> tile (lo, hi, mid), coalesced SoA reads of S
//   eval   thread per box: J(X) and F(x) into the tile, layout [q][box] with a padded
//          stride (conflict-free stores; the lin groups' column reads hit distinct banks)
//   lin    G lanes per box (lin_group: Gauss-Jordan, M = A J, g = A F(x) in place)
//   sweep  thread per box on the tile (the sweep of k_hs_sweep); outputs appended to F_next
// The arithmetic is operation-for-operation that of the three-kernel pipeline.  DRAM
// traffic per box: 16n B read, <= 2 (16n + 2) B written.
template <int N>
struct TileLayout {
    static constexpr int G = LinLayout<N>::G;
    static constexpr int BPW = 32 / G;
    static constexpr int rows = 2 * N * N + 5 * N;   // J/M lo, hi; F/g lo, hi; X lo, hi, mid
    static constexpr int oJl = 0, oJh = N * N, oFl = 2 * N * N, oFh = 2 * N * N + N;
    static constexpr int oXl = 2 * N * N + 2 * N, oXh = oXl + N, oXm = oXh + N;
    static constexpr int per_group = N * N + N + 1;  // A, pivot column
};
// bytes of shared memory of a TB-box tile (after the system tables of the table evaluator)
__host__ __device__ inline size_t tile_smem_bytes(int n, int tb, int tab_bytes) {
    const int G = n <= 2 ? 4 : (n <= 4 ? 8 : (n <= 8 ? 16 : 32));
    return (size_t)align16(tab_bytes) + sizeof(double) * ((size_t)(2 * n * n + 5 * n) * (tb + 1) +
                                                          (size_t)(tb / 32) * (32 / G) * (n * n + n + 1));
}

template <int N, class EV = TabEval>
__global__ void __launch_bounds__(128) k_hs_tile(TabMeta meta, const uint8_t* __restrict__ gtab, SBuf S,
                                                 int64_t n_in_arg, HsParams prm, Front out, Counters* ctr,
                                                 int64_t* tags) {
    pdl_enter();
    using L = TileLayout<N>;
    constexpr int G = L::G;
    constexpr int P = N * N + N;
    extern __shared__ __align__(16) uint8_t smem[];
    bool hs_on;
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S.cap, hs_on);
    if (n_in < 0 || n_in <= prm.fused_max) return;  // small counts: k_hs_fused
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->hs_on = hs_on ? 1ull : 0ull;
    if (!hs_on) {
        hs_passthrough<N>(S, n_in, out, ctr, tags);
        return;
    }
    const int TB = blockDim.x, SP = TB + 1;  // boxes per tile, padded row stride
    STab tab{};
    int tab_bytes = 0;
    if constexpr (EV::tables) {
        tab = load_stab(meta, gtab, smem, false);
        tab_bytes = stab_bytes(meta, false);
    }
    double* T = reinterpret_cast<double*>(smem + align16(tab_bytes));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane / G, l = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gi * G));
    double* grp = T + (size_t)L::rows * SP + (size_t)(warp * L::BPW + gi) * L::per_group;
    const int groups = (TB / 32) * L::BPW, my_group = warp * L::BPW + gi;
    const int t = threadIdx.x;
    double* cl = T + L::oXl * SP + t;  // this thread's box during load / eval / sweep: [j * SP]
    double* ch = T + L::oXh * SP + t;
    double* cm = T + L::oXm * SP + t;
    __shared__ uint8_t s_sing[128];
    unsigned long long ops_acc = 0, calls_acc = 0, exact_acc = 0;
    for (int64_t base = (int64_t)blockIdx.x * TB; base < n_in; base += (int64_t)gridDim.x * TB) {
        const int nb = (int)min((int64_t)TB, n_in - base);
        const int64_t b = base + t;
        const bool valid = t < nb;
        __syncthreads();  // the previous tile is consumed
        // ---- load + eval: J(X) (hansen.py:61-63), F(x) (poly.py:205-207), thread per box
        if (valid) {
            ExpRange rx, rm;
            rx.init();
            rm.init();
#pragma unroll
            for (int j = 0; j < N; j++) {
                const double lo = S.lo[j * S.cap + b], hi = S.hi[j * S.cap + b];
                const double m = mid_of(lo, hi);  // Box.midpoint, poly.py:114-115
                cl[j * SP] = lo;
                ch[j * SP] = hi;
                cm[j * SP] = m;
                rx.add(lo);
                rx.add(hi);
                rm.add(m);
            }
            const bool fastJ = poly_guard_ok(meta.j_ecmin, meta.j_ecmax, meta.j_deg, rx);
            const bool fastF = poly_guard_ok(meta.f_ecmin, meta.f_ecmax, meta.f_deg, rm);
            double* jl = T + L::oJl * SP + t;
            double* jh = T + L::oJh * SP + t;
            double* fl = T + L::oFl * SP + t;
            double* fh = T + L::oFh * SP + t;
            if constexpr (EV::whole_box) {
                if (fastJ) EV::template J<Fast>(cl, ch, SP, jl, jh, SP);
                else EV::template J<Exact>(cl, ch, SP, jl, jh, SP);
                if (fastF) EV::template F<Fast>(cm, cm, SP, fl, fh, SP);
                else EV::template F<Exact>(cm, cm, SP, fl, fh, SP);
            } else {
#pragma unroll 1
                for (int q = 0; q < P; q++) {
                    if (q < N * N) {
                        const ival v = fastJ ? eval_poly<Fast>(tab, N + q, cl, ch, SP)
                                             : eval_poly_exact(tab, N + q, cl, ch, SP);
                        jl[q * SP] = v.lo;
                        jh[q * SP] = v.hi;
                    } else {
                        const int i = q - N * N;
                        const ival v = fastF ? eval_poly<Fast>(tab, i, cm, cm, SP)
                                             : eval_poly_exact(tab, i, cm, cm, SP);
                        fl[i * SP] = v.lo;
                        fh[i * SP] = v.hi;
                    }
                }
            }
            exact_acc += !(fastJ && fastF);
        }
        __syncthreads();
        // ---- lin: A = mid(J)^-1, M = A J, g = A F(x), G lanes per box (linalg.py:102-172)
        for (int bb = my_group; bb - gi < nb; bb += groups) {  // warp-uniform trip count
            if (bb < nb) {
                const LinSink K{T + L::oJl * SP + bb, T + L::oJh * SP + bb, T + L::oFl * SP + bb,
                                T + L::oFh * SP + bb, SP};
                bool exact_lin;
                const bool singular = lin_group<N, G>(K, grp, grp + N * N, l, gmask, exact_lin, prm.force_exact);
                if (l == 0) s_sing[bb] = singular ? 1 : 0;
                __syncwarp(gmask);
            }
            __syncwarp();
        }
        __syncthreads();
        // ---- sweep (hansen.py:91-138), thread per box; the tile's X lo/hi become the current box
        int kind = HS_EMPTY;
        bool cert = false;
        int fork_i = -1;
        ival fp0 = mk(0.0, 0.0), fp1 = mk(0.0, 0.0);
        int rows = 0;
        if (valid) {
            const double* Ml = T + L::oJl * SP + t;
            const double* Mh = T + L::oJh * SP + t;
            if (s_sing[t]) {
                kind = HS_SKIP;
            } else {
                kind = HS_ONE;
#pragma unroll 1
                for (int i = 0; i < N; i++) {
                    rows = i + 1;
                    // p = -g_i - sum_{j != i, M_ij != [0,0]} M_ij (current_j - [x_j, x_j]), left to right
                    ival p = mk(-T[L::oFh * SP + i * SP + t], -T[L::oFl * SP + i * SP + t]);
#pragma unroll
                    for (int j = 0; j < N; j++) {
                        if (j == i) continue;
                        const ival m = mk(Ml[(i * N + j) * SP], Mh[(i * N + j) * SP]);
                        if (m.lo == 0.0 && m.hi == 0.0) continue;
                        const ival d = Fast::sub(mk(cl[j * SP], ch[j * SP]), mk(cm[j * SP], cm[j * SP]));
                        p = Fast::sub(p, gmul(m, d, prm.force_exact));
                    }
                    const ival mii = mk(Ml[(i * N + i) * SP], Mh[(i * N + i) * SP]);
                    const double xi = cm[i * SP];
                    ival q0 = mk(0.0, 0.0), q1 = mk(0.0, 0.0);
                    const int dk = div_extended_fast(p, mii, q0, q1, prm.force_exact);
                    if (dk == DIV_EMPTY) {
                        kind = HS_EMPTY;
                        break;
                    }
                    if (dk == DIV_WHOLE) continue;
                    const ival cur_i = mk(cl[i * SP], ch[i * SP]);
                    ival pieces[2];
                    int npieces = 0;
                    const int np = dk == DIV_SPLIT ? 2 : 1;
#pragma unroll
                    for (int q = 0; q < 2; q++) {
                        if (q < np) {
                            const ival y = Fast::add(mk(xi, xi), q == 0 ? q0 : q1);
                            const double lo = py_max(y.lo, cur_i.lo);  // Interval.intersect
                            const double hi = py_min(y.hi, cur_i.hi);
                            if (!(lo > hi)) pieces[npieces++] = mk(lo, hi);
                        }
                    }
                    if (npieces == 0) {
                        kind = HS_EMPTY;
                        break;
                    }
                    ival nc = pieces[0];
                    if (npieces == 2) {
                        nc = mk(py_min(pieces[0].lo, pieces[1].lo), py_max(pieces[0].hi, pieces[1].hi));  // hull
                        if (fork_i < 0) {
                            fork_i = i;
                            fp0 = pieces[0];
                            fp1 = pieces[1];
                        }
                    }
                    cl[i * SP] = nc.lo;
                    ch[i * SP] = nc.hi;
                }
                if (kind == HS_ONE && fork_i >= 0) kind = HS_TWO;
                if (kind == HS_ONE) {  // certified iff strictly inside the input (hansen.py:129-132)
                    cert = true;
#pragma unroll
                    for (int j = 0; j < N; j++)
                        cert = cert && (S.lo[j * S.cap + b] < cl[j * SP]) && (ch[j * SP] < S.hi[j * S.cap + b]);
                }
            }
            calls_acc++;
            ops_acc += meta.ops_hs_pre + (unsigned long long)meta.ops_hs_row * rows;
        }
        // outputs (bnb.py:197-210)
        int cnt = 0;
        bool use_input = false;
        if (valid) {
            if (kind == HS_SKIP) {
                cnt = 1;
                use_input = true;
                cert = false;
            } else if (kind == HS_EMPTY) {
                cnt = 0;
            } else if (!prm.contract_output) {
                cnt = 1;
                use_input = true;
            } else {
                cnt = kind == HS_TWO ? 2 : 1;
            }
        }
        const unsigned b1 = __ballot_sync(0xffffffffu, cnt == 1);
        const unsigned b2 = __ballot_sync(0xffffffffu, cnt == 2);
        const unsigned lt = lanemask_lt();
        const unsigned off = __popc(b1 & lt) + 2 * __popc(b2 & lt);
        const unsigned total = __popc(b1) + 2 * __popc(b2);
        unsigned long long wbase = 0;
        if (lane == 0 && total) wbase = atomicAdd(&ctr->n_next, (unsigned long long)total);
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        double wmax = 0.0;
        for (int q = 0; q < cnt; q++) {
            const unsigned long long slot = wbase + off + q;
            double w = 0.0;
#pragma unroll
            for (int j = 0; j < N; j++) {
                double lo, hi;
                if (use_input) {
                    lo = S.lo[j * S.cap + b];
                    hi = S.hi[j * S.cap + b];
                } else if (j == fork_i) {
                    lo = q == 0 ? fp0.lo : fp1.lo;
                    hi = q == 0 ? fp0.hi : fp1.hi;
                } else {
                    lo = cl[j * SP];
                    hi = ch[j * SP];
                }
                const double d = __dsub_rn(hi, lo);
                w = j == 0 ? d : (d > w ? d : w);
                if (slot < (unsigned long long)out.cap) {
                    out.lo[j * out.cap + slot] = canon0(lo);
                    out.hi[j * out.cap + slot] = canon0(hi);
                }
            }
            wmax = fmax(wmax, w);
            if (slot < (unsigned long long)out.cap) {
                out.cert[slot] = cert ? 1 : 0;
                out.unsplit[slot] = 0;
                if (tags) tags[slot] = 2 * b + q;
            }
        }
        unsigned long long wbits = (unsigned long long)__double_as_longlong(wmax);
        wbits = warp_max(wbits);
        if (lane == 0 && wbits) atomicMax(&ctr->wmax, wbits);
    }
    ops_acc = warp_sum(ops_acc);
    calls_acc = warp_sum(calls_acc);
    exact_acc = warp_sum(exact_acc);
    if (lane == 0) {
        if (ops_acc) atomicAdd(&ctr->hs_ops, ops_acc);
        if (calls_acc) atomicAdd(&ctr->hs_calls, calls_acc);
        if (exact_acc) atomicAdd(&ctr->exact_boxes, exact_acc);
    }
}

// ------------------------------------------------------------------ K2 fused
//
// k_hs_fused: the whole HS pass (K2a + K2b + K2c) for one box by the G lanes of a
// group, operands in a shared-memory tile instead of the HBM scratch:
//   eval   lane l evaluates polynomials l, l + G, ... of the n^2 + n (J(X), F(x))
//   lin    lin_group (Gauss-Jordan + M = A J, g = A F(x)) on the tile
//   sweep  row i: lane j forms M_ij (X_j - x_j) for its column in parallel, then
//          every lane folds the products left to right (the reference order) and
//          runs the same extended division, so control flow stays group-uniform
// The arithmetic is operation-for-operation that of the three-kernel pipeline.
// Stable in-place removal of the dead (duplicate) rows of f[0, n) by one block:
// chunk by chunk, every row of a chunk is read before any is written, and a row
// moves only to a lower index, so no unread row is overwritten.
template <int N>
__device__ void compact_inplace_block(Front f, int64_t n, const uint8_t* dead) {
    __shared__ unsigned s_warp[32];
    __shared__ long long s_written;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) s_written = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const bool live = i < n && !dead[i];
        double lo[N], hi[N];
        uint8_t c = 0, u = 0;
        if (live) {
#pragma unroll
            for (int j = 0; j < N; j++) lo[j] = f.lo[j * f.cap + i], hi[j] = f.hi[j * f.cap + i];
            c = f.cert[i];
            u = f.unsplit[i];
        }
        const unsigned b = __ballot_sync(0xffffffffu, live);
        if (lane == 0) s_warp[warp] = __popc(b);
        __syncthreads();
        long long pos = s_written + __popc(b & lanemask_lt());
        for (int w = 0; w < warp; w++) pos += s_warp[w];
        long long tot = 0;
        for (int w = 0; w < nw; w++) tot += s_warp[w];
        __syncthreads();  // every read of the chunk (and of s_warp / s_written) before the writes
        if (live) {
#pragma unroll
            for (int j = 0; j < N; j++) f.lo[j * f.cap + pos] = lo[j], f.hi[j * f.cap + pos] = hi[j];
            f.cert[pos] = c;
            f.unsplit[pos] = u;
        }
        if (threadIdx.x == 0) s_written += tot;
        __syncthreads();
    }
}

static __device__ __noinline__ bool round_end_warp(DevState* st, Counters* ctr, DevRoundStats* stats, int n,
                                                   int64_t s_cap, int* eq_order, const TabMeta& meta,
                                                   bool pingpong);

// End of a round inside the HS kernel (ping-pong round graph): the last block to
// finish removes duplicate rows and runs the round end (bnb.py:322-352).
// Only the blocks that can have written rows take part: `rows_per_block` rows (or
// boxes) per block in a grid-stride loop over `n` -- the others return at once, so the
// block-done counter sees a few atomics instead of one per block of the grid.
template <int N>
__device__ void hs_round_end(const HsParams& prm, Counters* ctr, const Front& out, const TabMeta& meta,
                             int64_t n, int rows_per_block) {
    __shared__ int s_last;
    const int64_t need = (n + rows_per_block - 1) / rows_per_block;
    const unsigned parts = (unsigned)(need < 1 ? 1 : (need > (int64_t)gridDim.x ? (int64_t)gridDim.x : need));
    if (blockIdx.x >= parts) return;  // block-uniform
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&ctr->tail_done, 1ull) == (unsigned long long)(parts - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (*(volatile unsigned long long*)&ctr->dups != 0ull)
        compact_inplace_block<N>(out, (int64_t)*(volatile unsigned long long*)&ctr->n_next, prm.dd.dead);
    __syncthreads();
    if (threadIdx.x < 32)
        round_end_warp(const_cast<DevState*>(prm.st), ctr, prm.rstats, N, prm.s_cap, prm.eq_order, meta, true);
}

#ifndef RB_FUSED_G32
#define RB_FUSED_G32 1  // one warp per box in k_hs_fused for n >= 3
#endif
template <int N>
struct FusedLayout {
    static constexpr int G = (RB_FUSED_G32 && N >= 3) ? 32 : LinLayout<N>::G;
    static constexpr int BPW = 32 / G;
    static constexpr int oXl = 0, oXh = N, oXm = 2 * N;
    static constexpr int oJl = 3 * N, oJh = 3 * N + N * N;
    static constexpr int oFl = 3 * N + 2 * N * N, oFh = oFl + N;
    static constexpr int oA = oFh + N;
    static constexpr int oCol = oA + N * N;
    static constexpr int doubles = oCol + N + 1;
};

__host__ __device__ inline int fused_off_tiles(const TabMeta& m) { return align16(stab_bytes(m, false)); }

template <int N, class EV = TabEval>
__device__ __forceinline__ void k_hs_fused_body(TabMeta meta, const uint8_t* __restrict__ gtab, SBuf S,
                                                  int64_t n_in_arg, HsParams prm, Front out, Counters* ctr,
                                                  int64_t* tags) {
    using L = FusedLayout<N>;
    constexpr int G = L::G;
    constexpr int P = N * N + N;
    extern __shared__ __align__(16) uint8_t smem[];
    bool hs_on;
    const bool prof = prm.prof && blockIdx.x == 0 && threadIdx.x == 0;
    if (prof) prm.prof[0] = gtimer(), prm.prof[1] = clock64();
    unsigned long long* btr = (prm.prof && threadIdx.x == 0 && blockIdx.x < kTraceBlocks) ? prm.prof + 48 + 3 * blockIdx.x : nullptr;
    if (btr) btr[0] = gtimer();
    // the system tables are constant: copied before waiting on the previous kernel (PDL),
    // and in flight while the survivor count is read
    STab tab{};
    if constexpr (EV::tables) tab = issue_stab(meta, gtab, smem, false);
    pdl_wait();
    // this group's first box, loaded speculatively (any row below S.cap is addressable)
    // so its latency overlaps the survivor-count read; used only if the box exists
    const int lane0 = threadIdx.x & 31, warp0 = threadIdx.x >> 5;
    const int64_t b_first = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp0) * L::BPW + lane0 / G;
    double pre_lo = 0.0, pre_hi = 0.0;
    if (lane0 % G < N && b_first < S.cap) {
        pre_lo = S.lo[(lane0 % G) * S.cap + b_first];
        pre_hi = S.hi[(lane0 % G) * S.cap + b_first];
    }
    if (prm.round_end && (prm.st->done || prm.st->bail)) {  // unrolled round after the end of the loop
        cp_async_wait();
        return;
    }
    const int64_t n_in = hs_count(prm, ctr, n_in_arg, S.cap, hs_on);
    if (prof) prm.prof[2] = clock64();
    if (prm.has_cond && blockIdx.x == 0 && threadIdx.x == 0)
        RB_SET_COND(prm.big_cond, n_in > prm.fused_max ? 1u : 0u);
    cp_async_wait();
    if (n_in < 0 || n_in > prm.fused_max) return;  // large counts: eval/lin/sweep
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->hs_on = hs_on ? 1ull : 0ull;
    if (!hs_on) {
        hs_passthrough<N>(S, n_in, out, ctr, tags, prm.dd);
        if (prm.round_end) hs_round_end<N>(prm, ctr, out, meta, n_in, (int)blockDim.x);
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane / G, l = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gi * G));
    const unsigned below = (G == 32) ? 0u : ((1u << (gi * G)) - 1u);  // lanes of the groups before mine
    double* s = reinterpret_cast<double*>(smem + fused_off_tiles(meta)) + (size_t)(warp * L::BPW + gi) * L::doubles;
    const LinSink K{s + L::oJl, s + L::oJh, s + L::oFl, s + L::oFh, 1};
    __syncthreads();
    if (prof) prm.prof[3] = clock64();
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t wglob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    unsigned long long ops_acc = 0, calls_acc = 0, exact_acc = 0;
    for (int64_t wb0 = wglob * L::BPW; wb0 < n_in; wb0 += warps_total * L::BPW) {
        const int64_t b = wb0 + gi;
        const bool valid = b < n_in;
        int kind = HS_EMPTY;
        bool cert = false;
        int fork_i = -1;
        ival fp0 = mk(0.0, 0.0), fp1 = mk(0.0, 0.0);
        ival cur = mk(0.0, 0.0);  // lane j < N: component j of the box being contracted
        int rows = 0;
        if (valid) {
            if (l < N) {
                const bool first = b == b_first;
                const double lo = first ? pre_lo : S.lo[l * S.cap + b], hi = first ? pre_hi : S.hi[l * S.cap + b];
                s[L::oXl + l] = lo;
                s[L::oXh + l] = hi;
                s[L::oXm + l] = mid_of(lo, hi);  // Box.midpoint, poly.py:114-115
                cur = mk(lo, hi);
            }
            __syncwarp(gmask);
            // ---- eval: J(X) (hansen.py:61-63) and F(x) (poly.py:205-207)
            if (prof && wb0 == 0) prm.prof[4] = clock64();
            unsigned long long* brec = (prm.prof && l == 0 && b < kTraceBoxes) ? prm.prof + kTraceBoxOff + 8 * b : nullptr;
            if (brec) brec[0] = gtimer();
            ExpRange rx, rm;
            rx.init();
            rm.init();
#pragma unroll
            for (int j = 0; j < N; j++) {
                rx.add(s[L::oXl + j]);
                rx.add(s[L::oXh + j]);
                rm.add(s[L::oXm + j]);
            }
            const bool fastJ = poly_guard_ok(meta.j_ecmin, meta.j_ecmax, meta.j_deg, rx);
            const bool fastF = poly_guard_ok(meta.f_ecmin, meta.f_ecmax, meta.f_deg, rm);
            if constexpr (EV::whole_box) {  // specialised evaluator: lane 0 of the group, straight-line code
                if (l == 0) {
                    if (fastJ) EV::template J<Fast>(s + L::oXl, s + L::oXh, 1, s + L::oJl, s + L::oJh, 1);
                    else EV::template J<Exact>(s + L::oXl, s + L::oXh, 1, s + L::oJl, s + L::oJh, 1);
                    if (fastF) EV::template F<Fast>(s + L::oXm, s + L::oXm, 1, s + L::oFl, s + L::oFh, 1);
                    else EV::template F<Exact>(s + L::oXm, s + L::oXm, 1, s + L::oFl, s + L::oFh, 1);
                }
            }
#pragma unroll 1
            for (int q = EV::whole_box ? P : l; q < P; q += G) {
                if (q < N * N) {
                    const ival v = fastJ ? eval_poly<Fast>(tab, N + q, s + L::oXl, s + L::oXh, 1)
                                         : eval_poly_exact(tab, N + q, s + L::oXl, s + L::oXh, 1);
                    s[L::oJl + q] = v.lo;
                    s[L::oJh + q] = v.hi;
                } else {
                    const int i = q - N * N;
                    const ival v = fastF ? eval_poly<Fast>(tab, i, s + L::oXm, s + L::oXm, 1)
                                         : eval_poly_exact(tab, i, s + L::oXm, s + L::oXm, 1);
                    s[L::oFl + i] = v.lo;
                    s[L::oFh + i] = v.hi;
                }
            }
            if (l == 0 && !(fastJ && fastF)) exact_acc++;
            __syncwarp(gmask);
            if (prof && wb0 == 0) prm.prof[5] = clock64();
            if (brec) brec[1] = gtimer();
            // ---- lin: A = mid(J)^-1, M = A J, g = A F(x)
            bool exact_lin;
            const bool singular = lin_group<N, G>(K, s + L::oA, s + L::oCol, l, gmask, exact_lin, prm.force_exact,
                                                  (prof && wb0 == 0) ? prm.prof + 11 : nullptr);
            __syncwarp(gmask);
            if (prof && wb0 == 0) prm.prof[6] = clock64();
            if (brec) brec[2] = gtimer();
            if (singular) {
                kind = HS_SKIP;
            } else {
                // ---- sweep (hansen.py:91-138)
                kind = HS_ONE;
                const double xj = l < N ? s[L::oXm + l] : 0.0;
                // directed reciprocals of the diagonal, off the sweep's dependency chain: lane l
                // holds 1/M_ll for row l (the single case of div_extended_fast, recip_dir)
                bool dfast = false;
                ival dinv = mk(0.0, 0.0);
                if (l < N) {
                    const ival y = mk(s[L::oJl + l * N + l], s[L::oJh + l * N + l]);
                    dfast = !prm.force_exact && !contains_zero(y) &&
                            fmin(fabs(y.lo), fabs(y.hi)) > 0x1p-990 && fmax(fabs(y.lo), fabs(y.hi)) < 0x1p990;
                    if (dfast) dinv = mk(recip_dir(y.hi, false), recip_dir(y.lo, true));
                }
#pragma unroll 1
                for (int i = 0; i < N; i++) {
                    rows = i + 1;
                    ival prod = mk(0.0, 0.0);
                    bool use = false;
                    if (l < N && l != i) {
                        const ival m = mk(s[L::oJl + i * N + l], s[L::oJh + i * N + l]);
                        use = !(m.lo == 0.0 && m.hi == 0.0);
                        if (use) prod = gmul(m, Fast::sub(cur, mk(xj, xj)), prm.force_exact);
                    }
                    const unsigned um = __ballot_sync(gmask, use) >> (gi * G);
                    // p = -g_i - sum_{j != i, M_ij != [0,0]} M_ij (current_j - [x_j, x_j]), left to right
                    ival p = mk(-s[L::oFh + i], -s[L::oFl + i]);
#pragma unroll(N <= 8 ? N : 1)  // a fully unrolled fold of 12+ shuffles trips ptxas (C7600)
                    for (int j = 0; j < N; j++) {
                        const double plo = gshfl<G>(gmask, prod.lo, j);
                        const double phi = gshfl<G>(gmask, prod.hi, j);
                        if (um & (1u << j)) p = Fast::sub(p, mk(plo, phi));
                    }
                    const ival mii = mk(s[L::oJl + i * N + i], s[L::oJh + i * N + i]);
                    const double xi = s[L::oXm + i];
                    const ival cur_i = mk(gshfl<G>(gmask, cur.lo, i), gshfl<G>(gmask, cur.hi, i));
                    ival q0 = mk(0.0, 0.0), q1 = mk(0.0, 0.0);
                    const bool fi = __shfl_sync(gmask, dfast, i, G);
                    const ival ri = mk(gshfl<G>(gmask, dinv.lo, i), gshfl<G>(gmask, dinv.hi, i));
                    int dk;
                    if (fi) {  // == div_extended_fast's single case
                        q0 = gmul(p, ri);
                        dk = DIV_SINGLE;
                    } else {
                        dk = div_extended(p, mii, q0, q1, prm.force_exact);
                    }
                    if (dk == DIV_EMPTY) {
                        kind = HS_EMPTY;
                        break;
                    }
                    if (dk == DIV_WHOLE) continue;
                    ival pieces[2];
                    int npieces = 0;
                    const int np = dk == DIV_SPLIT ? 2 : 1;
#pragma unroll
                    for (int q = 0; q < 2; q++) {
                        if (q < np) {
                            const ival y = Fast::add(mk(xi, xi), q == 0 ? q0 : q1);
                            const double lo = py_max(y.lo, cur_i.lo);  // Interval.intersect
                            const double hi = py_min(y.hi, cur_i.hi);
                            if (!(lo > hi)) pieces[npieces++] = mk(lo, hi);
                        }
                    }
                    if (npieces == 0) {
                        kind = HS_EMPTY;
                        break;
                    }
                    ival nc = pieces[0];
                    if (npieces == 2) {
                        nc = mk(py_min(pieces[0].lo, pieces[1].lo), py_max(pieces[0].hi, pieces[1].hi));  // hull
                        if (fork_i < 0) {
                            fork_i = i;
                            fp0 = pieces[0];
                            fp1 = pieces[1];
                        }
                    }
                    if (l == i) cur = nc;
                }
                if (kind == HS_ONE && fork_i >= 0) kind = HS_TWO;
                if (kind == HS_ONE) {  // certified iff strictly inside the input (hansen.py:129-132)
                    const bool in = l >= N || (s[L::oXl + l] < cur.lo && cur.hi < s[L::oXh + l]);
                    cert = __all_sync(gmask, in);
                }
            }
            if (l == 0) {
                calls_acc++;
                ops_acc += meta.ops_hs_pre + (unsigned long long)meta.ops_hs_row * rows;
            }
        }
        // outputs (bnb.py:197-210): group leaders reserve slots for the warp
        if (prof && wb0 == 0) prm.prof[7] = clock64();
        if (prm.prof && valid && l == 0 && b < kTraceBoxes) {
            unsigned long long* br = prm.prof + kTraceBoxOff + 8 * b;
            br[3] = gtimer();
            br[5] = (unsigned long long)rows | ((unsigned long long)kind << 8) | ((unsigned long long)smid() << 16);
            br[6] = prm.st ? (unsigned long long)prm.st->round_no : 0ull;
        }
        int cnt = 0;
        bool use_input = false;
        if (valid) {
            if (kind == HS_SKIP) {
                cnt = 1;
                use_input = true;
                cert = false;
            } else if (kind == HS_EMPTY) {
                cnt = 0;
            } else if (!prm.contract_output) {
                cnt = 1;
                use_input = true;
            } else {
                cnt = kind == HS_TWO ? 2 : 1;
            }
        }
        const unsigned b1 = __ballot_sync(0xffffffffu, l == 0 && cnt == 1);
        const unsigned b2 = __ballot_sync(0xffffffffu, l == 0 && cnt == 2);
        const unsigned off = __popc(b1 & below) + 2 * __popc(b2 & below);
        const unsigned total = __popc(b1) + 2 * __popc(b2);
        unsigned long long wbase = 0;
        if (lane == 0 && total) wbase = atomicAdd(&ctr->n_next, (unsigned long long)total);
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        double wmax = 0.0;
        for (int q = 0; q < cnt; q++) {  // group-uniform
            const unsigned long long slot = wbase + off + q;
            double w = 0.0, w_lo = 0.0, w_hi = 0.0;
            if (l < N) {
                double lo, hi;
                if (use_input) {
                    lo = s[L::oXl + l];
                    hi = s[L::oXh + l];
                } else if (l == fork_i) {
                    lo = q == 0 ? fp0.lo : fp1.lo;
                    hi = q == 0 ? fp0.hi : fp1.hi;
                } else {
                    lo = cur.lo;
                    hi = cur.hi;
                }
                w = __dsub_rn(hi, lo);
                w_lo = lo;
                w_hi = hi;
                if (slot < (unsigned long long)out.cap) {
                    out.lo[l * out.cap + slot] = canon0(lo);
                    out.hi[l * out.cap + slot] = canon0(hi);
                }
            }
            wmax = fmax(wmax, w);
            if (l == 0 && slot < (unsigned long long)out.cap) {
                out.cert[slot] = cert ? 1 : 0;
                out.unsplit[slot] = 0;
                if (tags) tags[slot] = 2 * b + q;
            }
            const bool any_thin = __any_sync(gmask, l < N && thin_comp(w_lo, w_hi));
            if ((prm.dd.table || prm.dd.etable) && !any_thin) {  // no duplicate possible (kThinUlps)
                if (l == 0 && slot < (unsigned long long)out.cap) {
                    prm.dd.dead[slot] = 0;
                    prm.dd.slot_of[slot] = 0xffffffffu;
                }
            } else if (prm.dd.table || prm.dd.etable) {  // group-uniform: gather the row into lane 0, insert it
                double rlo[N], rhi[N];
                const double mlo = canon0(w_lo), mhi = canon0(w_hi);
#pragma unroll
                for (int j = 0; j < N; j++) {
                    rlo[j] = gshfl<G>(gmask, mlo, j);
                    rhi[j] = gshfl<G>(gmask, mhi, j);
                }
                __syncwarp(gmask);  // the group's row stores before lane 0's release
                if (l == 0 && slot < (unsigned long long)out.cap)
                    dedup_insert_regs<N>(out, (int64_t)slot, rlo, rhi, cert ? 1 : 0, 0, prm.dd, ctr);
            }
        }
        if (prm.prof && valid && l == 0 && b < kTraceBoxes) prm.prof[kTraceBoxOff + 8 * b + 7] = gtimer();
        unsigned long long wbits = (unsigned long long)__double_as_longlong(wmax);
        wbits = warp_max(wbits);
        if (lane == 0 && wbits) atomicMax(&ctr->wmax, wbits);
        __syncwarp();  // the tile is reused by the next box of this group
        if (prof && wb0 == 0) prm.prof[8] = clock64();
        if (prm.prof && valid && l == 0 && b < kTraceBoxes) prm.prof[kTraceBoxOff + 8 * b + 4] = gtimer();
    }
    ops_acc = warp_sum(ops_acc);
    calls_acc = warp_sum(calls_acc);
    exact_acc = warp_sum(exact_acc);
    if (lane == 0) {
        if (ops_acc) atomicAdd(&ctr->hs_ops, ops_acc);
        if (calls_acc) atomicAdd(&ctr->hs_calls, calls_acc);
        if (exact_acc) atomicAdd(&ctr->exact_boxes, exact_acc);
    }
    if (prof) prm.prof[9] = clock64(), prm.prof[10] = gtimer();
    if (prm.prof) __syncthreads();  // block-uniform
    if (btr) {
        btr[1] = gtimer();
        btr[2] = smid();
    }
    if (prm.round_end) hs_round_end<N>(prm, ctr, out, meta, n_in, (int)(blockDim.x >> 5) * L::BPW);
}

template <int N, class EV = TabEval>
__global__ void RB_FUSED_BOUNDS k_hs_fused(TabMeta meta, const uint8_t* __restrict__ gtab, SBuf S,
                                                  int64_t n_in_arg, HsParams prm, Front out, Counters* ctr,
                                                  int64_t* tags) {
    pdl_launch();
    k_hs_fused_body<N, EV>(meta, gtab, S, n_in_arg, prm, out, ctr, tags);  // waits after the table copies
}

// ------------------------------------------------------------------ dedup

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {  // declared above
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

template <int N>
__device__ __forceinline__ unsigned long long row_hash(const Front& f, int64_t i) {
    unsigned long long h = 0x9e3779b97f4a7c15ull;
#pragma unroll
    for (int j = 0; j < N; j++) {
        h = mix64(h ^ (unsigned long long)__double_as_longlong(canon0(f.lo[j * f.cap + i])));
        h = mix64(h ^ (unsigned long long)__double_as_longlong(canon0(f.hi[j * f.cap + i])));
    }
    return h;
}

template <int N>
__device__ __forceinline__ bool rows_equal(const Front& f, int64_t a, int64_t b) {
#pragma unroll
    for (int j = 0; j < N; j++)
        if (!(f.lo[j * f.cap + a] == f.lo[j * f.cap + b]) || !(f.hi[j * f.cap + a] == f.hi[j * f.cap + b]))
            return false;
    return true;
}

__device__ __forceinline__ void atomic_or_u8(uint8_t* p, uint8_t v) { atomic_or_u8_(p, v); }

// The round's dedup runs without host knowledge of the frontier size: both
// kernels read n_next from the counters and do nothing when the round
// overflowed a buffer (the host then grows the buffers and redoes the round).
__device__ __forceinline__ bool round_ok(const Counters* c, int64_t s_cap, int64_t f_cap) {
    return c->n_surv <= (unsigned long long)s_cap && c->n_next <= (unsigned long long)f_cap;
}

// Open-addressing insert of every row; a row equal to an already inserted one
// is marked dead and ORs its flags into the keeper (dedup_sorted, _batch.py:253-266).
// slot_of[i] records the occupied slot so k_dedup_finish can leave the table clean.
template <int N>
__device__ __forceinline__ void k_dedup_insert_body(Front f, unsigned* table, unsigned long long mask, unsigned* slot_of, uint8_t* dead,
                               Counters* ctr, int64_t s_cap) {
    if (!round_ok(ctr, s_cap, f.cap)) return;
    const int64_t n = (int64_t)ctr->n_next;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long slot = row_hash<N>(f, i) & mask;
        bool dup = false;
        while (true) {
            const unsigned prev = atomicCAS(&table[slot], 0u, (unsigned)(i + 1));
            if (prev == 0u) break;
            const int64_t k = (int64_t)prev - 1;
            if (rows_equal<N>(f, k, i)) {
                dup = true;
                atomic_or_u8(&f.cert[k], f.cert[i]);
                atomic_or_u8(&f.unsplit[k], f.unsplit[i]);
                break;
            }
            slot = (slot + 1) & mask;
        }
        dead[i] = dup ? 1 : 0;
        slot_of[i] = dup ? 0xffffffffu : (unsigned)slot;
        if (dup) atomicAdd(&ctr->dups, 1ull);
    }
}

template <int N>
__global__ void k_dedup_insert(Front f, unsigned* table, unsigned long long mask, unsigned* slot_of, uint8_t* dead,
                               Counters* ctr, int64_t s_cap) {
    pdl_enter();
    k_dedup_insert_body<N>(f, table, mask, slot_of, dead, ctr, s_cap);
}

// Clear the used table slots; when duplicates were found, compact the live rows
// into dst (counter ctr->n_compact).
template <int N>
__device__ __forceinline__ void k_dedup_finish_body(Front src, Front dst, unsigned* table, const unsigned* slot_of, const uint8_t* dead,
                               Counters* ctr, int64_t s_cap) {
    if (!round_ok(ctr, s_cap, src.cap)) return;
    const int64_t n = (int64_t)ctr->n_next;
    const bool compact = ctr->dups != 0;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        if (i < n && slot_of[i] != 0xffffffffu) table[slot_of[i]] = 0u;
        if (!compact) continue;
        const bool live = i < n && !dead[i];
        const unsigned long long slot = warp_append(live, &ctr->n_compact);
        if (live) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                dst.lo[j * dst.cap + slot] = src.lo[j * src.cap + i];
                dst.hi[j * dst.cap + slot] = src.hi[j * src.cap + i];
            }
            dst.cert[slot] = src.cert[i];
            dst.unsplit[slot] = src.unsplit[i];
        }
    }
}

template <int N>
__global__ void k_dedup_finish(Front src, Front dst, unsigned* table, const unsigned* slot_of, const uint8_t* dead,
                               Counters* ctr, int64_t s_cap) {
    pdl_enter();
    k_dedup_finish_body<N>(src, dst, table, slot_of, dead, ctr, s_cap);
}

// ------------------------------------------------------------------ graph-mode round end

// Bring the round's frontier back into F[0]: k_dedup_finish already compacted
// into F[0] when duplicates were removed; otherwise copy F[1] -> F[0].
template <int N>
__global__ void k_settle(Front f1, Front f0, const Counters* ctr) {
    pdl_enter();
    if (ctr->dups != 0) return;
    const int64_t n = (int64_t)ctr->n_next;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int j = 0; j < N; j++) {
            f0.lo[j * f0.cap + i] = f1.lo[j * f1.cap + i];
            f0.hi[j * f0.cap + i] = f1.hi[j * f1.cap + i];
        }
        f0.cert[i] = f1.cert[i];
        f0.unsplit[i] = f1.unsplit[i];
    }
}

// Round statistics, termination (bnb.py:339-352) and the WHILE condition of the
// device round loop; also clears the counters for the next round.
// One thread.  Returns true when the device loop should run another round.
static __device__ __noinline__ bool round_end_body(DevState* st, Counters* ctr, DevRoundStats* stats, int n, int64_t s_cap,
                                            int* eq_order, const TabMeta& meta) {
    const Counters c = *ctr;
    filter_order(c.f_eval, c.f_rej, meta.cost_eq, n, eq_order);
    const unsigned long long after = c.n_next - c.dups;
    const double width = after ? __longlong_as_double((long long)c.wmax) : 0.0;
    const unsigned long long now = gtimer();
    DevRoundStats& r = stats[st->round_no - 1];
    r.round = st->round_no;
    r.boxes_in = (long long)st->n_cur;
    r.after_filter = (long long)(c.n_carried + c.n_surv);
    r.after_hs = (long long)after;
    r.children = (long long)(c.n_par << n);
    r.hs_calls = (long long)c.hs_calls;
    r.filter_ops = (long long)c.filter_ops;
    r.hs_ops = (long long)c.hs_ops;
    r.dups = (long long)c.dups;
    r.exact = (long long)c.exact_boxes;
    r.hs_on = (long long)c.hs_on;
    r.width = width;
    r.elapsed = (double)(now - st->t_round_ns) * 1e-9;
    st->t_round_ns = now;
    st->n_cur = after;
    st->nrounds = st->round_no;
    if (after == 0) {
        st->done = 1;
        st->status = 0;  // no_real_solution
    } else if (width <= st->target) {
        st->done = 1;
        st->status = 1;  // width_reached
    } else if ((long long)after > st->max_boxes || st->round_no >= st->max_rounds) {
        st->done = 1;
        st->status = 2;  // budget_exhausted
    } else {
        st->round_no += 1;
        if ((after << n) > (unsigned long long)s_cap) st->bail = 1;  // next round needs the host
    }
    unsigned long long* w = reinterpret_cast<unsigned long long*>(ctr);
    for (int i = 0; i < (int)(sizeof(Counters) / 8); i++) w[i] = 0ull;
    return !(st->done || st->bail);
}

#ifndef RB_KINST_TU
__global__ void k_round_end(DevState* st, Counters* ctr, DevRoundStats* stats, int n, int64_t s_cap,
                            cudaGraphConditionalHandle h_while, int* eq_order, TabMeta meta) {
    pdl_enter();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const bool cont = round_end_body(st, ctr, stats, n, s_cap, eq_order, meta);
    cudaGraphSetConditional(h_while, cont ? 1u : 0u);
}
#endif

// round_end_body by one warp (lane 0 of a warp, all 32 lanes present): the counters
// are staged in shared memory with one coalesced load, the equation order is ranked
// in parallel (the same stable descending sort as filter_order) and the counters
// are cleared by all lanes.  Returns the WHILE condition (every lane).
static __device__ __noinline__ bool round_end_warp(DevState* st, Counters* ctr, DevRoundStats* stats, int n,
                                            int64_t s_cap, int* eq_order, const TabMeta& meta,
                                            bool pingpong) {
    constexpr int W = (int)(sizeof(Counters) / 8);
    __shared__ __align__(128) unsigned long long sc[W];
    const int lane = threadIdx.x & 31;
    unsigned long long* w = reinterpret_cast<unsigned long long*>(ctr);
    for (int i = lane; i < W; i += 32) sc[i] = w[i];
    const int cur_e = lane < n ? eq_order[lane] : 0;
    const DevState s0 = *st;
    __syncwarp();
    const Counters& c = *reinterpret_cast<const Counters*>(sc);
    // filter_order: key of the equation at position `lane`, rank = #greater + #equal before
    double key = -1.0;
    if (lane < n) {
        const unsigned long long ev = c.f_eval[cur_e], rj = c.f_rej[cur_e];
        const int ops = meta.cost_eq[cur_e];
        key = ev ? ((double)rj / (double)ev) / (double)(ops > 0 ? ops : 1) : -1.0;
    }
    int rank = 0;
    for (int b = 0; b < n; b++) {
        const double kb = __shfl_sync(0xffffffffu, key, b);
        rank += (kb > key) || (b < lane && kb == key);
    }
    if (lane < n) eq_order[rank] = cur_e;
    for (int i = lane; i < W; i += 32) w[i] = 0ull;
    int cont = 0;
    if (lane == 0) {
        const unsigned long long after = c.n_next - c.dups;
        const double width = after ? __longlong_as_double((long long)c.wmax) : 0.0;
        const unsigned long long now = gtimer();
        DevRoundStats r;
        r.round = s0.round_no;
        r.boxes_in = (long long)s0.n_cur;
        r.after_filter = (long long)(c.n_carried + c.n_surv);
        r.after_hs = (long long)after;
        r.children = (long long)(c.n_par << n);
        r.hs_calls = (long long)c.hs_calls;
        r.filter_ops = (long long)c.filter_ops;
        r.hs_ops = (long long)c.hs_ops;
        r.dups = (long long)c.dups;
        r.exact = (long long)c.exact_boxes;
        r.hs_on = (long long)c.hs_on;
        r.width = width;
        r.elapsed = (double)(now - s0.t_round_ns) * 1e-9;
        stats[s0.round_no - 1] = r;
        DevState s = s0;
        s.t_round_ns = now;
        s.n_cur = after;
        s.nrounds = s0.round_no;
        if (pingpong) {  // the round's frontier is in the other buffer; fresh dedup table
            s.cur ^= 1;
            s.epoch += 1;
        }
        if (after == 0) {
            s.done = 1;
            s.status = 0;  // no_real_solution
        } else if (width <= s0.target) {
            s.done = 1;
            s.status = 1;  // width_reached
        } else if ((long long)after > s0.max_boxes || s0.round_no >= s0.max_rounds) {
            s.done = 1;
            s.status = 2;  // budget_exhausted
        } else {
            s.round_no += 1;
            if ((after << n) > (unsigned long long)s_cap) s.bail = 1;  // next round needs the host
        }
        *st = s;
        cont = !(s.done || s.bail);
    }
    return __shfl_sync(0xffffffffu, cont, 0) != 0;
}

// Graph-mode round tail: exact-dedup compaction (when k_dedup_insert found
// duplicates) or plain copy of the round's frontier F[1] -> F[0], hash-table
// cleanup, and -- in the last block to finish -- the round end.  One kernel
// instead of dedup-finish + settle + round-end.
template <int N>
__global__ void __launch_bounds__(256) k_round_tail(Front f1, Front f0, unsigned* table, const unsigned* slot_of,
                                                    const uint8_t* dead, int dedup, DevState* st, Counters* ctr,
                                                    DevRoundStats* stats, int64_t s_cap,
                                                    cudaGraphConditionalHandle h_while, int* eq_order,
                                                    TabMeta meta) {
    pdl_enter();
    __shared__ int s_last;
    if (st->done || st->bail) return;  // unrolled round after the end of the device loop
    const int64_t n = (int64_t)ctr->n_next;
    const bool compact = dedup && ctr->dups != 0;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        if (dedup && i < n && slot_of[i] != 0xffffffffu) table[slot_of[i]] = 0u;
        const bool live = i < n && !(compact && dead[i]);
        const unsigned long long slot = compact ? warp_append(live, &ctr->n_compact) : (unsigned long long)i;
        if (live) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                f0.lo[j * f0.cap + slot] = f1.lo[j * f1.cap + i];
                f0.hi[j * f0.cap + slot] = f1.hi[j * f1.cap + i];
            }
            f0.cert[slot] = f1.cert[i];
            f0.unsplit[slot] = f1.unsplit[i];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&ctr->tail_done, 1ull) == (unsigned long long)(gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || threadIdx.x >= 32) return;
    __threadfence();
    const bool cont = round_end_warp(st, ctr, stats, N, s_cap, eq_order, meta, false);
    if (threadIdx.x == 0) RB_SET_COND(h_while, cont ? 1u : 0u);
}

// ------------------------------------------------------------------ persistent small rounds
//
// k_small_rounds runs whole rounds inside ONE resident grid while they are small
// (n_cur * 2^n children <= mk_cap): classify, filter, fused HS, dedup and the round
// end are the bodies of the per-phase kernels, separated by grid barriers instead
// of kernel boundaries, and the frontier ping-pongs between F[0] and F[1] with no
// copy.  Rounds are latency-bound at these sizes; a kernel boundary (~2 us launch
// + drain, plus table reloads) costs more than the phase itself.  Launched
// cooperatively, so every block is resident and the barrier cannot deadlock.

struct SmallArgs {
    TabMeta meta;
    const uint8_t* gtab;
    Front f0, f1;
    SBuf S;
    uint32_t* parents;
    Counters* ctr;
    DevState* st;
    DevRoundStats* rstats;
    int* order;
    unsigned* table;
    unsigned long long table_mask;
    unsigned* slot_of;
    uint8_t* dead;
    HsParams prm;
    unsigned* bar;               // {arrivals, generation}
    long long mk_cap;            // run rounds here while n_cur << n <= mk_cap
    long long graph_cap;         // then the WHILE loop while n_cur << n <= graph_cap
    cudaGraphConditionalHandle h_while;
    int dedup;                   // SolverConfig exact round dedup
    unsigned long long* trace;   // RB_TRACE: phase timestamps [round][phase] (block 0)
};

__device__ __forceinline__ void mk_stamp(const SmallArgs& a, int round, int phase) {
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && round >= 0 && round < 256) a.trace[round * 8 + phase] = gtimer();
}

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

template <int N>
__global__ void __launch_bounds__(256) k_small_rounds(SmallArgs a) {
    const volatile DevState* vs = a.st;
    for (;;) {
        if (vs->done || (((unsigned long long)vs->n_cur) << N) > (unsigned long long)a.mk_cap) break;
        const int cur = vs->cur;
        const int rno = vs->round_no;
        const Front fc = cur ? a.f1 : a.f0, fn = cur ? a.f0 : a.f1;
        mk_stamp(a, rno, 0);
        k_classify_body<N>(a.meta, fc, 0, fn, a.parents, a.ctr, 0.0, a.st);
        grid_barrier(a.bar);
        mk_stamp(a, rno, 1);
        k_filter_body<N>(a.meta, a.gtab, fc, a.parents, a.ctr, a.S, nullptr, a.order);
        grid_barrier(a.bar);
        mk_stamp(a, rno, 2);
        HsParams p = a.prm;
        p.count_from_ctr = 1;
        p.st = a.st;
        p.fused_max = LLONG_MAX;
        p.has_cond = 0;
        k_hs_fused_body<N>(a.meta, a.gtab, a.S, 0, p, fn, a.ctr, nullptr);
        grid_barrier(a.bar);
        mk_stamp(a, rno, 3);
        if (a.dedup) {
            k_dedup_insert_body<N>(fn, a.table, a.table_mask, a.slot_of, a.dead, a.ctr, a.S.cap);
            grid_barrier(a.bar);
            k_dedup_finish_body<N>(fn, fc, a.table, a.slot_of, a.dead, a.ctr, a.S.cap);
            grid_barrier(a.bar);
        }
        mk_stamp(a, rno, 4);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const bool dups = a.ctr->dups != 0;  // k_dedup_finish compacted back into fc
            round_end_body(a.st, a.ctr, a.rstats, N, a.mk_cap, a.order, a.meta);
            a.st->cur = dups ? cur : cur ^ 1;
            a.st->bail = 0;  // the size test is at the loop head
        }
        mk_stamp(a, rno, 5);
        grid_barrier(a.bar);
        mk_stamp(a, rno, 6);
    }
    // leave the frontier in F[0] (the WHILE loop and the host expect it there)
    if (vs->cur) {
        const long long n = (long long)vs->n_cur;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x) {
#pragma unroll
            for (int j = 0; j < N; j++) {
                a.f0.lo[j * a.f0.cap + i] = a.f1.lo[j * a.f1.cap + i];
                a.f0.hi[j * a.f0.cap + i] = a.f1.hi[j * a.f1.cap + i];
            }
            a.f0.cert[i] = a.f1.cert[i];
            a.f0.unsplit[i] = a.f1.unsplit[i];
        }
        grid_barrier(a.bar);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        DevState* st = a.st;
        st->cur = 0;
        const bool cont = !st->done && ((st->n_cur << N) <= (unsigned long long)a.graph_cap);
        st->bail = (!st->done && !cont) ? 1 : 0;
        RB_SET_COND(a.h_while, cont ? 1u : 0u);
    }
}

// ------------------------------------------------------------------ sharding

// Owner rank of a row = row_hash % world (the same function is restated in
// paper_1802_00330_b200/dist.py).  Routing every row to its owner each round keeps
// exact duplicates on one shard, so per-shard dedup is global dedup.
template <int N>
__global__ void k_owner_count(Front f, int64_t n, int world, unsigned* owner, unsigned long long* counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned o = (unsigned)(row_hash<N>(f, i) % (unsigned long long)world);
        owner[i] = o;
        atomicAdd(&counts[o], 1ull);
    }
}

template <int N>
__global__ void k_owner_scatter(Front src, int64_t n, const unsigned* owner, unsigned long long* cursor, Front dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long slot = atomicAdd(&cursor[owner[i]], 1ull);
#pragma unroll
        for (int j = 0; j < N; j++) {
            dst.lo[j * dst.cap + slot] = src.lo[j * src.cap + i];
            dst.hi[j * dst.cap + slot] = src.hi[j * src.cap + i];
        }
        dst.cert[slot] = src.cert[i];
        dst.unsplit[slot] = src.unsplit[i];
    }
}

// Frontier routing between shards.  Only a row with a component at
// most kThinUlps wide can have an exact duplicate elsewhere (see kThinUlps above), so
// only thin rows go to their hash owner; every other row stays, except the surplus
// rows the rebalancing plan moves (any non-thin row will do: the round's results do
// not depend on where a row is processed).
//   pass 1 (k_route_count): dest[i] = hash owner for thin rows, 0xffffffff otherwise;
//           thin rows counted per owner, non-thin rows counted
//   pass 2 (k_route_assign): non-thin rows take a surplus slot t (atomic) while
//           t < move_total; slot t goes to the destination d with
//           move_off[d] <= t < move_off[d + 1]; the rest stay on `rank`; rows counted
//           per destination
//   then k_owner_scatter into [own rows | rows for rank 0 | rank 1 | ...]
template <int N>
__global__ void k_route_count(Front f, int64_t n, int world, unsigned* dest, unsigned long long* counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        bool thin = false;
#pragma unroll
        for (int j = 0; j < N; j++) thin = thin || thin_comp(f.lo[j * f.cap + i], f.hi[j * f.cap + i]);
        unsigned d = 0xffffffffu;
        if (thin) {
            d = (unsigned)(row_hash<N>(f, i) % (unsigned long long)world);
            atomicAdd(&counts[d], 1ull);
        } else {
            atomicAdd(&counts[world], 1ull);
        }
        dest[i] = d;
    }
}

static __global__ void k_route_assign(int64_t n, int world, int rank, unsigned* dest, const unsigned long long* move_off,
                               unsigned long long* taken, unsigned long long* counts) {
    const unsigned long long total = move_off[world];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned d = dest[i];
        if (d == 0xffffffffu) {
            d = (unsigned)rank;
            if (total) {
                const unsigned long long t = atomicAdd(taken, 1ull);
                if (t < total) {
                    int k = 0;
                    while (k + 1 < world && move_off[k + 1] <= t) k++;
                    d = (unsigned)k;
                }
            }
            dest[i] = d;
        }
        atomicAdd(&counts[d], 1ull);
    }
}

// max RN width over rows (bnb.py:329)
template <int N>
__global__ void k_width(Front f, int64_t n, Counters* ctr) {
    unsigned long long wb = 0;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        if (i < n) {
            double w = 0.0;
#pragma unroll
            for (int j = 0; j < N; j++) {
                const double d = __dsub_rn(f.hi[j * f.cap + i], f.lo[j * f.cap + i]);
                w = j == 0 ? d : (d > w ? d : w);
            }
            const unsigned long long b = (unsigned long long)__double_as_longlong(w);
            wb = b > wb ? b : wb;
        }
    }
    wb = warp_max(wb);
    if ((threadIdx.x & 31) == 0 && wb) atomicMax(&ctr->wmax, wb);
}

// ------------------------------------------------------------------ canonical order

__device__ __forceinline__ unsigned long long order_key(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(canon0(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// key k of row perm[i]: k < n -> lo_k, else hi_{k-n}  (np.lexsort key order, _batch.py:247-249)
#ifndef RB_KINST_TU
__global__ void k_sort_keys(Front f, int n, int64_t N, int k, const unsigned* perm, unsigned long long* keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = perm ? perm[i] : i;
        const double v = k < n ? f.lo[k * f.cap + r] : f.hi[(k - n) * f.cap + r];
        keys[i] = order_key(v);
    }
}
#endif

#ifndef RB_KINST_TU
__global__ void k_iota(unsigned* p, int64_t N) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (unsigned)i;
}
#endif

// gather rows in perm order into row-major outputs
#ifndef RB_KINST_TU
__global__ void k_gather_rows(Front f, int n, int64_t N, const unsigned* perm, double* olo, double* ohi,
                              uint8_t* ocert, uint8_t* ouns) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = perm ? perm[i] : i;
        for (int j = 0; j < n; j++) {
            olo[i * n + j] = canon0(f.lo[j * f.cap + r]);
            ohi[i * n + j] = canon0(f.hi[j * f.cap + r]);
        }
        ocert[i] = f.cert[r];
        ouns[i] = f.unsplit[r];
    }
}
#endif

// ------------------------------------------------------------------ graph prologue / epilogue
//
// A small solve is one graph launch: k_solve_start -> WHILE(rounds) -> k_solve_finish,
// with the host reading everything back from mapped pinned memory after one sync.

struct InitBox {
    double lo[MAX_N], hi[MAX_N];
};

struct HostX {                  // pinned, mapped host memory shared with the graph
    DevState start;             // host -> device: the state the solve starts from
    DevState state;             // device -> host: state after the device rounds
    int order[16];              // device -> host: filter equation order
    long long rows;             // device -> host: rows gathered (-1: none)
    unsigned long long done_seq;// device -> host: start.seq once everything above is visible
};

// initial frontier = the initial box (bnb.py:229-232), device state, counters, filter order
#ifndef RB_KINST_TU
__global__ void k_solve_start(DevState* st, const HostX* hx, Front f0, Counters* ctr, int* order, InitBox box,
                              int n) {
    pdl_enter();
    const int t = threadIdx.x;
    if (t == 0) {
        DevState s = hx->start;
        s.t_round_ns = gtimer();
        s.round0 = s.round_no;
        *st = s;
    }
    if (t < n) {
        f0.lo[t * f0.cap] = box.lo[t];
        f0.hi[t * f0.cap] = box.hi[t];
    }
    if (t == 0) {
        f0.cert[0] = 0;
        f0.unsplit[0] = 0;
    }
    if (t < 16) order[t] = t;
    unsigned long long* w = reinterpret_cast<unsigned long long*>(ctr);
    for (int i = t; i < (int)(sizeof(Counters) / 8); i += blockDim.x) w[i] = 0ull;
}
#endif

// WHILE condition of the ping-pong round graph, once per loop iteration
#ifndef RB_KINST_TU
__global__ void k_set_cond(const DevState* st, cudaGraphConditionalHandle h_while) {
    pdl_enter();
    if (threadIdx.x == 0) cudaGraphSetConditional(h_while, (st->done || st->bail) ? 0u : 1u);
}
#endif

// final state, round statistics and order to the host; when the solve finished on the
// device with at most max_rows boxes, also the boxes (row-major, unsorted)
#ifndef RB_KINST_TU
__global__ void k_solve_finish(const DevState* st, const DevRoundStats* rs, const int* order, HostX* hx,
                               DevRoundStats* hstats, Front fa, Front fb, int n, long long max_rows, double* hlo,
                               double* hhi, uint8_t* hc, uint8_t* hu) {
    pdl_enter();
    const DevState s = *st;
    const Front f0 = s.cur ? fb : fa;  // frontier in F[cur]
    const long long N = (long long)s.n_cur;
    const bool gather = s.done && N <= max_rows;
    // only the blocks with rows to gather take part (block 0 always: state + statistics);
    // the rest leave at once instead of each fencing and counting itself
    const long long rows = gather ? N : 0;
    const unsigned active = (unsigned)max(1ll, min((long long)gridDim.x, (rows + blockDim.x - 1) / blockDim.x));
    if (blockIdx.x >= active) return;
    if (blockIdx.x == 0) {
        const int first = s.round0 - 1;  // device copy: no PCIe read of hx->start
        for (int r = first + (int)threadIdx.x; r < s.nrounds; r += blockDim.x) hstats[r] = rs[r];
        if (threadIdx.x < 16) hx->order[threadIdx.x] = order[threadIdx.x];
        if (threadIdx.x == 0) {
            hx->state = s;
            hx->rows = gather ? N : -1;
        }
    }
    if (gather) {
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
             i += (long long)active * blockDim.x) {
            for (int j = 0; j < n; j++) {
                hlo[i * n + j] = canon0(f0.lo[j * f0.cap + i]);
                hhi[i * n + j] = canon0(f0.hi[j * f0.cap + i]);
            }
            hc[i] = f0.cert[i];
            hu[i] = f0.unsplit[i];
        }
    }
    // completion flag in mapped memory: every block's host writes are fenced before it
    // counts itself; the last block publishes the sequence number, so a host spinning on
    // done_seq may read the results without waiting for the stream (rb_solve fast return)
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&const_cast<DevState*>(st)->finish_blocks, 1u);
        if (prev == active - 1) {
            __threadfence_system();
            *reinterpret_cast<volatile unsigned long long*>(&hx->done_seq) = s.seq;
        }
    }
}
#endif

// row-major (host layout) -> SoA frontier rows [off, off+N)
#ifndef RB_KINST_TU
__global__ void k_rows_to_soa(const double* rlo, const double* rhi, const uint8_t* rc, const uint8_t* ru, int n,
                              int64_t N, Front f, int64_t off) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        for (int j = 0; j < n; j++) {
            f.lo[j * f.cap + off + i] = rlo[i * n + j];
            f.hi[j * f.cap + off + i] = rhi[i * n + j];
        }
        if (f.cert) f.cert[off + i] = rc ? rc[i] : 0;
        if (f.unsplit) f.unsplit[off + i] = ru ? ru[i] : 0;
    }
}
#endif

}  // namespace rb
