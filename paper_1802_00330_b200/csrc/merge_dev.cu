// merge_dev.cu -- the backtracking merge on the device:
// snap_to_grid + merge_to_width of rootbox/backtrack.py:118-242 as exact integer
// arithmetic on (level, index) keys, with parent index halving and sort-unique per
// level on the GPU.
//
// Fast path (everything else returns RB_ERR_LIMIT and the caller runs the host merge,
// rb_merge in merge.cpp, which handles every case the reference handles):
//   * every initial width hi_i - lo_i is a power of two 2^w_i (every BASELINE config and
//     every corpus system), so a level-L cell width is 2^(w_i - L) and every division of
//     snap_to_grid is a shift;
//   * the box endpoints, scaled by 2^S_i (S_i = the finest binary digit in use), fit 120-bit
//     integers, and every snapped level is at most 53 (cell index times cell width is then
//     an exact double product; eps 1e-8 on a width-4 box is level ~29).
// Snapping is thread per box in __int128 (the steps of snap_fast in merge.cpp); a merge
// level is: keys (L, k_0..k_{n-1}) sorted by LSD radix passes, exact duplicates merged with
// their flags OR-ed, cells absorbed by a coarser cell dropped with their flag OR-ed into the
// coarsest one (_drop_nested, backtrack.py:168-191), then every key halved (parent cells).
// Output cells are materialised with outward rounding (_float_down / _float_up,
// backtrack.py:40-51: RD / RU of the exact a + k 2^(w-L)) and put in Box.sort_key order.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rootbox_b200.h"

namespace {

using i128 = __int128;
using u128 = unsigned __int128;

constexpr int kMaxDim = 16;
constexpr int kMaxLevel = 53;

struct MGrid {
    int n;
    double a[kMaxDim];   // anchors (initial lower bounds)
    int w[kMaxDim];      // initial width = 2^w
    int S[kMaxDim];      // scale: every value * 2^S is an integer
};

__device__ __forceinline__ int low_exp_dev(double x) {  // exponent of the lowest set bit of a finite x != 0
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const int e = (int)((b >> 52) & 0x7ff);
    unsigned long long m = b & 0xfffffffffffffull;
    int ex;
    if (e) {
        m |= 1ull << 52;
        ex = e - 1075;
    } else {
        ex = -1074;
    }
    return ex + __ffsll((long long)m) - 1;
}

__global__ void k_merge_scale(int n, int64_t N, const double* lo, const double* hi, int* smax) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N * n; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % n);
        int s = INT_MIN;
        const double a = lo[t], b = hi[t];
        if (a != 0.0 && isfinite(a)) s = max(s, -low_exp_dev(a));
        if (b != 0.0 && isfinite(b)) s = max(s, -low_exp_dev(b));
        if (s != INT_MIN) atomicMax(&smax[i], s);
    }
}

__device__ __forceinline__ bool scaled(double x, int S, i128& out) {  // x * 2^S exactly (S >= -low_exp(x))
    if (x == 0.0) {
        out = 0;
        return true;
    }
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const int e = (int)((b >> 52) & 0x7ff);
    unsigned long long m = b & 0xfffffffffffffull;
    int ex;
    if (e) {
        m |= 1ull << 52;
        ex = e - 1075;
    } else {
        ex = -1074;
    }
    const int sh = ex + S;  // x * 2^S = m * 2^sh
    if (sh < 0) {
        if (-sh >= 64 || (m & ((1ull << -sh) - 1))) return false;
        out = (i128)(m >> -sh);
    } else {
        if (sh > 66) return false;
        out = (i128)m << sh;
    }
    if (x < 0) out = -out;
    return true;
}

__device__ __forceinline__ int bitlen128(u128 v) {
    const unsigned long long h = (unsigned long long)(v >> 64);
    return h ? 128 - __clzll((long long)h) : 64 - __clzll((long long)(unsigned long long)v);
}

// exactly representable as a double: <= 53 significant bits, normal range
__device__ __forceinline__ bool exact_dbl(i128 v, int S2) {
    if (v == 0) return true;
    u128 m = v < 0 ? (u128)(-v) : (u128)v;
    int tz = 0;
    while (!(m & 1)) {
        m >>= 1;
        tz++;
    }
    const int top = bitlen128(m) + tz - 1 - S2;  // exponent of the leading bit
    return bitlen128(m) <= 53 && top > -1022 && top < 1023;
}

// snap_to_grid (backtrack.py:118-158) of box r: level + indices, or a failure code
// (1 = leave the fast path: the host merge decides, including the reference's errors)
__global__ void k_merge_snap(MGrid g, int64_t N, const double* lo, const double* hi, int* lev,
                             unsigned long long* key, int* fail) {
    const int n = g.n;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        i128 dlo[kMaxDim], dhi[kMaxDim];
        int level = -1;
        bool bad = false;
        for (int i = 0; i < n && !bad; i++) {
            i128 A, xl, xh;
            if (!scaled(g.a[i], g.S[i], A) || !scaled(lo[r * n + i], g.S[i], xl) || !scaled(hi[r * n + i], g.S[i], xh)) {
                bad = true;
                break;
            }
            const int wS = g.w[i] + g.S[i];
            dlo[i] = xl - A;
            dhi[i] = xh - A;
            if (dlo[i] < 0 || dhi[i] > ((i128)1 << wS) || dhi[i] < dlo[i]) {
                bad = true;
                break;
            }
            const i128 wd = dhi[i] - dlo[i];
            if (wd == 0) continue;
            // li = bitlen(floor(2^wS / wd)) - 1
            const int b = bitlen128((u128)wd);
            const bool pow2 = (wd & (wd - 1)) == 0;
            const int li = pow2 ? wS - b + 1 : wS - b;
            level = level < 0 ? li : min(level, li);
        }
        if (bad) {
            atomicOr(fail, 1);
            continue;
        }
        if (level < 0) level = 52;  // a point box: snap to a deep cell
        if (level > kMaxLevel) {
            atomicOr(fail, 1);
            continue;
        }
        int L = level;
        unsigned long long idx[kMaxDim];
        for (; L > 0; L--) {
            bool ok = true;
            for (int i = 0; i < n && ok; i++) {
                const int sh = g.w[i] + g.S[i] - L;  // cell width 2^sh (scaled)
                u128 k = (u128)(dlo[i] >> sh);
                const u128 kmax = ((u128)1 << L) - 1;
                if (k > kmax) k = kmax;
                if (dhi[i] > (i128)((k + 1) << sh)) ok = false;  // straddles the cell boundary
                idx[i] = (unsigned long long)k;
            }
            if (ok) break;
        }
        if (L == 0)
            for (int i = 0; i < n; i++) idx[i] = 0;
        // the snapped cell's bounds must be exact (merge_to_width locates it again, backtrack.py:219)
        for (int i = 0; i < n && !bad; i++) {
            i128 A;
            scaled(g.a[i], g.S[i], A);
            const int sh = g.w[i] + g.S[i] - L;
            const i128 nlo = A + ((i128)idx[i] << sh), nhi = nlo + ((i128)1 << sh);
            if (!exact_dbl(nlo, g.S[i]) || !exact_dbl(nhi, g.S[i])) bad = true;
        }
        if (bad) {
            atomicOr(fail, 1);
            continue;
        }
        lev[r] = L;
        for (int i = 0; i < n; i++) key[(int64_t)i * N + r] = idx[i];
    }
}

__global__ void k_iota_u32(unsigned* p, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (unsigned)i;
}

// sort key of pass `pass` for the rows in permutation order: pass < n -> component n-1-pass... the
// caller chooses the component; level passes use lev
__global__ void k_gather_key(const unsigned long long* src, const unsigned* perm, int64_t M,
                             unsigned long long* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = src[perm[i]];
}
__global__ void k_gather_lev(const int* src, const unsigned* perm, int64_t M, unsigned long long* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (unsigned long long)src[perm[i]];
}

// rows in sorted order -> (lev, key, flag) arrays; heads[j] = row j differs from row j - 1
__global__ void k_apply_perm(int n, int64_t M, int64_t cap, const unsigned* perm, const int* lev,
                             const unsigned long long* key, const unsigned* flag, int* lev2,
                             unsigned long long* key2, unsigned* flag2) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        const unsigned p = perm[j];
        lev2[j] = lev[p];
        flag2[j] = flag[p];
        for (int i = 0; i < n; i++) key2[(int64_t)i * cap + j] = key[(int64_t)i * cap + p];
    }
}

__global__ void k_heads(int n, int64_t M, int64_t cap, const int* lev, const unsigned long long* key, unsigned* head) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        bool h = j == 0 || lev[j] != lev[j - 1];
        for (int i = 0; i < n && !h; i++) h = key[(int64_t)i * cap + j] != key[(int64_t)i * cap + j - 1];
        head[j] = h ? 1u : 0u;
    }
}

// unique: row j goes to pos[j] - 1 (pos = inclusive scan of heads), flags OR-ed per run
__global__ void k_unique(int n, int64_t M, int64_t cap, const unsigned* pos, const unsigned* head, const int* lev,
                         const unsigned long long* key, const unsigned* flag, int* lev2, unsigned long long* key2,
                         unsigned* flag2) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        const unsigned d = pos[j] - 1;
        if (head[j]) {
            lev2[d] = lev[j];
            for (int i = 0; i < n; i++) key2[(int64_t)i * cap + d] = key[(int64_t)i * cap + j];
        }
        if (flag[j]) atomicOr(&flag2[d], 1u);
    }
}

// _drop_nested: a cell with an ancestor among the coarser cells is absorbed by the coarsest
// one (it is kept: nothing coarser contains it), its flag OR-ed into that ancestor
__global__ void k_drop_nested(int n, int64_t M, int64_t cap, const int* lev, const unsigned long long* key,
                              unsigned* flag, const int* seg, int lmin, unsigned* keep) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        const int L = lev[j];
        bool absorbed = false;
        for (int L2 = lmin; L2 < L && !absorbed; L2++) {
            int lo = seg[L2], hi = seg[L2 + 1] - 1;
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                int c = 0;
                for (int i = 0; i < n && c == 0; i++) {
                    const unsigned long long a = key[(int64_t)i * cap + mid], b = key[(int64_t)i * cap + j] >> (L - L2);
                    c = a < b ? -1 : (a > b ? 1 : 0);
                }
                if (c == 0) {
                    if (flag[j]) atomicOr(&flag[mid], 1u);
                    absorbed = true;
                    break;
                }
                if (c < 0) lo = mid + 1;
                else hi = mid - 1;
            }
        }
        keep[j] = absorbed ? 0u : 1u;
    }
}

__global__ void k_compact(int n, int64_t M, int64_t cap, const unsigned* pos, const unsigned* keep, const int* lev,
                          const unsigned long long* key, const unsigned* flag, int* lev2, unsigned long long* key2,
                          unsigned* flag2) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        if (!keep[j]) continue;
        const unsigned d = pos[j] - 1;
        lev2[d] = lev[j];
        flag2[d] = flag[j];
        for (int i = 0; i < n; i++) key2[(int64_t)i * cap + d] = key[(int64_t)i * cap + j];
    }
}

__global__ void k_parents(int n, int64_t M, int64_t cap, int* lev, unsigned long long* key) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        lev[j] -= 1;
        for (int i = 0; i < n; i++) key[(int64_t)i * cap + j] >>= 1;
    }
}

__global__ void k_level_hist(int64_t M, const int* lev, int* hist) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[lev[j]], 1);
}

// cell bounds: RD(a + k 2^(w-L)), RU(a + (k+1) 2^(w-L)) (exact products: k < 2^53)
__global__ void k_materialize(MGrid g, int64_t M, int64_t cap, const int* lev, const unsigned long long* key,
                              double* blo, double* bhi) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        const int L = lev[j];
        for (int i = 0; i < g.n; i++) {
            const double cw = ldexp(1.0, g.w[i] - L);
            const unsigned long long k = key[(int64_t)i * cap + j];
            blo[(int64_t)i * cap + j] = __dadd_rd(g.a[i], (double)k * cw);
            bhi[(int64_t)i * cap + j] = __dadd_ru(g.a[i], (double)(k + 1) * cw);
        }
    }
}

__global__ void k_order_keys(const double* v, const unsigned* perm, int64_t M, unsigned long long* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long b = (unsigned long long)__double_as_longlong(__dadd_rn(v[perm[i]], 0.0));
        out[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    }
}

__global__ void k_out_rows(int n, int64_t M, int64_t cap, const unsigned* perm, const double* blo, const double* bhi,
                           const unsigned* flag, double* olo, double* ohi, uint8_t* oc) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < M; r += (int64_t)gridDim.x * blockDim.x) {
        const unsigned p = perm[r];
        for (int i = 0; i < n; i++) {
            olo[r * n + i] = blo[(int64_t)i * cap + p];
            ohi[r * n + i] = bhi[(int64_t)i * cap + p];
        }
        oc[r] = flag[p] ? 1 : 0;
    }
}

struct Fail {
    int code;
    std::string msg;
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Fail{RB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t c) {
        if (p) cudaFree(p);
        p = nullptr;
        n = std::max<size_t>(c, 1);
        ck(cudaMalloc(&p, n * sizeof(T)), "device merge alloc");
    }
    ~DBuf() {
        if (p) cudaFree(p);
    }
};

int grid(int64_t work) { return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 16)); }

}  // namespace

extern "C" int rb_merge_device(int device, int n, const double* init_lo, const double* init_hi, const double* lo,
                               const double* hi, const uint8_t* cert, int64_t N, double stop_width,
                               int stop_on_plateau, double* out_lo, double* out_hi, uint8_t* out_cert, int64_t cap,
                               int64_t* Mout, double* levels, int64_t cap_levels, int64_t* K, char* err,
                               int64_t err_len) {
    auto say = [&](int code, const std::string& m) {
        if (err && err_len > 0) {
            std::strncpy(err, m.c_str(), (size_t)err_len - 1);
            err[err_len - 1] = 0;
        }
        return code;
    };
    if (n < 1 || n > kMaxDim || N < 0 || !Mout || !K) return say(RB_ERR_ARG, "bad arguments");
    MGrid g{};
    g.n = n;
    for (int i = 0; i < n; i++) {
        const double W = init_hi[i] - init_lo[i];
        int e = 0;
        const double m = std::frexp(W, &e);
        if (!(W > 0) || m != 0.5 || init_lo[i] + W != init_hi[i] || init_hi[i] - W != init_lo[i])
            return say(RB_ERR_LIMIT, "device merge: an initial width is not a power of two (host merge)");
        g.a[i] = init_lo[i];
        g.w[i] = e - 1;
    }
    if (N == 0) {
        *Mout = 0;
        *K = 1;
        if (cap_levels > 0) {
            levels[0] = 0.0;
            levels[1] = 0.0;
        }
        return RB_OK;
    }
    try {
        ck(cudaSetDevice(device), "cudaSetDevice");
        const int64_t C = N;
        DBuf<double> dlo, dhi;
        dlo.alloc((size_t)N * n);
        dhi.alloc((size_t)N * n);
        ck(cudaMemcpy(dlo.p, lo, sizeof(double) * N * n, cudaMemcpyHostToDevice), "h2d");
        ck(cudaMemcpy(dhi.p, hi, sizeof(double) * N * n, cudaMemcpyHostToDevice), "h2d");
        // scale S_i: every value (and the anchor) * 2^S_i is an integer
        DBuf<int> smax;
        smax.alloc(kMaxDim);
        std::vector<int> hs(kMaxDim, INT_MIN);
        ck(cudaMemcpy(smax.p, hs.data(), sizeof(int) * kMaxDim, cudaMemcpyHostToDevice), "h2d");
        k_merge_scale<<<grid(N * n), 256>>>(n, N, dlo.p, dhi.p, smax.p);
        ck(cudaMemcpy(hs.data(), smax.p, sizeof(int) * kMaxDim, cudaMemcpyDeviceToHost), "d2h");
        for (int i = 0; i < n; i++) {
            int s = hs[i] == INT_MIN ? 0 : hs[i];
            for (double v : {init_lo[i], init_hi[i]})
                if (v != 0.0) {
                    int e;
                    const double mm = std::frexp(std::fabs(v), &e);
                    const uint64_t mi = (uint64_t)std::ldexp(mm, 53);
                    s = std::max(s, -(e - 53 + __builtin_ctzll(mi)));
                }
            // at least 54 - w_i so that a cell width 2^(w_i - L), L <= 53, is an integer once scaled
            g.S[i] = std::max({s, 0, 54 - g.w[i]});
            double amax = std::max(std::fabs(init_lo[i]), std::fabs(init_hi[i]));
            int ea;
            std::frexp(amax, &ea);
            if (ea + g.S[i] + 2 > 118 || g.w[i] + g.S[i] > 118)
                return say(RB_ERR_LIMIT, "device merge: endpoints need more than 120-bit integers (host merge)");
        }
        // snap
        DBuf<int> lev, lev2, fail;
        DBuf<unsigned long long> key, key2, skey0, skey1;
        DBuf<unsigned> flag, flag2, perm0, perm1, head, pos;
        lev.alloc(C);
        lev2.alloc(C);
        key.alloc((size_t)C * n);
        key2.alloc((size_t)C * n);
        flag.alloc(C);
        flag2.alloc(C);
        perm0.alloc(C);
        perm1.alloc(C);
        skey0.alloc(C);
        skey1.alloc(C);
        head.alloc(C);
        pos.alloc(C);
        fail.alloc(1);
        ck(cudaMemset(fail.p, 0, sizeof(int)), "memset");
        k_merge_snap<<<grid(N), 128>>>(g, N, dlo.p, dhi.p, lev.p, key.p, fail.p);
        int hfail = 0;
        ck(cudaMemcpy(&hfail, fail.p, sizeof(int), cudaMemcpyDeviceToHost), "d2h");
        if (hfail)
            return say(RB_ERR_LIMIT, "device merge: a box leaves the fast path (level > 53, inexact cell or "
                                     "outside the grid; host merge)");
        {
            std::vector<unsigned> hf(N);
            for (int64_t r = 0; r < N; r++) hf[r] = cert && cert[r] ? 1u : 0u;
            ck(cudaMemcpy(flag.p, hf.data(), sizeof(unsigned) * N, cudaMemcpyHostToDevice), "h2d");
        }
        // the key arrays use stride C (= N): cell count only shrinks
        size_t tmp_bytes = 0, scan_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, skey0.p, skey1.p, perm0.p, perm1.p, (int)C);
        cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, head.p, pos.p, (int)C);
        DBuf<uint8_t> tmp;
        tmp.alloc(std::max(tmp_bytes, scan_bytes));
        DBuf<int> hist;
        hist.alloc(kMaxLevel + 2);
        int64_t M = N;
        std::vector<int> hh(kMaxLevel + 2);

        // sort (L, k_0 .. k_{n-1}) ascending, merge exact duplicates (flag OR), drop nested cells
        auto normalize = [&]() {
            ck(cudaMemset(hist.p, 0, sizeof(int) * (kMaxLevel + 2)), "memset");
            k_iota_u32<<<grid(M), 256>>>(perm0.p, M);
            unsigned* pin = perm0.p;
            unsigned* pout = perm1.p;
            for (int pass = n; pass >= 0; pass--) {  // LSD: k_{n-1} first, level last
                if (pass == 0) k_gather_lev<<<grid(M), 256>>>(lev.p, pin, M, skey0.p);
                else k_gather_key<<<grid(M), 256>>>(key.p + (int64_t)(pass - 1) * C, pin, M, skey0.p);
                size_t b = tmp.n;
                ck(cub::DeviceRadixSort::SortPairs(tmp.p, b, skey0.p, skey1.p, pin, pout, (int)M), "radix");
                std::swap(pin, pout);
            }
            k_apply_perm<<<grid(M), 256>>>(n, M, C, pin, lev.p, key.p, flag.p, lev2.p, key2.p, flag2.p);
            k_heads<<<grid(M), 256>>>(n, M, C, lev2.p, key2.p, head.p);
            size_t b = tmp.n;
            ck(cub::DeviceScan::InclusiveSum(tmp.p, b, head.p, pos.p, (int)M), "scan");
            unsigned u = 0;
            ck(cudaMemcpy(&u, pos.p + (M - 1), sizeof(unsigned), cudaMemcpyDeviceToHost), "d2h");
            ck(cudaMemset(flag.p, 0, sizeof(unsigned) * M), "memset");
            k_unique<<<grid(M), 256>>>(n, M, C, pos.p, head.p, lev2.p, key2.p, flag2.p, lev.p, key.p, flag.p);
            M = (int64_t)u;
            // level segments (rows are sorted by level first)
            k_level_hist<<<grid(M), 256>>>(M, lev.p, hist.p);
            ck(cudaMemcpy(hh.data(), hist.p, sizeof(int) * (kMaxLevel + 2), cudaMemcpyDeviceToHost), "d2h");
            std::vector<int> seg(kMaxLevel + 3, 0);
            int lmin = -1, nlev = 0;
            for (int L = 0; L <= kMaxLevel; L++) {
                seg[L + 1] = seg[L] + hh[L];
                if (hh[L]) {
                    nlev++;
                    if (lmin < 0) lmin = L;
                }
            }
            if (nlev > 1) {
                DBuf<int> dseg;
                dseg.alloc(kMaxLevel + 3);
                ck(cudaMemcpy(dseg.p, seg.data(), sizeof(int) * (kMaxLevel + 3), cudaMemcpyHostToDevice), "h2d");
                k_drop_nested<<<grid(M), 256>>>(n, M, C, lev.p, key.p, flag.p, dseg.p, lmin, head.p);
                size_t b2 = tmp.n;
                ck(cub::DeviceScan::InclusiveSum(tmp.p, b2, head.p, pos.p, (int)M), "scan");
                ck(cudaMemcpy(&u, pos.p + (M - 1), sizeof(unsigned), cudaMemcpyDeviceToHost), "d2h");
                k_compact<<<grid(M), 256>>>(n, M, C, pos.p, head.p, lev.p, key.p, flag.p, lev2.p, key2.p, flag2.p);
                std::swap(lev.p, lev2.p);
                std::swap(key.p, key2.p);
                std::swap(flag.p, flag2.p);
                M = (int64_t)u;
                ck(cudaMemset(hist.p, 0, sizeof(int) * (kMaxLevel + 2)), "memset");
                k_level_hist<<<grid(M), 256>>>(M, lev.p, hist.p);
                ck(cudaMemcpy(hh.data(), hist.p, sizeof(int) * (kMaxLevel + 2), cudaMemcpyDeviceToHost), "d2h");
            }
        };
        // cur_width (backtrack.py:221-229): max over present levels and components of W_i / 2^L
        auto width_now = [&]() {
            int lmin = -1;
            for (int L = 0; L <= kMaxLevel; L++)
                if (hh[L]) {
                    lmin = L;
                    break;
                }
            if (lmin < 0 || M == 0) return 0.0;
            double w = 0.0;
            for (int i = 0; i < n; i++) w = std::max(w, std::ldexp(1.0, g.w[i] - lmin));
            return w;
        };
        normalize();
        std::vector<std::pair<double, int64_t>> log;
        log.push_back({width_now(), M});
        const bool has_stop = stop_width >= 0 && !std::isnan(stop_width);
        while (M > 0) {
            if (stop_on_plateau && log.size() >= 2 && log[log.size() - 1].second == log[log.size() - 2].second) break;
            if (has_stop && log.back().first >= stop_width) break;
            if (hh[0]) break;
            k_parents<<<grid(M), 256>>>(n, M, C, lev.p, key.p);
            normalize();
            log.push_back({width_now(), M});
        }
        // materialise (outward rounding) and order by Box.sort_key (lows, then highs)
        DBuf<double> blo, bhi;
        blo.alloc((size_t)C * n);
        bhi.alloc((size_t)C * n);
        k_materialize<<<grid(M), 256>>>(g, M, C, lev.p, key.p, blo.p, bhi.p);
        k_iota_u32<<<grid(M), 256>>>(perm0.p, M);
        unsigned* pin = perm0.p;
        unsigned* pout = perm1.p;
        for (int k = 2 * n - 1; k >= 0; k--) {
            const double* src = k >= n ? bhi.p + (int64_t)(k - n) * C : blo.p + (int64_t)k * C;
            k_order_keys<<<grid(M), 256>>>(src, pin, M, skey0.p);
            size_t b = tmp.n;
            if (M > 0) ck(cub::DeviceRadixSort::SortPairs(tmp.p, b, skey0.p, skey1.p, pin, pout, (int)M), "radix");
            std::swap(pin, pout);
        }
        *Mout = M;
        *K = (int64_t)log.size();
        for (int64_t r = 0; r < (int64_t)log.size() && r < cap_levels; r++) {
            levels[2 * r] = log[r].first;
            levels[2 * r + 1] = (double)log[r].second;
        }
        if (M <= cap && M > 0) {
            DBuf<double> olo, ohi;
            DBuf<uint8_t> oc;
            olo.alloc((size_t)M * n);
            ohi.alloc((size_t)M * n);
            oc.alloc(M);
            k_out_rows<<<grid(M), 256>>>(n, M, C, pin, blo.p, bhi.p, flag.p, olo.p, ohi.p, oc.p);
            ck(cudaMemcpy(out_lo, olo.p, sizeof(double) * M * n, cudaMemcpyDeviceToHost), "d2h");
            ck(cudaMemcpy(out_hi, ohi.p, sizeof(double) * M * n, cudaMemcpyDeviceToHost), "d2h");
            ck(cudaMemcpy(out_cert, oc.p, M, cudaMemcpyDeviceToHost), "d2h");
        }
        ck(cudaGetLastError(), "device merge");
        return RB_OK;
    } catch (const Fail& f) {
        cudaGetLastError();
        return say(f.code, f.msg);
    }
}
