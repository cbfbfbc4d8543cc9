// merge.cpp -- native backtracking merge.
//
// snap_to_grid + merge_to_width of rootbox/backtrack.py:118-242, exactly: every
// alignment decision in exact integer arithmetic.  The reference uses Python
// Fractions; all quantities here are dyadic rationals (doubles and the initial
// widths divided by powers of two), so each variable is scaled by 2^S_i to make
// every anchor, width and box endpoint an integer (Big below), and cell bounds
// are materialised with correctly rounded outward conversion (_float_down /
// _float_up, backtrack.py:40-51).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/rootbox_b200.h"

namespace {

// ---------------------------------------------------------------- minimal big integers

constexpr int LIMBS = 40;  // 2560 bits: every scaled double and product below fits

struct Big {
    uint64_t w[LIMBS];  // limbs >= n are undefined (never read)
    int n = 0;          // used limbs (w[n-1] != 0 unless n == 0)
    bool neg = false;
};

void norm(Big& a) {
    while (a.n > 0 && a.w[a.n - 1] == 0) a.n--;
    if (a.n == 0) a.neg = false;
}

Big from_u128(unsigned __int128 v) {
    Big a;
    a.w[0] = (uint64_t)v;
    a.w[1] = (uint64_t)(v >> 64);
    a.n = 2;
    norm(a);
    return a;
}

inline uint64_t limb(const Big& a, int i) { return i < a.n ? a.w[i] : 0ull; }

int cmp_mag(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; i--)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

Big add_mag(const Big& a, const Big& b) {
    Big r;
    const int n = std::max(a.n, b.n);
    unsigned __int128 c = 0;
    for (int i = 0; i < n; i++) {
        c += (unsigned __int128)limb(a, i) + limb(b, i);
        r.w[i] = (uint64_t)c;
        c >>= 64;
    }
    r.n = n;
    if (c) r.w[r.n++] = (uint64_t)c;
    return r;
}

Big sub_mag(const Big& a, const Big& b) {  // |a| >= |b|
    Big r;
    __int128 br = 0;
    for (int i = 0; i < a.n; i++) {
        __int128 d = (__int128)a.w[i] - limb(b, i) - br;
        br = d < 0;
        r.w[i] = (uint64_t)d;
    }
    r.n = a.n;
    norm(r);
    return r;
}

Big add(const Big& a, const Big& b) {
    Big r;
    if (a.neg == b.neg) {
        r = add_mag(a, b);
        r.neg = a.neg;
    } else if (cmp_mag(a, b) >= 0) {
        r = sub_mag(a, b);
        r.neg = a.neg;
    } else {
        r = sub_mag(b, a);
        r.neg = b.neg;
    }
    norm(r);
    return r;
}

Big neg(Big a) {
    if (a.n) a.neg = !a.neg;
    return a;
}

Big sub(const Big& a, const Big& b) { return add(a, neg(b)); }

int cmp(const Big& a, const Big& b) {
    if (a.neg != b.neg) return a.neg ? -1 : 1;
    const int m = cmp_mag(a, b);
    return a.neg ? -m : m;
}

int sign(const Big& a) { return a.n == 0 ? 0 : (a.neg ? -1 : 1); }

int bitlen(const Big& a) {
    if (a.n == 0) return 0;
    return 64 * (a.n - 1) + (64 - __builtin_clzll(a.w[a.n - 1]));
}

Big shl(const Big& a, int s) {
    Big r;
    if (a.n == 0) return r;
    const int q = s / 64, b = s % 64;
    if (a.n + q + 1 > LIMBS) throw std::string("integer too large");
    for (int i = 0; i < a.n + q + 1; i++) r.w[i] = 0;
    for (int i = 0; i < a.n; i++) {
        r.w[i + q] |= a.w[i] << b;
        if (b) r.w[i + q + 1] |= a.w[i] >> (64 - b);
    }
    r.n = a.n + q + 1;
    r.neg = a.neg;
    norm(r);
    return r;
}

Big shr_mag(const Big& a, int s) {  // floor(|a| / 2^s)
    Big r;
    const int q = s / 64, b = s % 64;
    for (int i = q; i < a.n; i++) {
        uint64_t v = a.w[i] >> b;
        if (b && i + 1 < a.n) v |= a.w[i + 1] << (64 - b);
        r.w[i - q] = v;
    }
    r.n = std::max(0, a.n - q);
    norm(r);
    return r;
}

bool low_bits_nonzero(const Big& a, int s) {  // any of the lowest s bits set
    const int q = s / 64, b = s % 64;
    for (int i = 0; i < q && i < a.n; i++)
        if (a.w[i]) return true;
    if (b && q < a.n && (a.w[q] & ((1ull << b) - 1))) return true;
    return false;
}

bool bit(const Big& a, int i) {
    const int q = i / 64;
    return q < a.n && ((a.w[q] >> (i % 64)) & 1);
}

Big mul_u128(const Big& a, unsigned __int128 m) {  // |a| * m, sign of a
    const Big mb = from_u128(m);
    Big r;
    const int rn = std::min(LIMBS, a.n + mb.n + 1);
    for (int i = 0; i < rn; i++) r.w[i] = 0;
    for (int i = 0; i < a.n; i++) {
        unsigned __int128 c = 0;
        for (int j = 0; j < mb.n; j++) {
            if (i + j >= LIMBS) throw std::string("integer too large");
            c += (unsigned __int128)a.w[i] * mb.w[j] + r.w[i + j];
            r.w[i + j] = (uint64_t)c;
            c >>= 64;
        }
        int k = i + mb.n;
        while (c) {
            if (k >= LIMBS) throw std::string("integer too large");
            c += r.w[k];
            r.w[k] = (uint64_t)c;
            c >>= 64;
            k++;
        }
    }
    r.n = std::min(LIMBS, a.n + mb.n + 1);
    r.neg = a.neg;
    norm(r);
    return r;
}

// floor(a / b) for a >= 0, b > 0 (binary long division; 128-bit fast path)
Big div_floor(const Big& a, const Big& b) {
    Big q;
    if (cmp_mag(a, b) < 0) return q;
    if (a.n <= 2) {
        const unsigned __int128 x = (unsigned __int128)limb(a, 0) | ((unsigned __int128)limb(a, 1) << 64);
        const unsigned __int128 y = (unsigned __int128)limb(b, 0) | ((unsigned __int128)limb(b, 1) << 64);
        return from_u128(x / y);
    }
    const int shift = bitlen(a) - bitlen(b);
    for (int i = 0; i <= shift / 64; i++) q.w[i] = 0;
    Big rem = a, d = shl(b, shift);
    for (int s = shift; s >= 0; s--) {
        if (cmp_mag(rem, d) >= 0) {
            rem = sub_mag(rem, d);
            q.w[s / 64] |= 1ull << (s % 64);
            q.n = std::max(q.n, s / 64 + 1);
        }
        d = shr_mag(d, 1);
    }
    norm(q);
    return q;
}

unsigned __int128 to_u128(const Big& a) {
    if (a.n > 2) throw std::string("cell index beyond 2^128");
    return (unsigned __int128)limb(a, 0) | ((unsigned __int128)limb(a, 1) << 64);
}

// lowest set bit exponent of a finite nonzero double
int low_exp(double x) {
    int e;
    double m = std::frexp(std::fabs(x), &e);  // x = m 2^e, m in [0.5, 1)
    uint64_t mi = (uint64_t)std::ldexp(m, 53);
    return e - 53 + __builtin_ctzll(mi);
}

// x * 2^S exactly (requires S >= -low_exp(x))
Big from_double(double x, int S) {
    Big r;
    if (x == 0.0) return r;
    int e;
    const double m = std::frexp(std::fabs(x), &e);
    uint64_t mi = (uint64_t)std::ldexp(m, 53);  // x = mi * 2^(e-53)
    const int sh = e - 53 + S;
    if (sh < 0) {
        mi >>= -sh;  // exact by the choice of S
        r = from_u128(mi);
    } else {
        r = shl(from_u128(mi), sh);
    }
    r.neg = x < 0;
    norm(r);
    return r;
}

// round-to-nearest-even double of v / 2^S
double to_double_rn(const Big& v, int S) {
    if (v.n == 0) return 0.0;
    const int b = bitlen(v);
    const int e_top = b - 1 - S;  // |value| in [2^e_top, 2^(e_top+1))
    int p = 53;
    if (e_top < -1022) p = std::max(0, 53 - (-1022 - e_top));
    const int drop = b - p;
    double r;
    if (drop <= 0) {
        r = std::ldexp((double)to_u128(v), -S);  // exact: fits 53 bits
    } else {
        Big M = shr_mag(v, drop);
        const bool half = bit(v, drop - 1);
        const bool sticky = low_bits_nonzero(v, drop - 1);
        unsigned __int128 m = to_u128(M);
        if (half && (sticky || (m & 1))) m += 1;
        r = std::ldexp((double)m, drop - S);
    }
    return v.neg ? -r : r;
}

// ---------------------------------------------------------------- grid (GridContext, backtrack.py:54-107)

struct Grid {
    int n;
    std::vector<int> S;      // per-variable scale
    std::vector<Big> W;      // width * 2^S
    std::vector<double> a;   // anchors (doubles)
    std::vector<Big> A;      // anchor * 2^S
};

// ---- 128-bit fast path: every scaled quantity of the box fits comfortably
using i128 = __int128;
using u128 = unsigned __int128;

int bitlen128(u128 v) {
    if (v == 0) return 0;
    const uint64_t hi = (uint64_t)(v >> 64);
    return hi ? 128 - __builtin_clzll(hi) : 64 - __builtin_clzll((uint64_t)v);
}

// x * 2^S as a 128-bit integer; false when not exact or |value| >= 2^120
bool scaled_i128(double x, int S, i128& out) {
    if (x == 0.0) {
        out = 0;
        return true;
    }
    int e;
    const double m = std::frexp(std::fabs(x), &e);
    uint64_t mi = (uint64_t)std::ldexp(m, 53);
    const int sh = e - 53 + S;
    if (sh < 0) {
        if (-sh >= 64 || (mi & ((1ull << -sh) - 1))) return false;
        mi >>= -sh;
        out = (i128)mi;
    } else {
        if (sh > 66) return false;
        out = (i128)mi << sh;
    }
    if (x < 0) out = -out;
    return true;
}

bool big_to_i128(const Big& b, i128& out) {
    if (bitlen(b) > 120) return false;
    const u128 v = (u128)limb(b, 0) | ((u128)limb(b, 1) << 64);
    out = b.neg ? -(i128)v : (i128)v;
    return true;
}

inline int absbits(i128 v) { return bitlen128(v < 0 ? (u128)(-v) : (u128)v); }

// exactly representable as a double (53 significant bits, normal range)
bool exact_double(u128 num, int S2) {
    if (num == 0) return true;
    const int tz = __builtin_ctzll((uint64_t)num) + (((uint64_t)num) == 0 ? __builtin_ctzll((uint64_t)(num >> 64)) : 0);
    const u128 odd = num >> tz;
    return bitlen128(odd) <= 53 && (bitlen128(num) - 1 - S2) > -1022;
}

// snap_to_grid of one box on 128-bit integers; returns 0 ok, 1 fall back to Big, -1 error
int snap_fast(const std::vector<i128>& A, const std::vector<i128>& W, const std::vector<int>& S, int n,
              const double* blo, const double* bhi, int& L_out, std::vector<u128>& idx, std::string& err) {
    i128 dlo[16], dhi[16];
    int level = -1;
    for (int i = 0; i < n; i++) {
        i128 xl, xh;
        if (!scaled_i128(blo[i], S[i], xl) || !scaled_i128(bhi[i], S[i], xh)) return 1;
        dlo[i] = xl - A[i];
        dhi[i] = xh - A[i];
        if (dlo[i] < 0 || dhi[i] > W[i]) {
            err = "component " + std::to_string(i) + " lies outside the initial range";
            return -1;
        }
        const i128 w = dhi[i] - dlo[i];
        if (w == 0) continue;
        const int li = bitlen128((u128)(W[i] / w)) - 1;
        level = level < 0 ? li : std::min(level, li);
    }
    if (level < 0) level = 52;
    int bits = 0;  // every product / shift below stays under 2^126
    for (int i = 0; i < n; i++)
        bits = std::max({bits, absbits(A[i]), absbits(W[i]), absbits(dlo[i]), absbits(dhi[i])});
    if (bits + level + 2 > 125) return 1;
    int L = level;
    for (; L > 0; L--) {
        bool ok = true;
        for (int i = 0; i < n && ok; i++) {
            u128 k = (u128)((dlo[i] << L) / W[i]);
            const u128 kmax = (((u128)1) << L) - 1;
            if (k > kmax) k = kmax;
            if ((dhi[i] << L) > (i128)(k + 1) * W[i]) ok = false;
            idx[i] = k;
        }
        if (ok) break;
    }
    if (L == 0) std::fill(idx.begin(), idx.end(), (u128)0);
    for (int i = 0; i < n; i++) {
        const i128 num_lo = (A[i] << L) + (i128)idx[i] * W[i];
        const i128 num_hi = num_lo + W[i];
        const int S2 = S[i] + L;
        const bool e1 = num_lo < 0 ? exact_double((u128)(-num_lo), S2) : exact_double((u128)num_lo, S2);
        const bool e2 = num_hi < 0 ? exact_double((u128)(-num_hi), S2) : exact_double((u128)num_hi, S2);
        if (!e1 || !e2) {
            err = "snapped cell is not exactly representable (non-dyadic initial box)";
            return -1;
        }
    }
    L_out = L;
    return 0;
}

// |a| * |b| with the sign of a * b
Big mul_big(const Big& a, const Big& b) {
    Big r;
    if (a.n == 0 || b.n == 0) return r;
    const int rn = a.n + b.n;
    if (rn > LIMBS) throw std::string("integer too large");
    for (int i = 0; i < rn; i++) r.w[i] = 0;
    for (int i = 0; i < a.n; i++) {
        unsigned __int128 c = 0;
        for (int j = 0; j < b.n; j++) {
            c += (unsigned __int128)a.w[i] * b.w[j] + r.w[i + j];
            r.w[i + j] = (uint64_t)c;
            c >>= 64;
        }
        r.w[i + b.n] = (uint64_t)c;
    }
    r.n = rn;
    r.neg = a.neg != b.neg;
    norm(r);
    return r;
}

// ---- cell indices: 128-bit while every snapped level is at most 120, else wide keys
// (snap_to_grid has no level limit: a box of width ~1e-300 snaps to a level near 1000)
constexpr int KW = 18;  // 1152 bits: indices below 2^L for any level a double box can reach
struct KeyW {
    uint64_t w[KW];
};
inline bool operator<(const KeyW& a, const KeyW& b) {
    for (int i = KW - 1; i >= 0; i--)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
    return false;
}
inline bool operator==(const KeyW& a, const KeyW& b) {
    for (int i = 0; i < KW; i++)
        if (a.w[i] != b.w[i]) return false;
    return true;
}
inline bool operator!=(const KeyW& a, const KeyW& b) { return !(a == b); }
inline KeyW operator>>(const KeyW& a, int s) {
    KeyW r{};
    const int q = s / 64, b = s % 64;
    for (int i = q; i < KW; i++) {
        uint64_t v = a.w[i] >> b;
        if (b && i + 1 < KW) v |= a.w[i + 1] << (64 - b);
        r.w[i - q] = v;
    }
    return r;
}
KeyW keyw_of(const Big& b) {
    if (b.neg || b.n > KW) throw std::string("cell index beyond the wide key range");
    KeyW k{};
    for (int i = 0; i < b.n; i++) k.w[i] = b.w[i];
    return k;
}
KeyW keyw_of(u128 v) {
    KeyW k{};
    k.w[0] = (uint64_t)v;
    k.w[1] = (uint64_t)(v >> 64);
    return k;
}
Big big_of(u128 v) { return from_u128(v); }
Big big_of(const KeyW& k) {
    Big b;
    int n = KW;
    while (n > 0 && k.w[n - 1] == 0) n--;
    for (int i = 0; i < n; i++) b.w[i] = k.w[i];
    b.n = n;
    return b;
}

// _float_down / _float_up of (A + k W / 2^L) / 2^S
double cell_bound(const Grid& g, int i, int L, const Big& k, bool up) {
    // value * 2^(S+L) = A 2^L + k W
    const Big num = add(shl(g.A[i], L), mul_big(g.W[i], k));
    const int S2 = g.S[i] + L;
    double f = to_double_rn(num, S2);
    // exact comparison of f with the rational
    int fe_ok = f == 0.0 ? 1 : (S2 >= -low_exp(f));
    Big fb = fe_ok ? from_double(f, S2) : Big();
    const int c = fe_ok ? cmp(fb, num) : 0;
    if (!up && c > 0) f = std::nextafter(f, -INFINITY);
    if (up && c < 0) f = std::nextafter(f, INFINITY);
    return f;
}

// Cells of one level: flat keys (n indices per cell) + flags; sorted and unique
// after norm_level().  Cells keep a uniform level per box (snap_to_grid), as in
// the reference, so a cell is (L, k_0 .. k_{n-1}).
template <typename K>
struct LevelVec {
    std::vector<K> keys;
    std::vector<uint8_t> flags;
};
template <typename K>
using Cells = std::map<int, LevelVec<K>>;

// sort + unique with flag OR (dict assignment `cells[key] = cells.get(key) or flag`)
template <typename K>
void norm_level(LevelVec<K>& v, int n) {
    const size_t m = v.flags.size();
    std::vector<uint32_t> ord(m);
    for (size_t i = 0; i < m; i++) ord[i] = (uint32_t)i;
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
        const K* x = &v.keys[(size_t)a * n];
        const K* y = &v.keys[(size_t)b * n];
        for (int i = 0; i < n; i++)
            if (x[i] != y[i]) return x[i] < y[i];
        return false;
    });
    LevelVec<K> o;
    o.keys.reserve(v.keys.size());
    o.flags.reserve(m);
    for (size_t j = 0; j < m; j++) {
        const K* x = &v.keys[(size_t)ord[j] * n];
        if (!o.flags.empty() && std::equal(x, x + n, &o.keys[o.keys.size() - n])) {
            o.flags.back() |= v.flags[ord[j]];
            continue;
        }
        o.keys.insert(o.keys.end(), x, x + n);
        o.flags.push_back(v.flags[ord[j]]);
    }
    v = std::move(o);
}

// index of key in a normalised level, or -1
template <typename K>
int64_t find_key(const LevelVec<K>& v, const K* key, int n) {
    int64_t lo = 0, hi = (int64_t)v.flags.size() - 1;
    while (lo <= hi) {
        const int64_t mid = (lo + hi) / 2;
        const K* x = &v.keys[(size_t)mid * n];
        int c = 0;
        for (int i = 0; i < n && c == 0; i++) c = x[i] < key[i] ? -1 : (key[i] < x[i] ? 1 : 0);
        if (c == 0) return mid;
        if (c < 0) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

// _drop_nested (backtrack.py:168-191) for uniform-level cells: a cell inside a
// kept coarser cell is absorbed (flag OR into the coarsest such ancestor).
template <typename K>
Cells<K> drop_nested(Cells<K> cells, int n) {
    for (auto& kv : cells) norm_level(kv.second, n);
    if (cells.size() <= 1) return cells;
    Cells<K> kept;
    std::vector<K> anc(n);
    for (auto& [L, v] : cells) {  // coarse (small L) first
        LevelVec<K> out;
        for (size_t c = 0; c < v.flags.size(); c++) {
            const K* k = &v.keys[c * n];
            bool absorbed = false;
            for (auto& [L2, v2] : kept) {
                if (L2 >= L) break;
                for (int i = 0; i < n; i++) anc[i] = k[i] >> (L - L2);
                const int64_t j = find_key(v2, anc.data(), n);
                if (j >= 0) {
                    v2.flags[j] |= v.flags[c];
                    absorbed = true;
                    break;
                }
            }
            if (!absorbed) {
                out.keys.insert(out.keys.end(), k, k + n);
                out.flags.push_back(v.flags[c]);
            }
        }
        if (!out.flags.empty()) kept[L] = std::move(out);  // still sorted and unique
    }
    return kept;
}

template <typename K>
size_t count(const Cells<K>& c) {
    size_t s = 0;
    for (auto& kv : c) s += kv.second.flags.size();
    return s;
}

template <typename K>
double cur_width(const Grid& g, const Cells<K>& cells) {
    double w = 0.0;
    bool any = false;
    for (auto& [L, m] : cells) {
        if (m.flags.empty()) continue;
        for (int i = 0; i < g.n; i++) {
            const double x = to_double_rn(g.W[i], g.S[i] + L);  // float(W_i / 2^L)
            w = any ? std::max(w, x) : x;
            any = true;
        }
    }
    return any ? w : 0.0;
}

struct OutBox {
    std::vector<double> lo, hi;
    bool flag;
};

// merge_to_width (backtrack.py:194-242) of snapped cells, materialised in canonical
// order (Box.sort_key: lows then highs)
template <typename K>
void merge_levels(const Grid& g, Cells<K> cells, double stop_width, int stop_on_plateau, std::vector<OutBox>& out,
                  std::vector<std::pair<double, int64_t>>& log) {
    const int n = g.n;
    cells = drop_nested(std::move(cells), n);
    log.push_back({cur_width(g, cells), (int64_t)count(cells)});
    const bool has_stop = stop_width >= 0 && !std::isnan(stop_width);
    while (count(cells) > 0) {
        if (stop_on_plateau && log.size() >= 2 && log[log.size() - 1].second == log[log.size() - 2].second) break;
        if (has_stop && log.back().first >= stop_width) break;
        if (cells.count(0) && !cells[0].flags.empty()) break;
        Cells<K> parents;
        for (auto& [L, m] : cells) {
            auto& pv = parents[L - 1];
            pv.keys.resize(m.keys.size());
            for (size_t i = 0; i < m.keys.size(); i++) pv.keys[i] = m.keys[i] >> 1;
            pv.flags = m.flags;
        }
        cells = drop_nested(std::move(parents), n);
        log.push_back({cur_width(g, cells), (int64_t)count(cells)});
    }
    for (auto& [L, m] : cells)
        for (size_t c = 0; c < m.flags.size(); c++) {
            const K* k = &m.keys[c * n];
            OutBox b;
            b.lo.resize(n);
            b.hi.resize(n);
            for (int i = 0; i < n; i++) {
                const Big kb = big_of(k[i]);
                b.lo[i] = cell_bound(g, i, L, kb, false);
                b.hi[i] = cell_bound(g, i, L, add(kb, from_u128(1)), true);
            }
            b.flag = m.flags[c] != 0;
            out.push_back(std::move(b));
        }
    std::sort(out.begin(), out.end(), [&](const OutBox& x, const OutBox& y) {
        for (int i = 0; i < n; i++)
            if (x.lo[i] != y.lo[i]) return x.lo[i] < y.lo[i];
        for (int i = 0; i < n; i++)
            if (x.hi[i] != y.hi[i]) return x.hi[i] < y.hi[i];
        return false;
    });
}

}  // namespace

extern "C" {

// snap_to_grid (backtrack.py:118-158) of N boxes + merge_to_width (backtrack.py:194-242).
// lo/hi [N x n] row-major, cert [N]; initial box init_lo/init_hi [n]; stop_width < 0 or
// NaN = None.  Outputs (caller capacity `cap` boxes / `cap_levels` levels):
// out_lo/out_hi [M x n] canonical order (Box.sort_key), out_cert [M], levels [K x 2]
// (width, count).  Returns 0 or a negative code; *M / *K receive the true sizes.
int rb_merge(int n, const double* init_lo, const double* init_hi, const double* lo, const double* hi,
             const uint8_t* cert, int64_t N, double stop_width, int stop_on_plateau, double* out_lo, double* out_hi,
             uint8_t* out_cert, int64_t cap, int64_t* M, double* levels, int64_t cap_levels, int64_t* K,
             char* err, int64_t err_len) {
    auto fail = [&](const std::string& msg) {
        if (err && err_len > 0) {
            std::strncpy(err, msg.c_str(), (size_t)err_len - 1);
            err[err_len - 1] = 0;
        }
        return RB_ERR_ARG;
    };
    try {
        if (n < 1 || n > RB_MAX_DIM || N < 0) return fail("bad arguments");
        Grid g;
        g.n = n;
        g.S.assign(n, 0);
        for (int i = 0; i < n; i++) {
            if (!(init_hi[i] > init_lo[i])) return fail("initial box must have positive widths");
            int s = 0;
            auto need = [&](double x) {
                if (x != 0.0 && std::isfinite(x)) s = std::max(s, -low_exp(x));
            };
            need(init_lo[i]);
            need(init_hi[i]);
            for (int64_t r = 0; r < N; r++) {
                need(lo[r * n + i]);
                need(hi[r * n + i]);
            }
            g.S[i] = s;
            g.a.push_back(init_lo[i]);
            g.A.push_back(from_double(init_lo[i], s));
            g.W.push_back(sub(from_double(init_hi[i], s), g.A.back()));
        }
        // ---- snap_to_grid per box: 128-bit indices (fast path) or big ones, then the merge
        // runs on 128-bit keys when every level is at most 120, else on wide keys
        Cells<u128> cells;
        std::vector<std::pair<int, std::vector<Big>>> deep;  // (level, indices) of boxes snapped beyond 120
        std::vector<uint8_t> deep_flags;
        std::vector<i128> fA(n), fW(n);
        bool fast = true;
        for (int i = 0; i < n; i++) fast = fast && big_to_i128(g.A[i], fA[i]) && big_to_i128(g.W[i], fW[i]);
        for (int64_t r = 0; r < N; r++) {
            const uint8_t flag = cert && cert[r] ? 1 : 0;
            if (fast) {
                std::vector<u128> fidx(n, 0);
                int fL = 0;
                std::string ferr;
                const int rc = snap_fast(fA, fW, g.S, n, lo + r * n, hi + r * n, fL, fidx, ferr);
                if (rc < 0) return fail(ferr);
                if (rc == 0) {
                    auto& lv = cells[fL];
                    lv.keys.insert(lv.keys.end(), fidx.begin(), fidx.end());
                    lv.flags.push_back(flag);
                    continue;
                }
            }
            std::vector<Big> dlo(n), dhi(n);
            int level = -1;
            for (int i = 0; i < n; i++) {
                dlo[i] = sub(from_double(lo[r * n + i], g.S[i]), g.A[i]);
                dhi[i] = sub(from_double(hi[r * n + i], g.S[i]), g.A[i]);
                if (sign(dlo[i]) < 0 || cmp(dhi[i], g.W[i]) > 0)
                    return fail("component " + std::to_string(i) + " lies outside the initial range");
                const Big w = sub(dhi[i], dlo[i]);
                if (w.n == 0) continue;
                const int li = bitlen(div_floor(g.W[i], w)) - 1;  // ratio >= 1
                level = level < 0 ? li : std::min(level, li);
            }
            if (level < 0) level = 52;  // a point box: snap to a deep cell
            std::vector<Big> idx(n);
            int L = level;
            for (; L > 0; L--) {
                bool ok = true;
                for (int i = 0; i < n && ok; i++) {
                    // k = floor((lo - a) / cw), cw = W / 2^L;  k = min(k, 2^L - 1)
                    Big kb = div_floor(shl(dlo[i], L), g.W[i]);
                    const Big kmax = sub(shl(from_u128(1), L), from_u128(1));
                    if (cmp(kb, kmax) > 0) kb = kmax;
                    // straddles when hi > a + (k+1) cw  <=>  (hi - a) 2^L > (k+1) W
                    if (cmp(shl(dhi[i], L), mul_big(g.W[i], add(kb, from_u128(1)))) > 0) ok = false;
                    idx[i] = kb;
                }
                if (ok) break;
            }
            if (L == 0) std::fill(idx.begin(), idx.end(), Big());
            // merge_to_width: locate() of the snapped cell box is exact only when its
            // materialised bounds are exact (dyadic initial box, backtrack.py:1-9)
            for (int i = 0; i < n; i++) {
                const Big num_lo = add(shl(g.A[i], L), mul_big(g.W[i], idx[i]));
                const Big num_hi = add(num_lo, g.W[i]);
                const double flo = cell_bound(g, i, L, idx[i], false);
                const double fhi = cell_bound(g, i, L, add(idx[i], from_u128(1)), true);
                const int S2 = g.S[i] + L;
                if ((flo != 0.0 && S2 < -low_exp(flo)) || (fhi != 0.0 && S2 < -low_exp(fhi)) ||
                    cmp(from_double(flo, S2), num_lo) != 0 || cmp(from_double(fhi, S2), num_hi) != 0)
                    return fail(L > 120 ? "snapped cell is not exactly representable at its level: the reference's "
                                          "locate() would give it per-component levels, which rb_merge does not handle"
                                        : "snapped cell is not exactly representable (non-dyadic initial box)");
            }
            if (L <= 120) {
                auto& lv = cells[L];
                for (int i = 0; i < n; i++) lv.keys.push_back(to_u128(idx[i]));
                lv.flags.push_back(flag);
            } else {
                deep.emplace_back(L, std::move(idx));
                deep_flags.push_back(flag);
            }
        }
        const bool timing = std::getenv("RB_MERGE_TIMING") != nullptr;
        auto tnow = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
        double t_snap = tnow();
        std::vector<std::pair<double, int64_t>> log;
        std::vector<OutBox> out;
        if (deep.empty()) {
            merge_levels(g, std::move(cells), stop_width, stop_on_plateau, out, log);
        } else {  // some box snapped beyond level 120: every key goes wide
            Cells<KeyW> wide;
            for (auto& [L, m] : cells) {
                auto& lv = wide[L];
                for (const u128 k : m.keys) lv.keys.push_back(keyw_of(k));
                lv.flags = m.flags;
            }
            for (size_t d = 0; d < deep.size(); d++) {
                auto& lv = wide[deep[d].first];
                for (const Big& k : deep[d].second) lv.keys.push_back(keyw_of(k));
                lv.flags.push_back(deep_flags[d]);
            }
            merge_levels(g, std::move(wide), stop_width, stop_on_plateau, out, log);
        }
        if (timing) std::fprintf(stderr, "rb_merge: merge levels %.3fs\n", tnow() - t_snap);
        *M = (int64_t)out.size();
        for (int64_t r = 0; r < (int64_t)out.size() && r < cap; r++) {
            for (int i = 0; i < n; i++) {
                out_lo[r * n + i] = out[r].lo[i];
                out_hi[r * n + i] = out[r].hi[i];
            }
            out_cert[r] = out[r].flag ? 1 : 0;
        }
        *K = (int64_t)log.size();
        for (int64_t r = 0; r < (int64_t)log.size() && r < cap_levels; r++) {
            levels[2 * r] = log[r].first;
            levels[2 * r + 1] = (double)log[r].second;
        }
        return RB_OK;
    } catch (const std::string& e) {
        return fail(e);
    }
}

}  // extern "C"
