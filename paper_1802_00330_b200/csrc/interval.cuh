// interval.cuh -- outward-rounded FP64 interval arithmetic for sm_100a.
//
// Two arithmetic policies with identical interfaces:
//
//  * Fast  -- IEEE directed-rounding instructions (__dadd_rd/__dmul_ru/...):
//             one DADD/DMUL per bound, case-split interval multiply (2 products
//             unless both operands straddle zero) and single-multiply pow chains.
//  * Exact -- a literal device restatement of the reference's error-free-
//             transformation rounding (rootbox/interval.py:66-205), including
//             its "untrusted" band: products with |a| or |b| > 2^995 or
//             |RN(a*b)| < 2^-970 always step one ulp outward (interval.py:98-136),
//             quotients likewise (interval.py:139-190), and Python's
//             first-extreme min/max over the four products (interval.py:322-326).
//
// Fast == Exact bit for bit (up to the sign of a zero result, which no
// comparison, product, sum or quotient on the solver path can observe and
// which the engine canonicalises to +0.0 on output) whenever every product is
// inside the trusted band.  The kernels prove that per box with exponent-range
// guards (see guard_* in engine.cuh) and fall back to Exact otherwise.
#pragma once
#ifdef __CUDACC_RTC__
// NVRTC (system-specialised kernels, codegen.cpp): no host C++ headers
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long int64_t;
typedef unsigned long uint64_t;
#define INT_MAX 2147483647
#define INT_MIN (-INT_MAX - 1)
#define LLONG_MAX 9223372036854775807LL
#define RB_KINST_TU 1
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif
#include <math_constants.h>

namespace rb {

struct ival {
    double lo, hi;
};

__device__ __forceinline__ ival mk(double lo, double hi) {
    ival r;
    r.lo = lo;
    r.hi = hi;
    return r;
}

#define RB_MAXF 1.7976931348623157e308
#define RB_TINY 0x1p-970
#define RB_BIG 0x1p995

__device__ __forceinline__ bool contains_zero(ival x) { return x.lo <= 0.0 && 0.0 <= x.hi; }

// Interval.mid (interval.py:269-281) / _batch.midpoints (_batch.py:212-217): RN, clipped.
__device__ __forceinline__ double mid_of(double lo, double hi) {
    double m = __dmul_rn(0.5, __dadd_rn(lo, hi));
    if (isinf(m)) m = __dadd_rn(__dmul_rn(0.5, lo), __dmul_rn(0.5, hi));
    if (m < lo) m = lo;
    if (m > hi) m = hi;
    return m;
}

__device__ __forceinline__ double next_down(double x) { return nextafter(x, -CUDART_INF); }
__device__ __forceinline__ double next_up(double x) { return nextafter(x, CUDART_INF); }

// Python min()/max() over a sequence keep the first extreme element.
__device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }

// ------------------------------------------------------------------ Fast policy
struct Fast {
    static constexpr bool exact = false;
    __device__ __forceinline__ static double add_rd(double a, double b) { return __dadd_rd(a, b); }
    __device__ __forceinline__ static double add_ru(double a, double b) { return __dadd_ru(a, b); }
    __device__ __forceinline__ static double mul_rd(double a, double b) { return __dmul_rd(a, b); }
    __device__ __forceinline__ static double mul_ru(double a, double b) { return __dmul_ru(a, b); }

    __device__ __forceinline__ static ival add(ival x, ival y) {
        return mk(__dadd_rd(x.lo, y.lo), __dadd_ru(x.hi, y.hi));
    }
    __device__ __forceinline__ static ival sub(ival x, ival y) {
        return mk(__dadd_rd(x.lo, -y.hi), __dadd_ru(x.hi, -y.lo));
    }
    // [c,c] * y  (4-product min/max of interval.py:322-326 reduces to 2 products)
    __device__ __forceinline__ static ival mul_point(double c, ival y) {
        double a = (c >= 0.0) ? y.lo : y.hi;
        double b = (c >= 0.0) ? y.hi : y.lo;
        return mk(__dmul_rd(c, a), __dmul_ru(c, b));
    }
    // interval.py:322-326 / _batch.i_mul (_batch.py:94-105): min of the four RD products,
    // max of the four RU products, as the pairwise tree of _batch.i_mul.  Eight
    // independent DMULs and two select trees: a short dependency chain (the
    // sign-case split it replaces waited on four compares and a branch first).
    __device__ __forceinline__ static ival mul(ival x, ival y) {
        const double p0 = __dmul_rd(x.lo, y.lo), p1 = __dmul_rd(x.lo, y.hi);
        const double p2 = __dmul_rd(x.hi, y.lo), p3 = __dmul_rd(x.hi, y.hi);
        const double q0 = __dmul_ru(x.lo, y.lo), q1 = __dmul_ru(x.lo, y.hi);
        const double q2 = __dmul_ru(x.hi, y.lo), q3 = __dmul_ru(x.hi, y.hi);
        return mk(py_min(py_min(p0, p1), py_min(p2, p3)), py_max(py_max(q0, q1), py_max(q2, q3)));
    }
    // interval.py:328-345 / _batch.py:122-138.  Odd powers use the identity
    // -chain_ru(-l) == chain of RD multiplications by |l| started at l (and
    // mirror for the upper bound), one product per step.
    __device__ __forceinline__ static ival pow(ival x, int k) {
        if (k == 1) return x;
        if (k == 0) return mk(1.0, 1.0);
        if ((k & 1) == 0) {
            const double al = fabs(x.lo), ah = fabs(x.hi);
            const double mlo = contains_zero(x) ? 0.0 : fmin(al, ah);
            const double mhi = fmax(al, ah);
            double rl = mlo, rh = mhi;
            for (int i = 1; i < k; i++) {
                rl = __dmul_rd(rl, mlo);
                rh = __dmul_ru(rh, mhi);
            }
            return mk(rl, rh);
        }
        const double al = fabs(x.lo), ah = fabs(x.hi);
        double rl = x.lo, rh = x.hi;
        for (int i = 1; i < k; i++) {
            rl = __dmul_rd(rl, al);
            rh = __dmul_ru(rh, ah);
        }
        return mk(rl, rh);
    }
};

// interval.py:98-108: Dekker product error by FMA-free Veltkamp splitting,
// exactly as the reference computes it (NaN = "untrusted").
static __device__ __noinline__ double prod_err_ref(double a, double b, double p) {
    if (fabs(a) > RB_BIG || fabs(b) > RB_BIG || fabs(p) < RB_TINY) return CUDART_NAN;
    const double S = 134217729.0;
    double ah = __dmul_rn(S, a);
    ah = __dsub_rn(ah, __dsub_rn(ah, a));
    double al = __dsub_rn(a, ah);
    double bh = __dmul_rn(S, b);
    bh = __dsub_rn(bh, __dsub_rn(bh, b));
    double bl = __dsub_rn(b, bh);
    return __dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(ah, bh), p), __dmul_rn(ah, bl)),
                               __dmul_rn(al, bh)),
                     __dmul_rn(al, bl));
}

// ------------------------------------------------------------------ Exact policy
struct Exact {
    static constexpr bool exact = true;
    // interval.py:66-79
    __device__ __noinline__ static double add_rd(double a, double b) {
        double s = __dadd_rn(a, b);
        if (s == -CUDART_INF) return s;
        if (s == CUDART_INF) return (a == CUDART_INF || b == CUDART_INF) ? s : RB_MAXF;
        if (s != s) return -CUDART_INF;
        if (s == 0.0) return s;             // exact zero: the RN sum (its sign included)
        return __dadd_rd(a, b);             // TwoSum-based RD == IEEE RD for finite sums
    }
    // interval.py:82-95
    __device__ __noinline__ static double add_ru(double a, double b) {
        double s = __dadd_rn(a, b);
        if (s == CUDART_INF) return s;
        if (s == -CUDART_INF) return (a == -CUDART_INF || b == -CUDART_INF) ? s : -RB_MAXF;
        if (s != s) return CUDART_INF;
        if (s == 0.0) return s;
        return __dadd_ru(a, b);
    }
    // interval.py:98-122
    __device__ __noinline__ static double mul_rd(double a, double b) {
        if (a == 0.0 || b == 0.0) return 0.0;
        double p = __dmul_rn(a, b);
        if (p == -CUDART_INF) return p;
        if (p == CUDART_INF) return (isinf(a) || isinf(b)) ? p : RB_MAXF;
        double err = prod_err_ref(a, b, p);
        if (!(err >= 0.0)) return next_down(p);
        return p;
    }
    // interval.py:125-136
    __device__ __noinline__ static double mul_ru(double a, double b) {
        if (a == 0.0 || b == 0.0) return 0.0;
        double p = __dmul_rn(a, b);
        if (p == CUDART_INF) return p;
        if (p == -CUDART_INF) return (isinf(a) || isinf(b)) ? p : -RB_MAXF;
        double err = prod_err_ref(a, b, p);
        if (!(err <= 0.0)) return next_up(p);
        return p;
    }
    __device__ __noinline__ static ival add(ival x, ival y) { return mk(add_rd(x.lo, y.lo), add_ru(x.hi, y.hi)); }
    __device__ __noinline__ static ival sub(ival x, ival y) { return mk(add_rd(x.lo, -y.hi), add_ru(x.hi, -y.lo)); }
    // interval.py:322-326 (literal)
    __device__ __noinline__ static ival mul(ival x, ival y) {
        double lo = mul_rd(x.lo, y.lo);
        lo = py_min(lo, mul_rd(x.lo, y.hi));
        lo = py_min(lo, mul_rd(x.hi, y.lo));
        lo = py_min(lo, mul_rd(x.hi, y.hi));
        double hi = mul_ru(x.lo, y.lo);
        hi = py_max(hi, mul_ru(x.lo, y.hi));
        hi = py_max(hi, mul_ru(x.hi, y.lo));
        hi = py_max(hi, mul_ru(x.hi, y.hi));
        return mk(lo, hi);
    }
    __device__ __noinline__ static ival mul_point(double c, ival y) { return mul(mk(c, c), y); }
    // interval.py:193-205, 328-345 (literal)
    __device__ static double chain_rd(double t, int k) {
        double r = t;
        for (int i = 1; i < k; i++) r = mul_rd(r, t);
        return r;
    }
    __device__ static double chain_ru(double t, int k) {
        double r = t;
        for (int i = 1; i < k; i++) r = mul_ru(r, t);
        return r;
    }
    __device__ __noinline__ static ival pow(ival x, int k) {
        if (k == 0) return mk(1.0, 1.0);
        if (k == 1) return x;
        if ((k & 1) == 0) {
            double mag_lo = contains_zero(x) ? 0.0 : py_min(fabs(x.lo), fabs(x.hi));
            double mag_hi = py_max(fabs(x.lo), fabs(x.hi));
            return mk(chain_rd(mag_lo, k), chain_ru(mag_hi, k));
        }
        double lo = x.lo >= 0 ? chain_rd(x.lo, k) : -chain_ru(-x.lo, k);
        double hi = x.hi >= 0 ? chain_ru(x.hi, k) : -chain_rd(-x.hi, k);
        return mk(lo, hi);
    }
};

// ------------------------------------------------------------------ division (always exact)
// interval.py:139-154

static __device__ __noinline__ double div_err_sign(double a, double b, double q) {
    if (isinf(a) || isinf(b) || isinf(q)) return CUDART_NAN;
    double p = __dmul_rn(q, b);
    if (fabs(q) > RB_BIG || fabs(b) > RB_BIG || (p != 0.0 && fabs(p) < RB_TINY)) return CUDART_NAN;
    double err = prod_err_ref(q, b, p);
    if (err != err) return CUDART_NAN;
    double d = __dsub_rn(a, p);
    double r = __dsub_rn(d, err);
    return r != 0.0 ? copysign(1.0, __ddiv_rn(r, b)) : 0.0;
}

// interval.py:157-172
static __device__ __noinline__ double div_rd(double a, double b) {
    if (a == 0.0) return 0.0;
    if (isinf(a) && !isinf(b)) return ((a < 0) == (b < 0) || a > 0) ? a : -CUDART_INF;
    double q = __ddiv_rn(a, b);
    if (q == -CUDART_INF) return q;
    if (q == CUDART_INF) return isinf(a) ? q : RB_MAXF;
    if (q != q) return -CUDART_INF;
    double s = div_err_sign(a, b, q);
    if (!(s >= 0.0)) return next_down(q);
    return q;
}

// interval.py:175-190
static __device__ __noinline__ double div_ru(double a, double b) {
    if (a == 0.0) return 0.0;
    if (isinf(a) && !isinf(b)) return (a > 0 || (a < 0) == (b < 0)) ? a : CUDART_INF;
    double q = __ddiv_rn(a, b);
    if (q == CUDART_INF) return q;
    if (q == -CUDART_INF) return isinf(a) ? q : -RB_MAXF;
    if (q != q) return CUDART_INF;
    double s = div_err_sign(a, b, q);
    if (!(s <= 0.0)) return next_up(q);
    return q;
}

// ------------------------------------------------------------------ exponent guards

// Unbiased binary exponent of a finite double's magnitude; zero -> INT_MAX/INT_MIN
// sentinels are handled by callers.  Subnormals report -1075 (conservative).
__device__ __forceinline__ int exp_of(double v) {
    const int hiw = __double2hiint(v);
    const int f = (hiw >> 20) & 0x7ff;
    return f ? f - 1023 : -1075;
}

// Track min exponent over nonzero values and max exponent over all values.
struct ExpRange {
    int emin, emax;
    __device__ __forceinline__ void init() { emin = 4096; emax = -4096; }
    __device__ __forceinline__ void add(double v) {
        if (v != 0.0) {
            const int e = exp_of(v);
            emin = min(emin, e);
            emax = max(emax, e);
        }
    }
};

}  // namespace rb
