// Dependent-chain latency of interval-product variants on sm_100a (dev tool).
#include <cstdio>
#include "kernels.cuh"
using namespace rb;
#define ITERS 512

__device__ __forceinline__ ival mul4(ival x, ival y) {
    const double p0 = __dmul_rd(x.lo, y.lo), p1 = __dmul_rd(x.lo, y.hi), p2 = __dmul_rd(x.hi, y.lo), p3 = __dmul_rd(x.hi, y.hi);
    const double q0 = __dmul_ru(x.lo, y.lo), q1 = __dmul_ru(x.lo, y.hi), q2 = __dmul_ru(x.hi, y.lo), q3 = __dmul_ru(x.hi, y.hi);
    return mk(fmin(fmin(p0, p1), fmin(p2, p3)), fmax(fmax(q0, q1), fmax(q2, q3)));
}
__device__ __forceinline__ double sel_min(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double sel_max(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ ival mul4s(ival x, ival y) {
    const double p0 = __dmul_rd(x.lo, y.lo), p1 = __dmul_rd(x.lo, y.hi), p2 = __dmul_rd(x.hi, y.lo), p3 = __dmul_rd(x.hi, y.hi);
    const double q0 = __dmul_ru(x.lo, y.lo), q1 = __dmul_ru(x.lo, y.hi), q2 = __dmul_ru(x.hi, y.lo), q3 = __dmul_ru(x.hi, y.hi);
    return mk(sel_min(sel_min(p0, p1), sel_min(p2, p3)), sel_max(sel_max(q0, q1), sel_max(q2, q3)));
}

__global__ void k_lat(double* out, long long* cyc, double a0, double b0) {
    volatile double vb = b0;
    double a = a0 + threadIdx.x * 1e-30, b = vb;
    ival x = mk(a - 0.5, a + 1.0), y = mk(b - 0.7, b + 0.3);
    long long t0, t1;
    int k = 0;
#define MEASURE(body)                                                  \
    t0 = clock64();                                                    \
    _Pragma("unroll 1") for (int i = 0; i < ITERS; i++) { body; }      \
    t1 = clock64();                                                    \
    if (threadIdx.x == 0) cyc[k] = (t1 - t0) / ITERS;                  \
    k++;
    MEASURE(a = __dadd_rd(a, b); b = vb);
    MEASURE(a = __dmul_ru(a, b); b = vb);
    MEASURE(a = fmin(a, b); b = b + a * 0.0);
    MEASURE(a = sel_min(a, b); b = b + a * 0.0);
    MEASURE(x = Fast::mul(x, y); y = mk(y.lo + x.lo * 1e-300, y.hi));
    MEASURE(x = mul4(x, y); y = mk(y.lo + x.lo * 1e-300, y.hi));
    MEASURE(x = mul4s(x, y); y = mk(y.lo + x.lo * 1e-300, y.hi));
    MEASURE(x = gmul(x, y); y = mk(y.lo + x.lo * 1e-300, y.hi));
    MEASURE(x = pmul_minmax(a, x); a = a + x.lo * 1e-300);
    MEASURE(a = __drcp_rn(a));
    MEASURE(a = __ddiv_rn(1.0, a));
    MEASURE(a = __ddiv_rd(1.0, a));
    MEASURE(a = __fma_rn(-a, b, 1.0) + a);
    out[threadIdx.x] = a + x.lo + x.hi;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 32 * 8);
    cudaMallocManaged(&cyc, 64 * 8);
    for (int r = 0; r < 2; r++) k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    cudaDeviceSynchronize();
    const char* names[] = {"dadd_rd", "dmul_ru", "fmin(+dep)", "sel_min(+dep)", "Fast::mul(+dep)", "mul4 fmin",
                           "mul4 sel", "gmul", "pmul_minmax", "drcp_rn", "ddiv_rn(1,x)", "ddiv_rd(1,x)", "fma+add"};
    for (int i = 0; i < 13; i++) printf("%-18s %lld cycles\n", names[i], cyc[i]);
    return 0;
}
