// Dependent-chain latency of the FP64 building blocks on sm_100a (dev tool).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../../paper_1802_00330_b200/csrc lat.cu -o lat
#include <cstdio>
#include "kernels.cuh"
using namespace rb;

#define ITERS 256
__global__ void k_lat(double* out, long long* cyc, double a0, double b0) {
    double a = a0 + threadIdx.x * 1e-300, b = b0;
    ival x = mk(a, a + 1.0), y = mk(b - 1.0, b);
    long long t0, t1;
    int k = 0;
#define MEASURE(name, body)                                   \
    t0 = clock64();                                           \
    for (int i = 0; i < ITERS; i++) { body; }                 \
    t1 = clock64();                                           \
    if (threadIdx.x == 0) cyc[k] = (t1 - t0) / ITERS;         \
    k++;
    MEASURE("dadd_rd", a = __dadd_rd(a, b));
    MEASURE("dmul_ru", a = __dmul_ru(a, b));
    MEASURE("dfma_rn", a = __fma_rn(a, b, 1e-300));
    MEASURE("fmin", a = fmin(a, b) + 1e-300);
    MEASURE("ddiv_rn", a = __ddiv_rn(a, b));
    MEASURE("drcp_rn", a = __drcp_rn(a));
    MEASURE("ddiv_rd", a = __ddiv_rd(1.0, a));
    MEASURE("drcp_rd", a = __drcp_rd(a));
    MEASURE("Fast::add", x = Fast::add(x, y));
    MEASURE("pmul_minmax", x = pmul_minmax(a, x));
    MEASURE("Fast::mul", x = Fast::mul(x, y));
    MEASURE("gmul", x = gmul(x, y));
    MEASURE("shfl", a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31));
    MEASURE("mid_of", a = mid_of(a, b));
    out[threadIdx.x] = a + x.lo + x.hi;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 32 * 8);
    cudaMallocManaged(&cyc, 64 * 8);
    k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    cudaDeviceSynchronize();
    const char* names[] = {"dadd_rd", "dmul_ru", "dfma_rn", "fmin+dadd", "ddiv_rn", "drcp_rn", "ddiv_rd(1,x)",
                           "drcp_rd", "Fast::add", "pmul_minmax", "Fast::mul", "gmul", "shfl", "mid_of"};
    for (int i = 0; i < 14; i++) printf("%-14s %lld cycles\n", names[i], cyc[i]);
    return 0;
}
