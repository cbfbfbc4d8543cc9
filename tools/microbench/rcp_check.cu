// recip_dir == __ddiv_rd/ru(1, y) on random normal y (dev check)
#include <cstdio>
#include <cstdlib>
#include "kernels.cuh"
using namespace rb;
__global__ void k(const double* y, int n, unsigned long long* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = y[i];
        if (recip_dir(v, false) != __ddiv_rd(1.0, v) || recip_dir(v, true) != __ddiv_ru(1.0, v)) atomicAdd(bad, 1ull);
    }
}
int main() {
    const int n = 1 << 24;
    double* h = (double*)malloc(n * 8);
    srand(1);
    for (int i = 0; i < n; i++) {
        unsigned long long m = ((unsigned long long)rand() << 31) ^ rand() ^ ((unsigned long long)rand() << 52);
        double f = 1.0 + (double)(m & ((1ull << 52) - 1)) / (double)(1ull << 52);
        if (i % 7 == 0) f = (double)(1 + rand() % 4096);  // exact reciprocals too
        int e = rand() % 1900 - 950;
        h[i] = ldexp(f, e) * ((rand() & 1) ? -1 : 1);
    }
    double* d; unsigned long long* bad;
    cudaMalloc(&d, n * 8); cudaMallocManaged(&bad, 8); *bad = 0;
    cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
    k<<<1024, 256>>>(d, n, bad);
    cudaDeviceSynchronize();
    printf("recip_dir mismatches: %llu of %d\n", *bad, n);
    return 0;
}
