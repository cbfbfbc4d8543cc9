// Latency of a dependent global atomicAdd with return, one thread (dev aid).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void k(unsigned long long* p, int iters, int stride, unsigned long long* out) {
    unsigned long long v = 0;
    const unsigned long long t0 = gt();
    for (int i = 0; i < iters; i++) v = atomicAdd(p + (v & 1) * stride + (size_t)i * stride, 1ull);
    const unsigned long long t1 = gt();
    out[0] = t1 - t0;
    out[1] = v;
}
__global__ void k_ld(unsigned long long* p, int iters, unsigned long long* out) {
    unsigned long long v = 0;
    const unsigned long long t0 = gt();
    for (int i = 0; i < iters; i++) v = __ldcg(p + (v & 1) + (size_t)i * 16);
    const unsigned long long t1 = gt();
    out[0] = t1 - t0;
    out[1] = v;
}
int main() {
    unsigned long long *p, *out, h[2];
    cudaMalloc(&p, 1 << 26);
    cudaMemset(p, 0, 1 << 26);
    cudaMalloc(&out, 16);
    for (int stride : {0, 16}) {
        k<<<1, 1>>>(p, 1000, stride, out);
        k<<<1, 1>>>(p, 1000, stride, out);
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("atomicAdd with return, stride %d: %.3f us each\n", stride, h[0] * 1e-3 / 1000);
    }
    k_ld<<<1, 1>>>(p, 1000, out);
    k_ld<<<1, 1>>>(p, 1000, out);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("dependent ld.cg (L2): %.3f us each\n", h[0] * 1e-3 / 1000);
    return 0;
}
