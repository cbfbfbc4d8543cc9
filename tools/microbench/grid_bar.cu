// Latency of a hand-rolled grid barrier over G resident blocks vs cooperative
// groups grid.sync (dev aid).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// monotone counter: arrive with atomicAdd, wait until it reaches (it+1)*G
__global__ void k_bar(unsigned* bar, int iters, unsigned long long* out) {
    unsigned long long t0 = gt();
    for (int it = 0; it < iters; it++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned target = (unsigned)(it + 1) * gridDim.x;
            __threadfence();
            atomicAdd(bar, 1u);
            while (ld_acq(bar) < target) {
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = gt() - t0;
}
__global__ void k_cg(int iters, unsigned long long* out) {
    cg::grid_group g = cg::this_grid();
    unsigned long long t0 = gt();
    for (int it = 0; it < iters; it++) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = gt() - t0;
}
int main() {
    unsigned* bar;
    unsigned long long* out;
    cudaMalloc(&bar, 64);
    cudaMalloc(&out, 8);
    int iters = 2000;
    for (int G : {148, 296, 592}) {
        unsigned long long t = 0;
        for (int rep = 0; rep < 2; rep++) {
            cudaMemset(bar, 0, 64);
            k_bar<<<G, 256>>>(bar, iters, out);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(&t, out, 8, cudaMemcpyDeviceToHost);
        printf("counter barrier, %d blocks: %.3f us (%s)\n", G, t * 1e-3 / iters, cudaGetErrorString(cudaGetLastError()));
        void* args[] = {(void*)&iters, (void*)&out};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k_cg, G, 256, args, 0, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(&t, out, 8, cudaMemcpyDeviceToHost);
        printf("cg grid.sync, %d blocks: %.3f us (%s)\n", G, t * 1e-3 / iters, cudaGetErrorString(e));
    }
    return 0;
}
