// Cost of dependent kernel nodes inside a CUDA-graph WHILE body on this GPU (dev aid).
// body = K tiny kernels (1 block or 148 blocks), optional IF node; the last kernel
// decrements a device counter and sets the WHILE condition.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_touch(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p + 1, 1); }
__global__ void k_last(int* p, cudaGraphConditionalHandle h) {
    if (threadIdx.x == 0 && blockIdx.x == 0) { int r = --p[0]; cudaGraphSetConditional(h, r > 0); }
}
__global__ void k_setif(cudaGraphConditionalHandle h) { if (threadIdx.x == 0 && blockIdx.x == 0) cudaGraphSetConditional(h, 0); }
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
    int* d; CK(cudaMalloc(&d, 64));
    cudaStream_t st; CK(cudaStreamCreate(&st));
    for (int blocks : {1, 148, 592}) for (int withif = 0; withif < 2; withif++) for (int K = 1; K <= 6; K++) {
        cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle hw; CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = hw;
        cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
        cudaGraphNode_t wn; CK(cudaGraphAddNode(&wn, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < K - 1; k++) k_touch<<<blocks, 256, 0, st>>>(d);
        if (withif) {
            cudaGraphConditionalHandle hi; CK(cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault));
            k_setif<<<1, 32, 0, st>>>(hi);
            cudaStreamCaptureStatus cs; const cudaGraphNode_t* deps; size_t nd; cudaGraph_t cg;
            CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
            cudaGraphNodeParams ip = {}; ip.type = cudaGraphNodeTypeConditional; ip.conditional.handle = hi;
            ip.conditional.type = cudaGraphCondTypeIf; ip.conditional.size = 1;
            cudaGraphNode_t in; CK(cudaGraphAddNode(&in, cg, deps, nd, &ip));
            CK(cudaStreamUpdateCaptureDependencies(st, &in, 1, cudaStreamSetCaptureDependencies));
            cudaGraph_t ib = ip.conditional.phGraph_out[0];
            cudaGraphNode_t kn; cudaKernelNodeParams kp = {}; void* args[] = {&d};
            kp.func = (void*)k_touch; kp.gridDim = dim3(blocks); kp.blockDim = dim3(256); kp.kernelParams = args;
            CK(cudaGraphAddKernelNode(&kn, ib, nullptr, 0, &kp));
        }
        k_last<<<blocks, 256, 0, st>>>(d, hw);
        cudaGraph_t tmp; CK(cudaStreamEndCapture(st, &tmp));
        cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge, g, 0));
        const int iters = 1000;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        float best = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            int h0[2] = {iters, 0}; CK(cudaMemcpy(d, h0, 8, cudaMemcpyHostToDevice));
            cudaEventRecord(a, st); CK(cudaGraphLaunch(ge, st)); cudaEventRecord(b, st); CK(cudaStreamSynchronize(st));
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("blocks %3d if %d K %d: %.2f us per WHILE iteration (%.2f us per node)\n", blocks, withif, K,
               best * 1e3 / iters, best * 1e3 / iters / (K + withif));
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    return 0;
}
