// kat.cu -- rb_interval_kat: the device interval layer (interval.cuh, the guarded
// helpers of kernels.cuh) on caller-supplied operands, so the tests can compare
// each policy with the reference's own known answers (tests/golden/kat_interval.npz,
// generated from rootbox/interval.py:66-432 by make_golden.py).
#define RB_KINST_TU 1  // the shared non-template kernels are defined in engine.cu
#include "../../include/rootbox_b200.h"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <vector>

using namespace rb;

namespace {

__global__ void k_interval_kat(int op, int policy, int64_t m, const double* xl, const double* xh, const double* yl,
                               const double* yh, double* o0, double* o1, double* o2, double* o3, int8_t* kind) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = xl[i], b = yl[i];
        const ival x = mk(xl[i], xh[i]), y = mk(yl[i], yh[i]);
        double r0 = CUDART_NAN, r1 = CUDART_NAN, r2 = CUDART_NAN, r3 = CUDART_NAN;
        int k8 = -1;
        if (op >= 0 && op <= 5) {
            if (policy == 1) {
                switch (op) {
                    case 0: r0 = Exact::add_rd(a, b); break;
                    case 1: r0 = Exact::add_ru(a, b); break;
                    case 2: r0 = Exact::mul_rd(a, b); break;
                    case 3: r0 = Exact::mul_ru(a, b); break;
                    case 4: r0 = div_rd(a, b); break;
                    default: r0 = div_ru(a, b); break;
                }
            } else if (policy == 2 && (op == 2 || op == 3)) {
                const ival p = gmul(mk(a, a), mk(b, b));
                r0 = op == 2 ? p.lo : p.hi;
            } else {
                switch (op) {
                    case 0: r0 = __dadd_rd(a, b); break;
                    case 1: r0 = __dadd_ru(a, b); break;
                    case 2: r0 = __dmul_rd(a, b); break;
                    case 3: r0 = __dmul_ru(a, b); break;
                    case 4: r0 = policy == 2 ? div_rd(a, b) : __ddiv_rd(a, b); break;
                    default: r0 = policy == 2 ? div_ru(a, b) : __ddiv_ru(a, b); break;
                }
            }
        } else if (op == 10) {
            const ival p = policy == 0 ? Fast::mul(x, y) : (policy == 1 ? Exact::mul(x, y) : gmul(x, y));
            r0 = p.lo;
            r1 = p.hi;
        } else if (op == 11) {
            if (!contains_zero(x)) {
                if (policy == 0) {
                    r0 = recip_dir(x.hi, false);
                    r1 = recip_dir(x.lo, true);
                } else {
                    r0 = div_rd(1.0, x.hi);
                    r1 = div_ru(1.0, x.lo);
                }
            }
        } else if (op == 12) {
            r0 = mid_of(x.lo, x.hi);
        } else if (op >= 20 && op < 30) {
            const ival p = policy == 0 ? Fast::pow(x, op - 20) : Exact::pow(x, op - 20);
            r0 = p.lo;
            r1 = p.hi;
        } else if (op == 40) {
            ival q0 = mk(CUDART_NAN, CUDART_NAN), q1 = mk(CUDART_NAN, CUDART_NAN);
            if (policy == 0) k8 = div_extended_fast(x, y, q0, q1);
            else k8 = div_extended(x, y, q0, q1, policy == 1);
            r0 = q0.lo;
            r1 = q0.hi;
            r2 = q1.lo;
            r3 = q1.hi;
            if (k8 == DIV_EMPTY) r0 = r1 = CUDART_NAN;
            if (k8 != DIV_SPLIT) r2 = r3 = CUDART_NAN;
        }
        o0[i] = r0;
        o1[i] = r1;
        o2[i] = r2;
        o3[i] = r3;
        kind[i] = (int8_t)k8;
    }
}

}  // namespace

extern "C" int rb_interval_kat(int device, int op, int policy, int64_t m, const double* xl, const double* xh,
                               const double* yl, const double* yh, double* o0, double* o1, double* o2, double* o3,
                               int8_t* kind) {
    if (m < 0 || policy < 0 || policy > 2) return RB_ERR_ARG;
    if (m == 0) return RB_OK;
    if (!xl || !xh || !yl || !yh || !o0 || !o1 || !o2 || !o3 || !kind) return RB_ERR_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return RB_ERR_CUDA;
    const size_t B = sizeof(double) * (size_t)m;
    double* d = nullptr;
    int8_t* dk = nullptr;
    if (cudaMalloc(&d, 8 * B) != cudaSuccess) {
        cudaGetLastError();
        return RB_ERR_NOMEM;
    }
    if (cudaMalloc(&dk, (size_t)m) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(d);
        return RB_ERR_NOMEM;
    }
    double* in[4] = {d, d + m, d + 2 * m, d + 3 * m};
    double* out[4] = {d + 4 * m, d + 5 * m, d + 6 * m, d + 7 * m};
    cudaError_t e = cudaSuccess;
    const double* hin[4] = {xl, xh, yl, yh};
    for (int k = 0; k < 4 && e == cudaSuccess; k++) e = cudaMemcpy(in[k], hin[k], B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        k_interval_kat<<<148 * 4, 256>>>(op, policy, m, in[0], in[1], in[2], in[3], out[0], out[1], out[2], out[3],
                                          dk);
        e = cudaGetLastError();
    }
    double* hout[4] = {o0, o1, o2, o3};
    for (int k = 0; k < 4 && e == cudaSuccess; k++) e = cudaMemcpy(hout[k], out[k], B, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(kind, dk, (size_t)m, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(dk);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return RB_ERR_CUDA;
    }
    return RB_OK;
}
