// kinst.cu -- explicit instantiation of the per-dimension launchers (and their
// kernels) for dimensions RB_K0 .. RB_K1; compiled once per range (Makefile).
#define RB_KINST_TU 1
#include "launchers.cuh"

#ifndef RB_K0
#error "build with -DRB_K0=<first dimension> -DRB_K1=<last dimension>"
#endif

#define RB_INST(K) RB_LAUNCHERS(template struct, K)
#if RB_K0 <= 1 && 1 <= RB_K1
RB_INST(1)
#endif
#if RB_K0 <= 2 && 2 <= RB_K1
RB_INST(2)
#endif
#if RB_K0 <= 3 && 3 <= RB_K1
RB_INST(3)
#endif
#if RB_K0 <= 4 && 4 <= RB_K1
RB_INST(4)
#endif
#if RB_K0 <= 5 && 5 <= RB_K1
RB_INST(5)
#endif
#if RB_K0 <= 6 && 6 <= RB_K1
RB_INST(6)
#endif
#if RB_K0 <= 7 && 7 <= RB_K1
RB_INST(7)
#endif
#if RB_K0 <= 8 && 8 <= RB_K1
RB_INST(8)
#endif
#if RB_K0 <= 9 && 9 <= RB_K1
RB_INST(9)
#endif
#if RB_K0 <= 10 && 10 <= RB_K1
RB_INST(10)
#endif
#if RB_K0 <= 11 && 11 <= RB_K1
RB_INST(11)
#endif
#if RB_K0 <= 12 && 12 <= RB_K1
RB_INST(12)
#endif
#if RB_K0 <= 13 && 13 <= RB_K1
RB_INST(13)
#endif
#if RB_K0 <= 14 && 14 <= RB_K1
RB_INST(14)
#endif
#if RB_K0 <= 15 && 15 <= RB_K1
RB_INST(15)
#endif
#if RB_K0 <= 16 && 16 <= RB_K1
RB_INST(16)
#endif
