// codegen.h -- system-specialised kernels.
//
// The reference compiles a system into per-equation term tuples (compile_system,
// _batch.py:144-164) that its inclusion functions walk term by term.  The table
// kernels in kernels.cuh do the same walk on the device (an interpreter over flat
// tables in shared memory).  Here each polynomial of F is instead emitted as
// straight-line CUDA -- the same interval operations on the same operands in the
// same order, so the results are bit-identical -- and compiled for sm_100a with
// NVRTC at engine creation.  The generated translation unit includes kernels.cuh
// and instantiates the filter kernels with the generated evaluator (GenEval); no
// table copy, no per-term decode, and the terms of an equation are independent
// instructions the scheduler can overlap.
//
// Compiled cubins are cached on disk (key: generated source + headers + NVRTC
// version), so a system is compiled once per machine; build() fills the cache for
// the benchmark and test systems.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace rbg {

struct SystemTerms {  // host copy of rb_system's polynomial tables
    int n = 0;
    std::vector<int32_t> poly_off;  // [n + n*n + 1]
    std::vector<double> coeff;
    std::vector<int32_t> fac_off;
    std::vector<uint8_t> fac_var, fac_exp;
};

struct Compiled {
    std::string key;
    std::vector<char> cubin;
    std::string name_cf;      // lowered names of the instantiated kernels
    std::string name_filter;
    std::string name_hs_fused;
    std::string name_hs_eval;
    std::string name_hs_tile;
    std::string name_filter_tab;
    std::string name_filter_wt;
};

// CUDA source of the specialised translation unit
std::string source(const SystemTerms& s);

// compile (or read from the cache); returns false with a reason on failure
bool compile(const SystemTerms& s, Compiled& out, std::string& err);
// read from the cache only; false when not compiled yet
bool cached(const SystemTerms& s, Compiled& out);

struct Loaded {
    bool ok = false;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t cf = nullptr;      // k_classify_filter<N, GenEval>
    cudaKernel_t filter = nullptr;  // k_filter<N, GenEval>
    cudaKernel_t hs_fused = nullptr;  // k_hs_fused<N, GenEval>
    cudaKernel_t hs_eval = nullptr;   // k_hs_eval<N, GenEval>
    cudaKernel_t hs_tile = nullptr;   // k_hs_tile<N, GenEval>
    cudaKernel_t filter_tab = nullptr;  // k_filter_tab<N, GenEval>
    cudaKernel_t filter_wt = nullptr;   // k_filter_wt<N, GenEval>
};

// load the compiled kernels into the current device's context (process-wide cache)
bool load(const Compiled& c, int device, Loaded& out, std::string& err);

}  // namespace rbg
