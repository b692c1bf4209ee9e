// tc_final.cuh -- k_final launcher template, instantiated for prime-count
// ranges in tc_final_*.cu (separate translation units compile in parallel).
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include "tc_kernels.cuh"

#ifndef TC_FINAL_384
#define TC_FINAL_384 1     // 384-thread CTAs (2 per SM at up to 85 registers) where the rounds' items divide evenly
#endif

namespace tc {

template <int P>
cudaError_t launch_final_t(bool dump, FinalArgs A, const CrtConst& cc, unsigned grid, size_t smem,
                           cudaStream_t st) {
    // a tile too large for two CTAs per SM gets 32 warps in one CTA
    const char* ev = getenv("TC_FINAL_THREADS");
    const int ft = ev && *ev ? atoi(ev) : 0;
    const bool big = smem > 112 * 1024 || ft == 1024;
    cudaError_t e = cudaSuccess;
#define TC_LAUNCH(DUMP, NT)                                                                       \
    do {                                                                                          \
        e = ensure_smem((const void*)k_final<P, DUMP, NT>, smem);                                \
        if (e != cudaSuccess) return e;                                                           \
        k_final<P, DUMP, NT><<<grid, NT, smem, st>>>(A, cc);                                     \
    } while (0)
    static const int stage_env = [] { const char* v = getenv("TC_CO_STAGE"); return v && *v ? atoi(v) : 1; }();
    if (dump) { if (big) TC_LAUNCH(true, 1024); else TC_LAUNCH(true, 512); }
    else if (big) {
        const size_t stage = (size_t)(1024 / 32) * co_stage_words<P>() * 4;    // one CTA per SM anyway
        if (stage_env && P <= 8 && A.co_aw > 0 && smem + stage <= 224 * 1024) { A.co_stage = 1; smem += stage; }
        TC_LAUNCH(false, 1024);
    }
    // 256 threads when >= 3 CTAs fit an SM (C3: 22.7 -> 19.2 ms), 512 at 2 per SM (C2)
    else if (ft == 256 || (ft == 0 && smem <= 76 * 1024)) TC_LAUNCH(false, 256);
#if TC_FINAL_384
    // 384 threads (80 registers instead of 64: fewer spills in the CRT, smaller barriers) when the
    // multi-tile rounds' P n / 16 groups divide evenly over them (C3: k_final 10.10 -> 9.70 ms;
    // C2's 1280 groups do not: 142 -> 150 us)
    else if (ft == 384 || (ft == 0 && A.multi && P >= 2 && A.lgL >= 5 &&
                           ((size_t)P << (A.lgL + A.yl - 4)) % 384 == 0)) TC_LAUNCH(false, 384);
#endif
    else {
        // 512 threads: a dedicated region for the grouped ConvertOut's per-warp
        // staging of product words when it still leaves two CTAs per SM (else
        // the kernel stages in the warps' dead limb slots: C2 152 vs 156 us)
        const size_t stage = (size_t)(512 / 32) * co_stage_words<P>() * 4;
        if (stage_env && P <= 8 && A.co_aw > 0 && smem + stage <= 112 * 1024) { A.co_stage = 1; smem += stage; }
        TC_LAUNCH(false, 512);
    }
#undef TC_LAUNCH
    return cudaGetLastError();
}

}  // namespace tc
