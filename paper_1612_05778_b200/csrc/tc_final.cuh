// tc_final.cuh -- k_final launcher template, instantiated for prime-count
// ranges in tc_final_*.cu (separate translation units compile in parallel).
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include "tc_kernels.cuh"

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
