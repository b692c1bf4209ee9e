// k_final instantiations for P in [13, 16] (see tc_final.cuh).
#include "tc_final.cuh"

namespace tc {
cudaError_t launch_final_p13_16(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid,
                                 size_t smem, cudaStream_t st) {
    switch (P) {
        case 13: return launch_final_t<13>(dump, A, cc, grid, smem, st);
        case 14: return launch_final_t<14>(dump, A, cc, grid, smem, st);
        case 15: return launch_final_t<15>(dump, A, cc, grid, smem, st);
        case 16: return launch_final_t<16>(dump, A, cc, grid, smem, st);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace tc
