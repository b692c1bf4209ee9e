// k_final instantiations for P in [5, 8] (see tc_final.cuh).
#include "tc_final.cuh"

namespace tc {
cudaError_t launch_final_p5_8(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid,
                                 size_t smem, cudaStream_t st) {
    switch (P) {
        case 5: return launch_final_t<5>(dump, A, cc, grid, smem, st);
        case 6: return launch_final_t<6>(dump, A, cc, grid, smem, st);
        case 7: return launch_final_t<7>(dump, A, cc, grid, smem, st);
        case 8: return launch_final_t<8>(dump, A, cc, grid, smem, st);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace tc
