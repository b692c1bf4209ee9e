// k_final instantiations for P in [9, 12] (see tc_final.cuh).
#include "tc_final.cuh"

namespace tc {
cudaError_t launch_final_p9_12(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid,
                                 size_t smem, cudaStream_t st) {
    switch (P) {
        case 9: return launch_final_t<9>(dump, A, cc, grid, smem, st);
        case 10: return launch_final_t<10>(dump, A, cc, grid, smem, st);
        case 11: return launch_final_t<11>(dump, A, cc, grid, smem, st);
        case 12: return launch_final_t<12>(dump, A, cc, grid, smem, st);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace tc
