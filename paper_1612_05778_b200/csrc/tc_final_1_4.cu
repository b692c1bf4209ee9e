// k_final instantiations for P in [1, 4] (see tc_final.cuh).
#include "tc_final.cuh"

namespace tc {
cudaError_t launch_final_p1_4(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid,
                                 size_t smem, cudaStream_t st) {
    switch (P) {
        case 1: return launch_final_t<1>(dump, A, cc, grid, smem, st);
        case 2: return launch_final_t<2>(dump, A, cc, grid, smem, st);
        case 3: return launch_final_t<3>(dump, A, cc, grid, smem, st);
        case 4: return launch_final_t<4>(dump, A, cc, grid, smem, st);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace tc
