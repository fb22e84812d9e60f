// spmm_inst_sum_base.cu -- gSpMM instantiations: reducer sum, copy_u / u_mul_e.
#define FG_RED R_SUM
#define FG_OPSET 0
#include "spmm_inst.cuh"

namespace fgspmm {
fg_status launch_hybrid(const Args& A, int G, cudaStream_t st) {
    switch (G) {
        case 1: return launch_t<1, 1, OP_COPY, R_SUM, false, false, true>(A, st);
        case 2: return launch_t<2, 1, OP_COPY, R_SUM, false, false, true>(A, st);
        case 4: return launch_t<4, 1, OP_COPY, R_SUM, false, false, true>(A, st);
        case 8: return launch_t<8, 1, OP_COPY, R_SUM, false, false, true>(A, st);
        case 16: return launch_t<16, 1, OP_COPY, R_SUM, false, false, true>(A, st);
        default: return launch_t<32, 1, OP_COPY, R_SUM, false, false, true>(A, st);
    }
}

fg_status launch_seg_pass(const Args& A, int G, int NV, cudaStream_t st) {
    switch (G) {
        case 1: return launch_t<1, 1, OP_UMULE, R_SUM, false, false, false, true>(A, st);
        case 2: return launch_t<2, 1, OP_UMULE, R_SUM, false, false, false, true>(A, st);
        case 4: return launch_t<4, 1, OP_UMULE, R_SUM, false, false, false, true>(A, st);
        case 8: return launch_t<8, 1, OP_UMULE, R_SUM, false, false, false, true>(A, st);
        case 16: return launch_t<16, 1, OP_UMULE, R_SUM, false, false, false, true>(A, st);
        default:
            if (NV == 1) return launch_t<32, 1, OP_UMULE, R_SUM, false, false, false, true>(A, st);
            if (NV == 2) return launch_t<32, 2, OP_UMULE, R_SUM, false, false, false, true>(A, st);
            if (NV == 3) return launch_t<32, 3, OP_UMULE, R_SUM, false, false, false, true>(A, st);
            return launch_t<32, 4, OP_UMULE, R_SUM, false, false, false, true>(A, st);
    }
}
}  // namespace fgspmm
