// spmm_inst_x16.cu -- gSpMM instantiations with bf16 storage of the source
// features X (row f4: "bf16 feature storage"): copy_u / u_mul_e x {sum, max}.
// Gathers read 8 bytes per 4 features instead of 16; the message and the
// reduction are fp32 exactly as in the fp32 path (bf16 -> fp32 is exact).
#include "spmm_impl.cuh"

namespace fgspmm {
namespace {

template <int G, int NV, int RED>
fg_status inst_op_x16(const Args& A, int op, cudaStream_t st) {
    if (op == OP_COPY) return launch_t<G, NV, OP_COPY, RED, true>(A, st);
    if (op == OP_UMULE) return launch_t<G, NV, OP_UMULE, RED, true>(A, st);
    return launch_t<G, NV, OP_UMULE_GEN, RED, true>(A, st);
}

template <int RED>
fg_status dispatch_x16_impl(const Args& A, int G, int NV, int op, cudaStream_t st) {
    switch (G) {
        case 1: return inst_op_x16<1, 1, RED>(A, op, st);
        case 2: return inst_op_x16<2, 1, RED>(A, op, st);
        case 4: return inst_op_x16<4, 1, RED>(A, op, st);
        case 8: return inst_op_x16<8, 1, RED>(A, op, st);
        case 16: return inst_op_x16<16, 1, RED>(A, op, st);
        default:
            if (NV == 1) return inst_op_x16<32, 1, RED>(A, op, st);
            if (NV == 2) return inst_op_x16<32, 2, RED>(A, op, st);
            if (NV == 3) return inst_op_x16<32, 3, RED>(A, op, st);
            return inst_op_x16<32, 4, RED>(A, op, st);
    }
}

}  // namespace

template <>
fg_status dispatch_x16<R_SUM>(const Args& A, int G, int NV, int op, cudaStream_t st) {
    return dispatch_x16_impl<R_SUM>(A, G, NV, op, st);
}
template <>
fg_status dispatch_x16<R_MAX>(const Args& A, int G, int NV, int op, cudaStream_t st) {
    return dispatch_x16_impl<R_MAX>(A, G, NV, op, st);
}

}  // namespace fgspmm
