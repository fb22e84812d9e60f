// spmm_inst_x16.cuh -- body of spmm_inst_x16_{sum,max}.cu: gSpMM instantiations with bf16 storage of the source
// features X (row f4: "bf16 feature storage"): copy_u / u_mul_e x {sum, max}.
// Gathers read 8 bytes per 4 features instead of 16; the message and the
// reduction are fp32 exactly as in the fp32 path (bf16 -> fp32 is exact).
#include "spmm_impl.cuh"

namespace fgspmm {
namespace {

template <int G, int NV, int RED, bool PAIR = false>
fg_status inst_op_x16(const Args& A, int op, cudaStream_t st) {
    if (op == OP_COPY) return launch_t<G, NV, OP_COPY, RED, true, PAIR>(A, st);
    if (op == OP_UMULE) return launch_t<G, NV, OP_UMULE, RED, true, PAIR>(A, st);
    return launch_t<G, NV, OP_UMULE_GEN, RED, true, PAIR>(A, st);
}

template <int RED>
fg_status dispatch_x16_impl(const Args& A, int G, int NV, int op, bool pair, cudaStream_t st) {
    if (pair) {   // 16-byte loads of chunk pairs: G lanes x NV/2 pairs
        switch (G) {
            case 1: return inst_op_x16<1, 2, RED, true>(A, op, st);
            case 2: return inst_op_x16<2, 2, RED, true>(A, op, st);
            case 4: return inst_op_x16<4, 2, RED, true>(A, op, st);
            case 8: return inst_op_x16<8, 2, RED, true>(A, op, st);
            case 16: return inst_op_x16<16, 2, RED, true>(A, op, st);
            default:
                if (NV == 2) return inst_op_x16<32, 2, RED, true>(A, op, st);
                return inst_op_x16<32, 4, RED, true>(A, op, st);   // wider rows: column tiles (grid.y)
        }
    }
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

// one reducer per translation unit (spmm_inst_x16_sum.cu / _max.cu: parallel builds)
template <>
fg_status dispatch_x16<FG_RED>(const Args& A, int G, int NV, int op, bool pair, cudaStream_t st) {
    return dispatch_x16_impl<FG_RED>(A, G, NV, op, pair, st);
}

}  // namespace fgspmm
