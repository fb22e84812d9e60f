// spmm_inst.cuh -- body of one spmm_inst_*.cu translation unit: defines
// dispatch_inst<FG_RED, FG_OPSET> (spmm_impl.cuh) for the reducer FG_RED and
// the message-op set FG_OPSET (0: copy_u, u_mul_e; 1: u_add_e, copy_e).
#include "spmm_impl.cuh"

namespace fgspmm {
namespace {

template <int G, int NV>
fg_status inst_op(const Args& A, int op, cudaStream_t st) {
#if FG_OPSET == 0
    if (op == OP_COPY) return launch_t<G, NV, OP_COPY, FG_RED>(A, st);
    if (op == OP_UMULE) return launch_t<G, NV, OP_UMULE, FG_RED>(A, st);
    return launch_t<G, NV, OP_UMULE_GEN, FG_RED>(A, st);
#else
    if (op == OP_UADDE) return launch_t<G, NV, OP_UADDE, FG_RED>(A, st);
    return launch_t<G, NV, OP_COPYE, FG_RED>(A, st);
#endif
}

}  // namespace

template <>
fg_status dispatch_inst<FG_RED, FG_OPSET>(const Args& A, int G, int NV, int op, cudaStream_t st) {
    switch (G) {   // the (G, NV) pairs launch_spmm_gather (spmm.cu) chooses
        case 1: return inst_op<1, 1>(A, op, st);
        case 2: return inst_op<2, 1>(A, op, st);
        case 4: return inst_op<4, 1>(A, op, st);
        case 8: return inst_op<8, 1>(A, op, st);
        case 16: return inst_op<16, 1>(A, op, st);
        default:
            if (NV == 1) return inst_op<32, 1>(A, op, st);
            if (NV == 2) return inst_op<32, 2>(A, op, st);
            if (NV == 3) return inst_op<32, 3>(A, op, st);
            return inst_op<32, 4>(A, op, st);
    }
}

#if FG_OPSET == 0
// fp32 chunk pairs (32-byte loads): the (G, NV) the host chose from F8 = F4 / 2
template <>
fg_status dispatch_pair32<FG_RED>(const Args& A, int G, int NV, int op, cudaStream_t st) {
    (void)op;   // copy_u only
    switch (G) {
        case 1: return launch_t<1, 2, OP_COPY, FG_RED, false, true>(A, st);
        case 2: return launch_t<2, 2, OP_COPY, FG_RED, false, true>(A, st);
        case 4: return launch_t<4, 2, OP_COPY, FG_RED, false, true>(A, st);
        case 8: return launch_t<8, 2, OP_COPY, FG_RED, false, true>(A, st);
        case 16: return launch_t<16, 2, OP_COPY, FG_RED, false, true>(A, st);
        default:
            if (NV == 2) return launch_t<32, 2, OP_COPY, FG_RED, false, true>(A, st);
            return launch_t<32, 4, OP_COPY, FG_RED, false, true>(A, st);   // wider rows: column tiles (grid.y)
    }
}
#endif

}  // namespace fgspmm
