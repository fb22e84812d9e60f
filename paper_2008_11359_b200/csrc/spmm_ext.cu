// spmm_ext.cu -- the remaining DGL message builtins on the gathered-message
// gSpMM template (FeatGraph plugs
// into DGL's builtin message / reduce family):
//   u_add_e: phi[h,d] = X[u][h][d] + E[e][h]     (E [nnz][H], broadcast over D)
//   copy_e : phi      = E[e]                      (E [nnz][H*D]; no source gather)
// x {sum, max, min, mean}.  Same schedule as spmm.cu (spmm_impl.cuh); a separate
// translation unit so the instantiations compile in parallel.
#include "spmm_impl.cuh"

namespace fgspmm {

template <int G, int NV>
fg_status dispatch_ext(const Args& A, int op, int red, cudaStream_t st) {
    if (op == OP_UADDE) return dispatch_red<G, NV, OP_UADDE>(A, red, st);
    if (op == OP_COPYE) return dispatch_red<G, NV, OP_COPYE>(A, red, st);
    return fgk::set_error(FG_EINVAL, "fg_spmm: bad message op %d", op);
}

template fg_status dispatch_ext<1, 1>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<2, 1>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<4, 1>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<8, 1>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<16, 1>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<32, 1>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<32, 2>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<32, 3>(const Args&, int, int, cudaStream_t);
template fg_status dispatch_ext<32, 4>(const Args&, int, int, cudaStream_t);

}  // namespace fgspmm
