// sddmm_ext.cu -- elementwise gSDDMM edge functions:
// the u_OP_v members of the DGL builtin family FeatGraph plugs into
// (PAPER.md P:372-375), Eq. (2) with
//     out[eid(p)][j] = X[u][j] OP Y[v][j],   OP in {+, -, *},  p = (u -> v).
//
// Unlike u_dot_v there is no reduction: the output is an [nnz][F] edge tensor,
// so the kernel is bound by the m*F*4 bytes it writes (plus the X[u] gather).
// Traversal: one warp per SDDMM work unit (<= unit_chunk edges of one
// destination row, the fg_graph unit table); the unit's (edge, column) pairs
// are flattened so consecutive lanes touch consecutive float4 columns of the
// same edge -- coalesced X[u] reads and, with identity edge ids, one
// contiguous streaming store (st.global.cs) for the whole unit at any F.
#include "fg_internal.h"

namespace {

constexpr int THREADS = 256;
enum { BOP_ADD = 1, BOP_SUB = 2, BOP_MUL = 3 };   // == fg_edge_op values

template <int OP>
__device__ __forceinline__ float bop(float x, float y) {
    if constexpr (OP == BOP_ADD) return __fadd_rn(x, y);
    else if constexpr (OP == BOP_SUB) return __fsub_rn(x, y);
    else return __fmul_rn(x, y);
}

template <int OP>
__global__ void __launch_bounds__(THREADS) sddmm_binary_kernel(
    const int32_t* __restrict__ unit_row, const int64_t* __restrict__ unit_p0, int64_t n_units, int chunk,
    const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx, const int32_t* __restrict__ eid,
    unsigned F4, const float4* __restrict__ X, const float4* __restrict__ Y, float4* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    if (w >= n_units) return;
    const int64_t v = unit_row[w];
    const int64_t s = unit_p0[w];
    const int64_t e = min(s + chunk, row_ptr[v + 1]);
    const float4* yr = Y + v * F4;
    const unsigned total = unsigned(e - s) * F4;   // <= chunk * F4 < 2^31 (host-checked)
    for (unsigned q = lane; q < total; q += 32) {
        const unsigned t = q / F4, c = q - t * F4;
        const int64_t p = s + t;
        const float4 x = __ldg(X + int64_t(__ldg(col_idx + p)) * F4 + c);
        const float4 y = __ldg(yr + c);
        const float4 r = make_float4(bop<OP>(x.x, y.x), bop<OP>(x.y, y.y), bop<OP>(x.z, y.z), bop<OP>(x.w, y.w));
        const int64_t ed = eid ? int64_t(__ldg(eid + p)) : p;
        __stcs(out + ed * F4 + c, r);
    }
}

}  // namespace

namespace fgk {

fg_status launch_sddmm_binary(const fg_graph* g, int op, int F, const float* X, const float* Y, float* out,
                              cudaStream_t st) {
    if (g->n_units == 0) return FG_OK;
    const unsigned F4 = unsigned(F / 4);
    if (int64_t(g->unit_chunk) * F4 >= (int64_t(1) << 31))
        return set_error(FG_ESHAPE, "fg_sddmm: H*D too large for the elementwise kernel");
    const int64_t blocks = (g->n_units * 32 + THREADS - 1) / THREADS;
    const float4* X4 = reinterpret_cast<const float4*>(X);
    const float4* Y4 = reinterpret_cast<const float4*>(Y);
    float4* O4 = reinterpret_cast<float4*>(out);
#define FG_LAUNCH(OPV)                                                                                       \
    sddmm_binary_kernel<OPV><<<unsigned(blocks), THREADS, 0, st>>>(g->unit_row, g->unit_p0, g->n_units,      \
                                                                   g->unit_chunk, g->row_ptr, g->col_idx, \
                                                                   g->eid, F4, X4, Y4, O4)
    if (op == BOP_ADD) FG_LAUNCH(BOP_ADD);
    else if (op == BOP_SUB) FG_LAUNCH(BOP_SUB);
    else FG_LAUNCH(BOP_MUL);
#undef FG_LAUNCH
    return check_launch("sddmm_binary_kernel");
}

}  // namespace fgk
