// api.cu -- the C ABI of include/fg.h: argument validation (host, before any
// launch) and dispatch to the sm_100a kernels.
#include <cstdarg>
#include <cstdio>

#include "fg_internal.h"

namespace {
thread_local char g_err[512] = "";
}  // namespace

namespace fgk {
fg_status set_error(fg_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

fg_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(FG_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return FG_OK;
}
}  // namespace fgk

using fgk::set_error;
using fgk::aligned16;

extern "C" const char* fg_status_string(fg_status s) {
    switch (s) {
        case FG_OK: return "FG_OK";
        case FG_EINVAL: return "FG_EINVAL: invalid argument (null/misaligned pointer or bad enum)";
        case FG_ESHAPE: return "FG_ESHAPE: inconsistent or unsupported dimensions";
        case FG_EUNSUPPORTED: return "FG_EUNSUPPORTED: combination not implemented";
        case FG_EGRAPH: return "FG_EGRAPH: CSR invariant violated";
        case FG_ECUDA: return "FG_ECUDA: CUDA error";
        case FG_ENOMEM: return "FG_ENOMEM: out of memory";
        case FG_ENCCL: return "FG_ENCCL: NCCL error";
    }
    return "unknown fg_status";
}

extern "C" const char* fg_last_error(void) { return g_err; }
extern "C" int fg_abi_version(void) { return FG_ABI_VERSION; }

extern "C" fg_status fg_spmm_workspace_size(const fg_graph* g, fg_msg_op msg, fg_reduce_op, int H, int D, int d_in,
                                            size_t* bytes) {
    if (!g || !bytes) return set_error(FG_EINVAL, "fg_spmm_workspace_size: NULL argument");
    // no message needs scratch: heavy rows combine on chip, and the mlp producer
    // forms and splits x_u + x_v on the fly (kept in the ABI for future messages)
    (void)msg; (void)H; (void)D; (void)d_in;
    *bytes = 0;
    return FG_OK;
}

namespace fgk {
// Host-side argument checks of fg_spmm (before any launch; also run by
// fg_dist_spmm before it starts the all-gather).
fg_status check_spmm(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D, const float* X,
                     const float* E, const float* W, int d_in, const float* X_dst, const float* out,
                     const int32_t* arg_u, const int32_t* arg_e) {
    if (!g) return set_error(FG_EINVAL, "fg_spmm: NULL graph");
    if (msg != FG_MSG_COPY_U && msg != FG_MSG_U_MUL_E && msg != FG_MSG_MLP && msg != FG_MSG_U_ADD_E &&
        msg != FG_MSG_COPY_E)
        return set_error(FG_EINVAL, "fg_spmm: bad msg op %d", int(msg));
    if (red != FG_REDUCE_SUM && red != FG_REDUCE_MAX && red != FG_REDUCE_MIN && red != FG_REDUCE_MEAN)
        return set_error(FG_EINVAL, "fg_spmm: bad reduce op %d", int(red));
    if ((red == FG_REDUCE_SUM || red == FG_REDUCE_MEAN) && (arg_u || arg_e))
        return set_error(FG_EINVAL, "fg_spmm: arg_u/arg_e must be NULL for sum/mean");
    if (msg == FG_MSG_MLP && red != FG_REDUCE_SUM && red != FG_REDUCE_MAX)
        return set_error(FG_EUNSUPPORTED, "fg_spmm(mlp): only sum and max reducers");
    if (H < 1 || D < 1) return set_error(FG_ESHAPE, "fg_spmm: H=%d D=%d must be >= 1", H, D);
    const int64_t F = int64_t(H) * D;
    if (F % 4 != 0) return set_error(FG_ESHAPE, "fg_spmm: H*D=%lld must be a multiple of 4", (long long)F);
    if (F > (int64_t(1) << 20)) return set_error(FG_ESHAPE, "fg_spmm: H*D=%lld too large", (long long)F);
    if (!out && g->n_dst > 0) return set_error(FG_EINVAL, "fg_spmm: out is NULL");
    if (!aligned16(out) || !aligned16(X) || !aligned16(arg_u) || !aligned16(arg_e))
        return set_error(FG_EINVAL, "fg_spmm: X/out/arg pointers must be 16-byte aligned");
    if (msg == FG_MSG_MLP) {
        if (H != 1) return set_error(FG_ESHAPE, "fg_spmm(mlp): H must be 1 (got %d)", H);
        if (d_in < 1 || d_in > 32) return set_error(FG_ESHAPE, "fg_spmm(mlp): d_in=%d must be in [1,32]", d_in);
        if (!W) return set_error(FG_EINVAL, "fg_spmm(mlp): W is NULL");
        if (!X_dst && g->n_src != g->n_dst)
            return set_error(FG_ESHAPE, "fg_spmm(mlp): X_dst = NULL needs n_src == n_dst");
        if (E) return set_error(FG_EINVAL, "fg_spmm(mlp): E must be NULL");
        if (!aligned16(X_dst)) return set_error(FG_EINVAL, "fg_spmm(mlp): X_dst must be 16-byte aligned");
    } else {
        if (d_in != 0 || W || X_dst) return set_error(FG_EINVAL, "fg_spmm: W/X_dst/d_in are for mlp only");
        if ((msg == FG_MSG_U_MUL_E || msg == FG_MSG_U_ADD_E || msg == FG_MSG_COPY_E) && !E && g->nnz > 0)
            return set_error(FG_EINVAL, "fg_spmm(u_*_e / copy_e): E is NULL");
        if (msg == FG_MSG_COPY_U && E) return set_error(FG_EINVAL, "fg_spmm(copy_u): E must be NULL");
        if (msg == FG_MSG_COPY_E && X) return set_error(FG_EINVAL, "fg_spmm(copy_e): X must be NULL");
        if (msg == FG_MSG_COPY_E && !aligned16(E)) return set_error(FG_EINVAL, "fg_spmm(copy_e): E must be 16-byte aligned");
    }
    if (msg != FG_MSG_COPY_E && !X && g->nnz > 0) return set_error(FG_EINVAL, "fg_spmm: X is NULL");
    return FG_OK;
}

// Host-side argument checks of fg_sddmm (also run by fg_dist_sddmm before the all-gather).
fg_status check_sddmm(const fg_graph* g, fg_edge_op op, int H, int D, const float* X, const float* Y,
                      const float* out) {
    if (!g) return set_error(FG_EINVAL, "fg_sddmm: NULL graph");
    if (op != FG_EDGE_U_DOT_V && op != FG_EDGE_U_ADD_V && op != FG_EDGE_U_SUB_V && op != FG_EDGE_U_MUL_V)
        return set_error(FG_EINVAL, "fg_sddmm: bad edge op %d", int(op));
    if (H < 1 || D < 1) return set_error(FG_ESHAPE, "fg_sddmm: H=%d D=%d must be >= 1", H, D);
    const int64_t F = int64_t(H) * D;
    if (F % 4 != 0) return set_error(FG_ESHAPE, "fg_sddmm: H*D must be a multiple of 4");
    if (F > (int64_t(1) << 20)) return set_error(FG_ESHAPE, "fg_sddmm: H*D too large");
    if (g->nnz == 0) return FG_OK;
    if (!X || !Y || !out) return set_error(FG_EINVAL, "fg_sddmm: NULL tensor");
    if (!aligned16(X) || !aligned16(Y) || !aligned16(out))
        return set_error(FG_EINVAL, "fg_sddmm: X/Y/out must be 16-byte aligned");
    return FG_OK;
}
}  // namespace fgk

extern "C" fg_status fg_spmm(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D,
                             const float* X, const float* E, const float* W, int d_in, const float* X_dst,
                             float* out, int32_t* arg_u, int32_t* arg_e, void* workspace,
                             size_t workspace_bytes, fg_stream stream) {
    (void)workspace; (void)workspace_bytes;   // no op needs scratch (fg_spmm_workspace_size == 0)
    fg_status s = fgk::check_spmm(g, msg, red, H, D, X, E, W, d_in, X_dst, out, arg_u, arg_e);
    if (s != FG_OK) return s;
    if (g->n_dst == 0) return FG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (msg == FG_MSG_MLP)
        return fgk::launch_spmm_mlp(g, red, D, X, W, d_in, X_dst ? X_dst : X, out, arg_u, arg_e, st);
    return fgk::launch_spmm_gather(g, msg, red, H, D, X, E, out, arg_u, arg_e, st);
}

extern "C" fg_status fg_sddmm(const fg_graph* g, fg_edge_op op, int H, int D, const float* X, const float* Y,
                              float* out, fg_stream stream) {
    fg_status s = fgk::check_sddmm(g, op, H, D, X, Y, out);
    if (s != FG_OK) return s;
    if (g->nnz == 0) return FG_OK;
    const int64_t F = int64_t(H) * D;
    if (op != FG_EDGE_U_DOT_V)
        return fgk::launch_sddmm_binary(g, int(op), int(F), X, Y, out, reinterpret_cast<cudaStream_t>(stream));
    return fgk::launch_sddmm(g, H, D, X, Y, out, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" fg_status fg_sddmm_emul(const fg_graph* g, int H, int D, const float* X, const float* Y, const float* E,
                                   float* out, fg_stream stream) {
    if (!g) return set_error(FG_EINVAL, "fg_sddmm_emul: NULL graph");
    if (H < 1 || D < 1) return set_error(FG_ESHAPE, "fg_sddmm_emul: H=%d D=%d must be >= 1", H, D);
    const int64_t F = int64_t(H) * D;
    if (F % 4 != 0 || F > (int64_t(1) << 20)) return set_error(FG_ESHAPE, "fg_sddmm_emul: H*D must be a multiple of 4");
    if (g->nnz == 0) return FG_OK;
    if (!X || !Y || !E || !out) return set_error(FG_EINVAL, "fg_sddmm_emul: NULL tensor");
    if (!aligned16(X) || !aligned16(Y) || !aligned16(out))
        return set_error(FG_EINVAL, "fg_sddmm_emul: X/Y/out must be 16-byte aligned");
    {
        const uintptr_t o0 = reinterpret_cast<uintptr_t>(out), e0 = reinterpret_cast<uintptr_t>(E);
        const uintptr_t nb = uintptr_t(g->nnz) * uintptr_t(H) * 4u;
        if (o0 < e0 + nb && e0 < o0 + nb) return set_error(FG_EINVAL, "fg_sddmm_emul: out must not overlap E");
    }
    return fgk::launch_sddmm(g, H, D, X, Y, out, reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, E);
}

extern "C" fg_status fg_spmm_x16(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D,
                                 const uint16_t* X, const float* E, float* out, int32_t* arg_u, int32_t* arg_e,
                                 fg_stream stream) {
    if (!g) return set_error(FG_EINVAL, "fg_spmm_x16: NULL graph");
    if (msg != FG_MSG_COPY_U && msg != FG_MSG_U_MUL_E)
        return set_error(FG_EUNSUPPORTED, "fg_spmm_x16: only copy_u and u_mul_e (got msg %d)", int(msg));
    if (red != FG_REDUCE_SUM && red != FG_REDUCE_MAX && red != FG_REDUCE_MIN && red != FG_REDUCE_MEAN)
        return set_error(FG_EINVAL, "fg_spmm_x16: bad reducer %d", int(red));
    if ((red == FG_REDUCE_SUM || red == FG_REDUCE_MEAN) && (arg_u || arg_e))
        return set_error(FG_EINVAL, "fg_spmm_x16: arg_u/arg_e with sum / mean");
    if (H < 1 || D < 1) return set_error(FG_ESHAPE, "fg_spmm_x16: H=%d D=%d must be >= 1", H, D);
    const int64_t F = int64_t(H) * D;
    if (F % 4 != 0 || F > (int64_t(1) << 20))
        return set_error(FG_ESHAPE, "fg_spmm_x16: H*D=%lld must be a multiple of 4 (<= 2^20)", (long long)F);
    if (!out && g->n_dst > 0) return set_error(FG_EINVAL, "fg_spmm_x16: out is NULL");
    if (!X && g->nnz > 0) return set_error(FG_EINVAL, "fg_spmm_x16: X is NULL");
    if (msg == FG_MSG_U_MUL_E && !E && g->nnz > 0) return set_error(FG_EINVAL, "fg_spmm_x16(u_mul_e): E is NULL");
    if (msg == FG_MSG_COPY_U && E) return set_error(FG_EINVAL, "fg_spmm_x16(copy_u): E must be NULL");
    if ((reinterpret_cast<uintptr_t>(X) & 7u) != 0 || !aligned16(out) || !aligned16(arg_u) || !aligned16(arg_e))
        return set_error(FG_EINVAL, "fg_spmm_x16: X must be 8-byte, out/arg 16-byte aligned");
    if (g->n_dst == 0) return FG_OK;
    return fgk::launch_spmm_gather(g, msg, red, H, D, nullptr, E, out, arg_u, arg_e,
                                   reinterpret_cast<cudaStream_t>(stream), X);
}

extern "C" fg_status fg_sddmm_x16(const fg_graph* g, fg_edge_op op, int H, int D, const uint16_t* X,
                                  const uint16_t* Y, float* out, fg_stream stream) {
    if (!g) return set_error(FG_EINVAL, "fg_sddmm_x16: NULL graph");
    if (op != FG_EDGE_U_DOT_V) return set_error(FG_EUNSUPPORTED, "fg_sddmm_x16: only u_dot_v (got %d)", int(op));
    if (H < 1 || D < 1) return set_error(FG_ESHAPE, "fg_sddmm_x16: H=%d D=%d must be >= 1", H, D);
    const int64_t F = int64_t(H) * D;
    if (F % 4 != 0 || F > (int64_t(1) << 20)) return set_error(FG_ESHAPE, "fg_sddmm_x16: H*D must be a multiple of 4");
    if (H > 1 && (D % 4 != 0 || ((D / 4) & (D / 4 - 1)) != 0))
        return set_error(FG_ESHAPE, "fg_sddmm_x16: with H > 1, D must be 4 * 2^k (got D=%d)", D);
    if (g->nnz == 0) return FG_OK;
    if (!X || !Y || !out) return set_error(FG_EINVAL, "fg_sddmm_x16: NULL tensor");
    if ((reinterpret_cast<uintptr_t>(X) & 7u) != 0 || (reinterpret_cast<uintptr_t>(Y) & 7u) != 0 || !aligned16(out))
        return set_error(FG_EINVAL, "fg_sddmm_x16: X/Y must be 8-byte, out 16-byte aligned");
    return fgk::launch_sddmm(g, H, D, nullptr, nullptr, out, reinterpret_cast<cudaStream_t>(stream), X, Y);
}

extern "C" fg_status fg_edge_softmax(const fg_graph* g, int H, const float* scores, float* out, fg_stream stream) {
    if (!g) return set_error(FG_EINVAL, "fg_edge_softmax: NULL graph");
    if (H < 1 || H > 4096) return set_error(FG_ESHAPE, "fg_edge_softmax: H=%d out of range", H);
    if (g->nnz == 0) return FG_OK;
    if (!scores || !out) return set_error(FG_EINVAL, "fg_edge_softmax: NULL tensor");
    if (!aligned16(scores) || !aligned16(out))
        return set_error(FG_EINVAL, "fg_edge_softmax: scores/out must be 16-byte aligned");
    return fgk::launch_edge_softmax(g, H, scores, out, reinterpret_cast<cudaStream_t>(stream));
}
