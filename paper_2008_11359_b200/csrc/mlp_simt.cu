// mlp_simt.cu -- gSpMM with the MLP message on CUDA cores (FFMA): the
// ablation baseline for the tcgen05 kernel (mlp_tcgen05.cu), and the path for
// shapes the tensor-core kernel does not take.
//
// Fig. 3b: phi(u, v) = ReLU((x_u + x_v) W), W in R^{d1 x d2},
// aggregated by max (Fig. 1 "picking the maximum") or sum, in the paper's
// order: s_e = x_u + x_v (fp32), z_e = s_e W (d1*d2 FMAs in k order), then
//   max: out = ReLU(max_e z_e); arg = first argmax if that is > 0, else the
//        row's first edge (all messages are +0 then; first wins);
//   sum: out = sum_e ReLU(z_e).
// One warp per destination row (degree-descending order), lane owns NC columns;
// x_v (d_in <= 32 values) is held in registers for the row.
#include <cstdlib>

#include "fg_internal.h"

namespace {
constexpr int THREADS = 256;

template <int NC, bool MAX>
__global__ void __launch_bounds__(THREADS) mlp_simt_kernel(const int32_t* __restrict__ rows, int64_t n_rows,
                                                           const int64_t* __restrict__ rp,
                                                           const int32_t* __restrict__ ci,
                                                           const int32_t* __restrict__ eid,
                                                           const float* __restrict__ X,
                                                           const float* __restrict__ Xd,
                                                           const float* __restrict__ W, int d_in, int d2,
                                                           float* __restrict__ out, int32_t* __restrict__ arg_u,
                                                           int32_t* __restrict__ arg_e) {
    const int lane = threadIdx.x & 31;
    const int cbase = blockIdx.y * 32 * NC;
    __shared__ float sW[32][32 * NC];            // W[:, cbase : cbase + 32*NC] (d_in <= 32)
    for (int i = threadIdx.x; i < 32 * 32 * NC; i += THREADS) {
        const int k = i / (32 * NC), c = cbase + i % (32 * NC);
        sW[k][i % (32 * NC)] = (k < d_in && c < d2) ? W[int64_t(k) * d2 + c] : 0.f;
    }
    __syncthreads();
    const int64_t r = (int64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    if (r >= n_rows) return;
    const int64_t v = rows[r];
    const int64_t s = rp[v], e = rp[v + 1];
    float best[NC];
    int pos[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        best[j] = MAX ? -INFINITY : 0.f;
        pos[j] = -1;
    }
    const float xv_l = lane < d_in ? __ldg(Xd + v * d_in + lane) : 0.f;   // lane k holds x_v[k]
    for (int64_t p = s; p < e; ++p) {
        const int64_t u = __ldg(ci + p);
        const float xu_l = lane < d_in ? __ldg(X + u * d_in + lane) : 0.f;
        const float s_l = xu_l + xv_l;                                     // s_e[k] = x_u[k] + x_v[k]
        float a[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) a[j] = 0.f;
        for (int k = 0; k < d_in; ++k) {
            const float sk = __shfl_sync(0xffffffffu, s_l, k);
#pragma unroll
            for (int j = 0; j < NC; ++j) a[j] = fmaf(sk, sW[k][lane + 32 * j], a[j]);
        }
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            if (MAX) {
                if (a[j] > best[j]) { best[j] = a[j]; pos[j] = int(p); }
            } else {
                best[j] += fmaxf(a[j], 0.f);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        const int c = cbase + lane + 32 * j;
        if (c >= d2) continue;
        const int64_t o = v * d2 + c;
        if (!MAX) { out[o] = best[j]; continue; }
        if (e == s) {
            out[o] = 0.f;
            if (arg_u) arg_u[o] = -1;
            if (arg_e) arg_e[o] = -1;
            continue;
        }
        const float z = best[j];
        const int pw = (z > 0.f) ? pos[j] : int(s);
        out[o] = z > 0.f ? z : 0.f;
        if (arg_u) arg_u[o] = __ldg(ci + pw);
        if (arg_e) arg_e[o] = eid ? __ldg(eid + pw) : pw;
    }
}
}  // namespace

namespace fgk {
fg_status launch_spmm_mlp_simt(const fg_graph* g, fg_reduce_op red, int d2, const float* X, const float* W,
                               int d_in, const float* X_dst, float* out, int32_t* arg_u, int32_t* arg_e,
                               cudaStream_t st) {
    const int64_t n_rows = g->n_dst;
    constexpr int NC = 4;
    dim3 grid(unsigned((n_rows * 32 + THREADS - 1) / THREADS), unsigned((d2 + 32 * NC - 1) / (32 * NC)));
    if (red == FG_REDUCE_MAX)
        mlp_simt_kernel<NC, true><<<grid, THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr, g->col_idx, g->eid,
                                                            X, X_dst, W, d_in, d2, out, arg_u, arg_e);
    else
        mlp_simt_kernel<NC, false><<<grid, THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr, g->col_idx, g->eid,
                                                             X, X_dst, W, d_in, d2, out, arg_u, arg_e);
    return check_launch("mlp_simt_kernel");
}

// The product path is the tcgen05 3xTF32 kernel; FG_TUNE_MLP_IMPL selects the
// ablations (1: this FFMA kernel, CUDA cores instead of tensor cores; 2: the
// tcgen05 kernel with the bf16 2-split) -- same semantics.
fg_status launch_spmm_mlp(const fg_graph* g, fg_reduce_op red, int d2, const float* X, const float* W, int d_in,
                          const float* X_dst, float* out, int32_t* arg_u, int32_t* arg_e, cudaStream_t st) {
    if (g->tune.mlp_impl == 1) return launch_spmm_mlp_simt(g, red, d2, X, W, d_in, X_dst, out, arg_u, arg_e, st);
    return launch_spmm_mlp_tcgen05(g, red, d2, X, W, d_in, X_dst, out, arg_u, arg_e, g->tune.mlp_impl == 2, st);
}
}  // namespace fgk
