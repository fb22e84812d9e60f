// backward.cu -- gradients of the hot-path ops.
//
// The gradient duality of PAPER.md P:171-173: "the gradient computation of
// SpMM with respect to A requires a dot product between the gradients of
// source and destination vertex features, thus following the SDDMM pattern.
// Likewise, the gradient computation of SDDMM follows the SpMM pattern."
// Concretely (edge p = u -> v with edge id e, rows of g are destinations,
// rows of the transposed handle gT are sources):
//   spmm sum   dX = spmm(gT, dOut)            (u_mul_e: weighted by E via gT's eid)
//              dE = sddmm(g, X, dOut)         (u_mul_e)
//   spmm max   only the forward's winning edge of (v, j) gets dOut[v][j]:
//              dX[u][j] = sum_{v: arg_u[v][j] == u} dOut[v][j] (* E[e][j/D])   -- masked gather over gT
//              dE[e][h] = sum_{j in h: arg_u[v][j] == u} dOut[v][j] * X[u][j]  -- masked SDDMM over g
//   spmm min   as max (arg_u names the minimising edge)
//   spmm mean  as sum with dOut[v] replaced by dOut[v] / |N(v)|
//   sddmm      dX = spmm_{u_mul_e}(gT, Y, dS),  dY = spmm_{u_mul_e}(g, X, dS)
//   softmax    ds[e][h] = alpha[e][h] * (dalpha[e][h] - sum_row alpha * dalpha)
// Every kernel is a pull over rows (no atomics): deterministic.
#include <algorithm>
#include <vector>

#include "fg_internal.h"

namespace {
constexpr int THREADS = 256;

// dX[u][:] for max/min (MEAN = false: masked by the forward's arg_u) and mean
// (MEAN = true: every edge, dOut[v] scaled by 1/|N(v)|, rp = g's row_ptr).
// One warp per row u of gT, lanes over float4 columns.  The row's neighbour
// indices (and edge ids) are loaded 32 at a time by the lanes and broadcast by
// shuffles, and U edges' arg_u words are in flight per lane; dOut is read only
// for the (rare) edges whose forward winner is u (max / min) -- a source wins
// about 1/deg(v) of its (v, feature) pairs.  Per (u, column) the winning edges
// are added in ascending CSR order of gT: deterministic.
template <bool UMULE, bool MEAN>
__global__ void __launch_bounds__(THREADS) sel_backward_dx_kernel(
    const int32_t* __restrict__ rows, int64_t n_rows, const int64_t* __restrict__ rpT,
    const int32_t* __restrict__ ciT, const int32_t* __restrict__ eidT, const float4* __restrict__ dOut,
    const int4* __restrict__ arg_u, const int64_t* __restrict__ rp, const float* __restrict__ E, int H, int D, int F4,
    float4* __restrict__ dX) {
    constexpr int U = 4;
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    if (r >= n_rows) return;
    const int64_t u = rows[r];
    const int64_t s = rpT[u], e = rpT[u + 1];
    for (int c0 = 0; c0 < F4; c0 += 32) {
        const int c = c0 + lane;
        const bool cok = c < F4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t p0 = s; p0 < e; p0 += 32) {
            const int cnt = int(min((int64_t)32, e - p0));
            const int vl = lane < cnt ? __ldg(ciT + p0 + lane) : 0;
            const int el = (UMULE && lane < cnt) ? (eidT ? __ldg(eidT + p0 + lane) : int(p0 + lane)) : 0;
            for (int t0 = 0; t0 < cnt; t0 += U) {
                int64_t vv[U];
                int4 a[U];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    vv[k] = __shfl_sync(0xffffffffu, vl, min(t0 + k, cnt - 1));
                    a[k] = make_int4(int(u), int(u), int(u), int(u));
                    if (!MEAN && cok) a[k] = __ldg(arg_u + vv[k] * F4 + c);
                }
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const int ed = UMULE ? __shfl_sync(0xffffffffu, el, min(t0 + k, cnt - 1)) : 0;
                    if (t0 + k >= cnt || !cok) continue;
                    if (a[k].x != u && a[k].y != u && a[k].z != u && a[k].w != u) continue;
                    const int64_t v = vv[k];
                    float4 g = __ldg(dOut + v * F4 + c);
                    if (MEAN) {
                        const float dg = float(__ldg(rp + v + 1) - __ldg(rp + v));
                        g = make_float4(g.x / dg, g.y / dg, g.z / dg, g.w / dg);
                    }
                    float w0 = 1.f, w1 = 1.f, w2 = 1.f, w3 = 1.f;
                    if (UMULE) {
                        w0 = __ldg(E + int64_t(ed) * H + (4 * c + 0) / D);
                        w1 = __ldg(E + int64_t(ed) * H + (4 * c + 1) / D);
                        w2 = __ldg(E + int64_t(ed) * H + (4 * c + 2) / D);
                        w3 = __ldg(E + int64_t(ed) * H + (4 * c + 3) / D);
                    }
                    if (a[k].x == u) acc.x = fmaf(g.x, w0, acc.x);
                    if (a[k].y == u) acc.y = fmaf(g.y, w1, acc.y);
                    if (a[k].z == u) acc.z = fmaf(g.z, w2, acc.z);
                    if (a[k].w == u) acc.w = fmaf(g.w, w3, acc.w);
                }
            }
        }
        if (cok) dX[u * F4 + c] = acc;
    }
}

// dE[e][h] for u_mul_e max/min (masked) or mean (scaled): one thread per (edge, head) of g.
template <bool MEAN>
__global__ void __launch_bounds__(THREADS) sel_backward_de_kernel(
    int64_t n_dst, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const int32_t* __restrict__ eid,
    const float* __restrict__ X, const float* __restrict__ dOut, const int32_t* __restrict__ arg_u, int H, int D,
    int64_t nnz, float* __restrict__ dE) {
    const int64_t t = int64_t(blockIdx.x) * THREADS + threadIdx.x;
    if (t >= nnz * H) return;
    const int64_t p = t / H;
    const int h = int(t % H);
    // destination row of CSR position p: binary search on row_ptr
    int64_t lo = 0, hi = n_dst;   // largest v with rp[v] <= p
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(rp + mid) <= p) lo = mid; else hi = mid;
    }
    const int64_t v = lo, u = __ldg(ci + p);
    const int64_t F = int64_t(H) * D;
    float acc = 0.f;
    for (int d = 0; d < D; ++d) {
        const int64_t j = int64_t(h) * D + d;
        if (MEAN) {
            const float dg = float(__ldg(rp + v + 1) - __ldg(rp + v));
            acc = fmaf(__ldg(dOut + v * F + j) / dg, __ldg(X + u * F + j), acc);
        } else if (__ldg(arg_u + v * F + j) == u) {
            acc = fmaf(__ldg(dOut + v * F + j), __ldg(X + u * F + j), acc);
        }
    }
    dE[(eid ? int64_t(__ldg(eid + p)) : p) * H + h] = acc;
}

// softmax backward, H divides 32: warp per row, lane-strided over (edge, head).
__global__ void __launch_bounds__(THREADS) softmax_backward_warp_kernel(
    const int32_t* __restrict__ rows, int64_t n_rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ eid,
    int H, const float* __restrict__ alpha, const float* __restrict__ dalpha, float* __restrict__ ds) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    if (r >= n_rows) return;
    const int64_t v = rows[r];
    const int64_t s0 = rp[v], n = (rp[v + 1] - s0) * H;
    const int h = lane % H;
    float dot = 0.f;
    for (int64_t q = lane; q < n; q += 32) {
        const int64_t idx = eid ? int64_t(__ldg(eid + s0 + q / H)) * H + h : s0 * H + q;
        dot = fmaf(__ldg(alpha + idx), __ldg(dalpha + idx), dot);
    }
    for (int o = 16; o >= H; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    for (int64_t q = lane; q < n; q += 32) {
        const int64_t idx = eid ? int64_t(__ldg(eid + s0 + q / H)) * H + h : s0 * H + q;
        ds[idx] = __ldg(alpha + idx) * (__ldg(dalpha + idx) - dot);
    }
}

// softmax backward, H % 4 == 0, (H/4) | 32, identity edge ids: the row's
// alpha / dalpha are the contiguous 16-byte aligned spans [s0*H, s1*H); lane l
// reads float4 i = l + 32k (heads 4*(l % (H/4)) .. +3 for every k), UN float4
// of each in flight; lanes of equal l % (H/4) merge their partial dots with a
// butterfly (as the forward softmax_vec_kernel).
__global__ void __launch_bounds__(THREADS) softmax_backward_vec_kernel(
    const int32_t* __restrict__ rows, int64_t n_rows, const int64_t* __restrict__ rp, int H,
    const float* __restrict__ alpha, const float* __restrict__ dalpha, float* __restrict__ ds) {
    constexpr int UN = 4;
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    if (r >= n_rows) return;
    const int64_t v = rows[r];
    const int64_t s0 = rp[v], n4 = (rp[v + 1] - s0) * H / 4;
    const float4* A4 = reinterpret_cast<const float4*>(alpha + s0 * H);
    const float4* D4 = reinterpret_cast<const float4*>(dalpha + s0 * H);
    float4* O4 = reinterpret_cast<float4*>(ds + s0 * H);
    float4 dot = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i0 = lane; i0 < n4; i0 += 32 * UN) {
        float4 a[UN], d[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const int64_t i = i0 + 32 * k;
            a[k] = i < n4 ? __ldg(A4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            d[k] = i < n4 ? __ldg(D4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            dot.x = fmaf(a[k].x, d[k].x, dot.x);
            dot.y = fmaf(a[k].y, d[k].y, dot.y);
            dot.z = fmaf(a[k].z, d[k].z, dot.z);
            dot.w = fmaf(a[k].w, d[k].w, dot.w);
        }
    }
    const int hq = H / 4;   // lanes l and l ^ o share their heads for o >= hq
    for (int o = 16; o >= hq; o >>= 1) {
        dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o);
        dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o);
        dot.z += __shfl_xor_sync(0xffffffffu, dot.z, o);
        dot.w += __shfl_xor_sync(0xffffffffu, dot.w, o);
    }
    for (int64_t i0 = lane; i0 < n4; i0 += 32 * UN) {
        float4 a[UN], d[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const int64_t i = i0 + 32 * k;
            if (i < n4) {
                a[k] = __ldg(A4 + i);
                d[k] = __ldg(D4 + i);
            }
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const int64_t i = i0 + 32 * k;
            if (i < n4)
                O4[i] = make_float4(a[k].x * (d[k].x - dot.x), a[k].y * (d[k].y - dot.y), a[k].z * (d[k].z - dot.z),
                                    a[k].w * (d[k].w - dot.w));
        }
    }
}

// softmax backward, generic H: thread per (row, head).
__global__ void __launch_bounds__(THREADS) softmax_backward_thread_kernel(
    const int32_t* __restrict__ rows, int64_t n_rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ eid,
    int H, const float* __restrict__ alpha, const float* __restrict__ dalpha, float* __restrict__ ds) {
    const int64_t t = int64_t(blockIdx.x) * THREADS + threadIdx.x;
    if (t >= n_rows * H) return;
    const int64_t v = rows[t / H];
    const int h = int(t % H);
    float dot = 0.f;
    for (int64_t p = rp[v]; p < rp[v + 1]; ++p) {
        const int64_t idx = (eid ? int64_t(eid[p]) : p) * H + h;
        dot = fmaf(alpha[idx], dalpha[idx], dot);
    }
    for (int64_t p = rp[v]; p < rp[v + 1]; ++p) {
        const int64_t idx = (eid ? int64_t(eid[p]) : p) * H + h;
        ds[idx] = alpha[idx] * (dalpha[idx] - dot);
    }
}


bool is_transpose_of(const fg_graph* g, const fg_graph* gT) {
    return gT && gT->n_dst == g->n_src && gT->n_src == g->n_dst && gT->nnz == g->nnz;
}
}  // namespace

using fgk::set_error;

extern "C" fg_status fg_graph_transpose(const fg_graph* g, fg_stream stream, fg_graph** out) {
    if (!g || !out) return set_error(FG_EINVAL, "fg_graph_transpose: NULL argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nd = g->n_dst, ns = g->n_src, m = g->nnz;
    std::vector<int64_t> rp(static_cast<size_t>(nd + 1)), rpT(static_cast<size_t>(ns + 1), 0);
    std::vector<int32_t> ci(static_cast<size_t>(m)), eid(g->eid ? static_cast<size_t>(m) : 0),
        ciT(static_cast<size_t>(m)), eidT(static_cast<size_t>(m));
    cudaError_t e = cudaMemcpyAsync(rp.data(), g->row_ptr, sizeof(int64_t) * size_t(nd + 1), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(ci.data(), g->col_idx, sizeof(int32_t) * size_t(m), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && m && g->eid) e = cudaMemcpyAsync(eid.data(), g->eid, sizeof(int32_t) * size_t(m), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(FG_ECUDA, "fg_graph_transpose: %s", cudaGetErrorString(e));
    // counting sort by source; iterating destinations in order keeps every
    // transposed row ascending (deterministic CSC)
    for (int64_t p = 0; p < m; ++p) rpT[size_t(ci[size_t(p)]) + 1]++;
    for (int64_t u = 0; u < ns; ++u) rpT[size_t(u + 1)] += rpT[size_t(u)];
    std::vector<int64_t> cur(rpT.begin(), rpT.end() - 1);
    for (int64_t v = 0; v < nd; ++v)
        for (int64_t p = rp[size_t(v)]; p < rp[size_t(v + 1)]; ++p) {
            const int64_t q = cur[size_t(ci[size_t(p)])]++;
            ciT[size_t(q)] = int32_t(v);
            eidT[size_t(q)] = g->eid ? eid[size_t(p)] : int32_t(p);   // original edge id
        }
    int64_t* d_rp = nullptr;
    int32_t *d_ci = nullptr, *d_eid = nullptr;
    e = cudaMalloc(&d_rp, sizeof(int64_t) * size_t(ns + 1));
    if (e == cudaSuccess) e = cudaMalloc(&d_ci, sizeof(int32_t) * size_t(std::max<int64_t>(m, 1)));
    if (e == cudaSuccess) e = cudaMalloc(&d_eid, sizeof(int32_t) * size_t(std::max<int64_t>(m, 1)));
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_rp, rpT.data(), sizeof(int64_t) * size_t(ns + 1), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(d_ci, ciT.data(), sizeof(int32_t) * size_t(m), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(d_eid, eidT.data(), sizeof(int32_t) * size_t(m), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_eid);
        return set_error(e == cudaErrorMemoryAllocation ? FG_ENOMEM : FG_ECUDA, "fg_graph_transpose: %s",
                         cudaGetErrorString(e));
    }
    fg_graph* gT = nullptr;
    fg_status s = fg_graph_create(ns, nd, m, d_rp, d_ci, d_eid, 0, stream, &gT);
    if (s != FG_OK) {
        cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_eid);
        return s;
    }
    gT->owned_row_ptr = d_rp;
    gT->owned_col_idx = d_ci;
    gT->owned_eid = d_eid;
    gT->device_bytes += sizeof(int64_t) * (ns + 1) + 8 * m;
    *out = gT;
    return FG_OK;
}

extern "C" fg_status fg_spmm_backward(const fg_graph* g, const fg_graph* gT, fg_msg_op msg, fg_reduce_op red, int H,
                                      int D, const float* X, const float* E, const float* dOut,
                                      const int32_t* arg_u, float* dX, float* dE, fg_stream stream) {
    if (!g) return set_error(FG_EINVAL, "fg_spmm_backward: NULL graph");
    if (msg != FG_MSG_COPY_U && msg != FG_MSG_U_MUL_E)
        return set_error(FG_EUNSUPPORTED, "fg_spmm_backward: only copy_u / u_mul_e (SPEC non-goal: mlp through W)");
    if (red != FG_REDUCE_SUM && red != FG_REDUCE_MAX && red != FG_REDUCE_MIN && red != FG_REDUCE_MEAN)
        return set_error(FG_EINVAL, "fg_spmm_backward: bad reduce op");
    if (H < 1 || D < 1 || (int64_t(H) * D) % 4) return set_error(FG_ESHAPE, "fg_spmm_backward: H*D must be a multiple of 4");
    if (!dOut) return set_error(FG_EINVAL, "fg_spmm_backward: dOut is NULL");
    if (dX && !is_transpose_of(g, gT)) return set_error(FG_EINVAL, "fg_spmm_backward: dX needs gT = fg_graph_transpose(g)");
    if (msg == FG_MSG_U_MUL_E && !E) return set_error(FG_EINVAL, "fg_spmm_backward: u_mul_e needs E");
    if (dE && (msg != FG_MSG_U_MUL_E || !X)) return set_error(FG_EINVAL, "fg_spmm_backward: dE needs u_mul_e and X");
    const bool mean = red == FG_REDUCE_MEAN;
    if ((red == FG_REDUCE_MAX || red == FG_REDUCE_MIN) && !arg_u)
        return set_error(FG_EINVAL, "fg_spmm_backward: max/min need the forward's arg_u");
    if (!fgk::aligned16(dOut) || !fgk::aligned16(dX) || !fgk::aligned16(X) || !fgk::aligned16(arg_u))
        return set_error(FG_EINVAL, "fg_spmm_backward: tensors must be 16-byte aligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int F4 = H * D / 4;
    if (red == FG_REDUCE_SUM) {
        if (dX) {
            fg_status s = fgk::launch_spmm_gather(gT, msg, FG_REDUCE_SUM, H, D, dOut, msg == FG_MSG_U_MUL_E ? E : nullptr,
                                                  dX, nullptr, nullptr, st);
            if (s != FG_OK) return s;
        }
        if (dE) return fg_sddmm(g, FG_EDGE_U_DOT_V, H, D, X, dOut, dE, stream);
        return FG_OK;
    }
    if (dX && gT->n_dst > 0) {
        const int64_t blocks = (gT->n_dst * 32 + THREADS - 1) / THREADS;
        auto kern = msg == FG_MSG_U_MUL_E ? (mean ? sel_backward_dx_kernel<true, true> : sel_backward_dx_kernel<true, false>)
                                          : (mean ? sel_backward_dx_kernel<false, true> : sel_backward_dx_kernel<false, false>);
        kern<<<unsigned(blocks), THREADS, 0, st>>>(gT->rows_by_deg, gT->n_dst, gT->row_ptr, gT->col_idx, gT->eid,
                                                   reinterpret_cast<const float4*>(dOut),
                                                   reinterpret_cast<const int4*>(arg_u), g->row_ptr, E, H, D, F4,
                                                   reinterpret_cast<float4*>(dX));
        fg_status s = fgk::check_launch("sel_backward_dx_kernel");
        if (s != FG_OK) return s;
    }
    if (dE && g->nnz > 0) {
        const int64_t blocks = (g->nnz * H + THREADS - 1) / THREADS;
        auto kern = mean ? sel_backward_de_kernel<true> : sel_backward_de_kernel<false>;
        kern<<<unsigned(blocks), THREADS, 0, st>>>(g->n_dst, g->row_ptr, g->col_idx, g->eid, X, dOut, arg_u, H, D,
                                                   g->nnz, dE);
        return fgk::check_launch("sel_backward_de_kernel");
    }
    return FG_OK;
}

extern "C" fg_status fg_sddmm_backward(const fg_graph* g, const fg_graph* gT, fg_edge_op op, int H, int D,
                                       const float* X, const float* Y, const float* dS, float* dX, float* dY,
                                       fg_stream stream) {
    if (!g) return set_error(FG_EINVAL, "fg_sddmm_backward: NULL graph");
    if (op != FG_EDGE_U_DOT_V) return set_error(FG_EUNSUPPORTED, "fg_sddmm_backward: only u_dot_v");
    if (!dS) return set_error(FG_EINVAL, "fg_sddmm_backward: dS is NULL");
    if (dX && (!Y || !is_transpose_of(g, gT)))
        return set_error(FG_EINVAL, "fg_sddmm_backward: dX needs Y and gT = fg_graph_transpose(g)");
    if (dY && !X) return set_error(FG_EINVAL, "fg_sddmm_backward: dY needs X");
    // dX[u] = sum_{e = u->v} dS[e] * Y[v]  : u_mul_e-sum over gT with features Y
    if (dX) {
        fg_status s = fg_spmm(gT, FG_MSG_U_MUL_E, FG_REDUCE_SUM, H, D, Y, dS, nullptr, 0, nullptr, dX, nullptr, nullptr,
                              nullptr, 0, stream);
        if (s != FG_OK) return s;
    }
    // dY[v] = sum_{e = u->v} dS[e] * X[u]  : u_mul_e-sum over g with features X
    if (dY)
        return fg_spmm(g, FG_MSG_U_MUL_E, FG_REDUCE_SUM, H, D, X, dS, nullptr, 0, nullptr, dY, nullptr, nullptr,
                       nullptr, 0, stream);
    return FG_OK;
}

extern "C" fg_status fg_edge_softmax_backward(const fg_graph* g, int H, const float* alpha, const float* dalpha,
                                              float* dscores, fg_stream stream) {
    if (!g) return set_error(FG_EINVAL, "fg_edge_softmax_backward: NULL graph");
    if (H < 1 || H > 4096) return set_error(FG_ESHAPE, "fg_edge_softmax_backward: bad H");
    if (g->nnz == 0) return FG_OK;
    if (!alpha || !dalpha || !dscores) return set_error(FG_EINVAL, "fg_edge_softmax_backward: NULL tensor");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n_rows = g->n_nonempty;
    const bool a16 = ((reinterpret_cast<uintptr_t>(alpha) | reinterpret_cast<uintptr_t>(dalpha) |
                       reinterpret_cast<uintptr_t>(dscores)) & 15u) == 0;
    if (H % 4 == 0 && 32 % (H / 4) == 0 && g->eid == nullptr && a16) {
        const int64_t blocks = (n_rows * 32 + THREADS - 1) / THREADS;
        softmax_backward_vec_kernel<<<unsigned(blocks), THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr, H,
                                                                          alpha, dalpha, dscores);
    } else if (32 % H == 0) {
        const int64_t blocks = (n_rows * 32 + THREADS - 1) / THREADS;
        softmax_backward_warp_kernel<<<unsigned(blocks), THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr, g->eid,
                                                                           H, alpha, dalpha, dscores);
    } else {
        const int64_t blocks = (n_rows * H + THREADS - 1) / THREADS;
        softmax_backward_thread_kernel<<<unsigned(blocks), THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr,
                                                                             g->eid, H, alpha, dalpha, dscores);
    }
    return fgk::check_launch("edge_softmax_backward");
}
