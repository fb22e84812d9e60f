// gat_fused.cu -- the GAT attention layer in ONE row-resident pass
// (SURVEY §8(f) row f2): gSDDMM u_dot_v -> edge softmax -> gSpMM u_mul_e-sum.
//
//   s[e][h]   = <X[u][h,:], Y[v][h,:]>                 (Eq. (4), Fig. 5b; P:983 GAT uses dot attention)
//   a[e][h]   = exp(s[e][h] - max_row) / sum_row exp(.) (edge softmax over the in-edges of v)
//   out[v][h] = sum_e a[e][h] X[u][h,:]                (Eq. (1) with the u_mul_e message)
//
// This is the paper's fusion principle (UDFs inlined into the template, no
// per-edge message tensor materialised: P:378-379) applied across the
// three templates: every source row X[u] is gathered ONCE (it serves both the
// score and the aggregation) and neither s nor a round-trips through HBM
// (3.7 GB each for reddit at H = 8).  The softmax is the online (streaming)
// form: per lane and head a running max m, sum l and accumulator acc are
// rescaled when the max grows, so one pass over the row suffices.
//
// Mapping as in spmm.cu: a group of G lanes owns a destination row, each lane
// NV float4 columns (head of column chunk c = c / (D/4)); the per-edge scores are
// reduced over the D/4 lanes of a head (a reduce-scatter of the U x NV partial
// dots + one gather shuffle per score when NV = 2, else a butterfly).  Rows of degree >= T run
// CTA-per-row: the groups take contiguous edge ranges and their (m, l, acc)
// partials are merged in a fixed order (deterministic, no atomics).
#include <algorithm>
#include <cstdlib>

#include "device_common.cuh"
#include "fg_internal.h"

namespace {
using namespace fgdev;

constexpr int THREADS = 256;

struct Args {
    const int32_t* rows;
    int64_t n_heavy, n_rows;
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* eid;
    int H, D4, F4;
};

__device__ __forceinline__ float ex2(float x) {   // 2^x, MUFU.EX2 (rel. error ~2^-22)
    float y;
    asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int NV>
struct State {
    float m[NV], l[NV];
    float4 acc[NV];
};

// DWT > 0: the head width D/4 is DWT lanes (compile time): the U x NV per-head
// scores are reduced with one reduce-scatter over the DWT lanes and gathered back
// with U*NV shuffles (fewer shuffles and adds than a butterfly per score)
template <int G, int NV, int U, bool PIPE, int DWT>
__device__ __forceinline__ void attend_range(const Args& A, const float4* __restrict__ X, const float4 (&y)[NV],
                                             int64_t s, int64_t e, int gl, unsigned mask, State<NV>& st,
                                             float* __restrict__ scores, int* __restrict__ sidx) {
    // Compact loop (the fully unrolled 32-edge body was instruction-fetch bound):
    // indices staged in shared memory per batch, U edges' gathers in flight, then
    // the U x NV per-head scores (butterfly over the D/4 lanes of a head) and the
    // sequential online-softmax updates.
    constexpr int B = 32;
    const int F4 = A.F4, D4 = A.D4, H = A.H;
    const char* xl = reinterpret_cast<const char*>(X + gl);   // this lane's first column
    const uint32_t rowb = uint32_t(F4) * 16u;
    bool cin[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) cin[j] = gl + G * j < F4;
    for (int64_t p0 = s; p0 < e; p0 += B) {
        const int cnt = int(min((int64_t)B, e - p0));
        __syncwarp(mask);
        for (int t = gl; t < cnt; t += G) sidx[t] = __ldg(A.col_idx + p0 + t);
        __syncwarp(mask);
        float4 xn[U][NV];   // software pipeline: next U edges' gathers in flight
        // past the batch end the last edge's row is re-read (an L1 hit) instead of
        // predicating each load; those slots are never consumed (t >= cnt breaks below,
        // and every per-head score reduces one (edge, chunk) slot only).  Rows are
        // addressed with one 32x32 -> 64-bit multiply-add from the lane's column base.
        auto gather = [&](int tb, float4 (&dst)[U][NV]) {
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = min(tb + uu, cnt - 1);
                const char* xr = xl + uint64_t(uint32_t(sidx[t])) * rowb;
#pragma unroll
                for (int j = 0; j < NV; ++j)
                    dst[uu][j] = cin[j] ? __ldg(reinterpret_cast<const float4*>(xr) + G * j)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        if constexpr (PIPE) gather(0, xn);
        for (int t0 = 0; t0 < cnt; t0 += U) {
            float4 x[U][NV];
            if constexpr (PIPE) {
#pragma unroll
                for (int uu = 0; uu < U; ++uu)
#pragma unroll
                    for (int j = 0; j < NV; ++j) x[uu][j] = xn[uu][j];
                if (t0 + U < cnt) gather(t0 + U, xn);
            } else {
                gather(t0, x);
            }
            float sc[U][NV];
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
#pragma unroll
                for (int j = 0; j < NV; ++j) sc[uu][j] = dot4(x[uu][j], y[j]);
            if constexpr (DWT > 0) {
                constexpr int K = U * NV;
                static_assert(K <= DWT, "one reduced score per lane");
                float pv[K];
#pragma unroll
                for (int uu = 0; uu < U; ++uu)
#pragma unroll
                    for (int j = 0; j < NV; ++j) pv[uu * NV + j] = sc[uu][j];
                reduce_scatter<K, DWT, G>(pv, gl, mask);
                constexpr int SH = ilog2(DWT) - ilog2(K);   // lane of value id: base | (id << SH)
                const int base = gl & ~(DWT - 1);
#pragma unroll
                for (int id = 0; id < K; ++id) sc[id / NV][id % NV] = __shfl_sync(mask, pv[0], base | (id << SH), G);
            } else {
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1)
                    if (o < D4 && o < G) {
#pragma unroll
                        for (int uu = 0; uu < U; ++uu)
#pragma unroll
                            for (int j = 0; j < NV; ++j) sc[uu][j] += __shfl_xor_sync(mask, sc[uu][j], o, G);
                    }
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = t0 + uu;
                if (t >= cnt) break;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int c = gl + G * j;
                    if (c >= F4) continue;
                    if (scores && (gl & (D4 - 1)) == 0) {
                        const int64_t p = p0 + t;
                        scores[(A.eid ? int64_t(__ldg(A.eid + p)) : p) * H + c / D4] = sc[uu][j];
                    }
                    // log2 domain with a lazily updated reference max m: rescale only when a
                    // score exceeds it by 2^8 (rare), so each edge costs ONE ex2; acc / l is
                    // unchanged in real arithmetic
                    const float s2 = sc[uu][j] * 1.4426950408889634f;
                    if (s2 > st.m[j] + 8.f) {
                        const float cf = ex2(st.m[j] - s2);
                        st.l[j] *= cf;
                        st.acc[j].x *= cf; st.acc[j].y *= cf; st.acc[j].z *= cf; st.acc[j].w *= cf;
                        st.m[j] = s2;
                    }
                    const float w = ex2(s2 - st.m[j]);
                    st.l[j] += w;
                    st.acc[j].x = fmaf(w, x[uu][j].x, st.acc[j].x);
                    st.acc[j].y = fmaf(w, x[uu][j].y, st.acc[j].y);
                    st.acc[j].z = fmaf(w, x[uu][j].z, st.acc[j].z);
                    st.acc[j].w = fmaf(w, x[uu][j].w, st.acc[j].w);
                }
            }
        }
    }
}

template <int G, int NV, int U, int MINB, bool PIPE, int DWT>
__global__ void __launch_bounds__(THREADS, MINB) gat_fused_kernel(const Args A, const float4* __restrict__ X,
                                                            const float4* __restrict__ Y, float4* __restrict__ out,
                                                            float* __restrict__ scores) {
    constexpr int NG = THREADS / G, TW = G * NV;
    __shared__ float4 s_acc[NG][TW];
    __shared__ float s_m[NG][TW], s_l[NG][TW];
    __shared__ int s_idx[NG][32];
    const int lane = threadIdx.x & 31;
    const int gl = threadIdx.x & (G - 1);
    const int gi = threadIdx.x / G;
    const unsigned mask = group_mask<G>(lane);
    const int F4 = A.F4;
    State<NV> st;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        st.m[j] = -INFINITY;
        st.l[j] = 0.f;
        st.acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const bool heavy = int64_t(blockIdx.x) < A.n_heavy;
    int64_t r;
    if (heavy) {
        r = blockIdx.x;
    } else {
        r = A.n_heavy + (int64_t(blockIdx.x) - A.n_heavy) * NG + gi;
        if (r >= A.n_rows) return;
    }
    const int64_t v = A.rows[r];
    const int64_t s = A.row_ptr[v], e = A.row_ptr[v + 1];
    float4 y[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = gl + G * j;
        y[j] = (c < F4) ? __ldg(Y + v * F4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (heavy) {
        const int64_t len = (e - s + NG - 1) / NG;
        const int64_t gs = min(e, s + gi * len), ge = min(e, gs + len);
        attend_range<G, NV, U, PIPE, DWT>(A, X, y, gs, ge, gl, mask, st, scores, s_idx[gi]);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int c = gl + G * j;
            s_acc[gi][c] = st.acc[j];
            s_m[gi][c] = st.m[j];
            s_l[gi][c] = st.l[j];
        }
        __syncthreads();
        for (int c = threadIdx.x; c < TW && c < F4; c += THREADS) {
            float M = -INFINITY;
            for (int g2 = 0; g2 < NG; ++g2) M = fmaxf(M, s_m[g2][c]);
            float L = 0.f;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int g2 = 0; g2 < NG; ++g2) {   // fixed order: deterministic
                if (s_m[g2][c] == -INFINITY) continue;
                const float cf = ex2(s_m[g2][c] - M);
                const float4 a = s_acc[g2][c];
                L = fmaf(s_l[g2][c], cf, L);
                acc.x = fmaf(a.x, cf, acc.x); acc.y = fmaf(a.y, cf, acc.y);
                acc.z = fmaf(a.z, cf, acc.z); acc.w = fmaf(a.w, cf, acc.w);
            }
            const float inv = 1.f / L;
            out[v * F4 + c] = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        }
        return;
    }
    attend_range<G, NV, U, PIPE, DWT>(A, X, y, s, e, gl, mask, st, scores, s_idx[gi]);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = gl + G * j;
        if (c >= F4) continue;
        if (e == s) {
            out[v * F4 + c] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            const float inv = 1.f / st.l[j];
            out[v * F4 + c] = make_float4(st.acc[j].x * inv, st.acc[j].y * inv, st.acc[j].z * inv, st.acc[j].w * inv);
        }
    }
}

template <int G, int NV, int U = (NV >= 3 ? 2 : 4), int MINB = 2, bool PIPE = true, int DWT = 0>
fg_status launch_t(Args A, const fg_graph* g, const float* X, const float* Y, float* out, float* scores,
                   cudaStream_t st) {
    constexpr int NG = THREADS / G;
    {   // rows with degree >= FG_GAT_HEAVY_DEG (default 4096) run CTA-per-row: reddit
        // H=8 D=32 14.9 ms at 256 (8 groups x 32), 14.3 at 1024, 14.0 at 4096, 14.3 at 8192
        A.n_heavy = fgk::rows_with_degree_at_least(g, g->tune.gat_heavy_deg);
    }
    const int64_t blocks = A.n_heavy + (A.n_rows - A.n_heavy + NG - 1) / NG;
    if (blocks == 0) return FG_OK;
    gat_fused_kernel<G, NV, U, MINB, PIPE, DWT><<<unsigned(blocks), THREADS, 0, st>>>(A, reinterpret_cast<const float4*>(X),
                                                                  reinterpret_cast<const float4*>(Y),
                                                                  reinterpret_cast<float4*>(out), scores);
    return fgk::check_launch("gat_fused_kernel");
}


}  // namespace

extern "C" fg_status fg_gat_attention(const fg_graph* g, int H, int D, const float* X, const float* Y, float* out,
                                      float* scores, fg_stream stream) {
    using fgk::set_error;
    if (!g) return set_error(FG_EINVAL, "fg_gat_attention: NULL graph");
    if (H < 1 || D < 1 || (int64_t(H) * D) % 4 != 0)
        return set_error(FG_ESHAPE, "fg_gat_attention: H=%d D=%d (H*D must be a multiple of 4)", H, D);
    const int F4 = H * D / 4;
    if (D % 4 != 0 || ((D / 4) & (D / 4 - 1)) != 0 || D / 4 > 32 || F4 > 128) {
        // shapes outside the fused kernel (D not 4 * 2^k <= 128, or H*D > 512): the
        // unfused chain through the caller's scores buffer -- scores, alpha in place,
        // the alpha-weighted aggregation, then the pre-softmax scores again (the
        // contract of `scores`); no allocation
        if (!scores)
            return set_error(FG_EUNSUPPORTED, "fg_gat_attention: H=%d D=%d runs unfused and needs the scores buffer",
                             H, D);
        fg_status r = fg_sddmm(g, FG_EDGE_U_DOT_V, H, D, X, Y, scores, stream);
        if (r == FG_OK) r = fg_edge_softmax(g, H, scores, scores, stream);
        if (r == FG_OK)
            r = fg_spmm(g, FG_MSG_U_MUL_E, FG_REDUCE_SUM, H, D, X, scores, nullptr, 0, nullptr, out, nullptr, nullptr,
                        nullptr, 0, stream);
        if (r == FG_OK) r = fg_sddmm(g, FG_EDGE_U_DOT_V, H, D, X, Y, scores, stream);
        return r;
    }
    if (g->n_dst == 0) return FG_OK;
    if (!X || !Y || !out) return set_error(FG_EINVAL, "fg_gat_attention: NULL tensor");
    if (!fgk::aligned16(X) || !fgk::aligned16(Y) || !fgk::aligned16(out))
        return set_error(FG_EINVAL, "fg_gat_attention: X/Y/out must be 16-byte aligned");
    Args A;
    A.rows = g->rows_by_deg;
    A.n_rows = g->n_dst;
    A.row_ptr = g->row_ptr;
    A.col_idx = g->col_idx;
    A.eid = g->eid;
    A.H = H;
    A.D4 = D / 4;
    A.F4 = F4;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int G = 32, NV = 4;
    if (F4 <= 32) {
        NV = 1;
        G = 1;
        while (G < F4) G *= 2;
        if (G < A.D4) G = A.D4;
    } else if (F4 <= 64) {
        NV = 2;
    } else if (F4 <= 96) {
        NV = 3;
    }
    switch (G) {
        case 1: return launch_t<1, 1>(A, g, X, Y, out, scores, st);
        case 2: return launch_t<2, 1>(A, g, X, Y, out, scores, st);
        case 4: return launch_t<4, 1>(A, g, X, Y, out, scores, st);
        case 8: return launch_t<8, 1>(A, g, X, Y, out, scores, st);
        case 16: return launch_t<16, 1>(A, g, X, Y, out, scores, st);
        default:
            if (NV == 1) {   // reduce-scatter scores too (K = 4 edges x 1 chunk <= D/4 lanes)
                switch (A.D4) {
                    case 4: return launch_t<32, 1, 4, 2, true, 4>(A, g, X, Y, out, scores, st);
                    case 8: return launch_t<32, 1, 4, 2, true, 8>(A, g, X, Y, out, scores, st);
                    case 16: return launch_t<32, 1, 4, 2, true, 16>(A, g, X, Y, out, scores, st);
                    case 32: return launch_t<32, 1, 4, 2, true, 32>(A, g, X, Y, out, scores, st);
                    default: return launch_t<32, 1>(A, g, X, Y, out, scores, st);
                }
            }
            // H*D in (128, 256] (reddit GAT H = 8, D = 32): 2 edges in flight per lane,
            // no software pipeline, 4 CTAs per SM (<= 64 registers).  Measured on
            // reddit (tools/gat_exp.py): 14.9 ms vs 18.4 ms for 4 edges + pipeline at
            // 2 CTAs/SM (128 registers); occupancy beats per-warp memory parallelism
            if (NV == 2) {
                // per-head scores by one reduce-scatter over the head's D/4 lanes +
                // a gather (reddit H=8 D=32: 14.0 -> 11.8 ms vs a butterfly per score)
                switch (A.D4) {
                    case 4: return launch_t<32, 2, 2, 4, false, 4>(A, g, X, Y, out, scores, st);
                    case 8: return launch_t<32, 2, 2, 4, false, 8>(A, g, X, Y, out, scores, st);
                    case 16: return launch_t<32, 2, 2, 4, false, 16>(A, g, X, Y, out, scores, st);
                    case 32: return launch_t<32, 2, 2, 4, false, 32>(A, g, X, Y, out, scores, st);
                    default: return launch_t<32, 2, 2, 4, false>(A, g, X, Y, out, scores, st);
                }
            }
            if (NV == 3) return launch_t<32, 3>(A, g, X, Y, out, scores, st);
            // reduce-scatter scores (K = 2 edges x 4 chunks <= D/4 lanes), no software
            // pipeline (reddit H=8 D=64: 32.2 vs 34.3 ms with it; 3 CTAs/SM or 1 edge: 38+)
            switch (A.D4) {
                case 8: return launch_t<32, 4, 2, 2, false, 8>(A, g, X, Y, out, scores, st);
                case 16: return launch_t<32, 4, 2, 2, false, 16>(A, g, X, Y, out, scores, st);
                case 32: return launch_t<32, 4, 2, 2, false, 32>(A, g, X, Y, out, scores, st);
                default: return launch_t<32, 4>(A, g, X, Y, out, scores, st);
            }
    }
}
