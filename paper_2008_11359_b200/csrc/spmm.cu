// spmm.cu -- gSpMM with gathered messages: copy_u and u_mul_e x {sum, max}
// (SURVEY §8(a) rows a1, a2).
//
// Eq. (1): out[v] = (+)_{u -> v} phi(x_u, x_uv), with
//   copy_u : phi = X[u]                    (GCN aggregation, Fig. 3a, Eq. (3))
//   u_mul_e: phi[h,d] = X[u][h][d] * E[e][h] (DGL vertex-x-edge builtin P:375; GAT P:983)
//
// B200 design (the paper's V100 schedule -- a CUDA block per adjacency row,
// threads over the feature dimension, P:521-524 -- re-derived for sm_100a):
//   * a "group" of G lanes (G = 1..32, a power of two) owns one destination row
//     and a column tile of G*NV float4s; each lane owns NV 128-bit column chunks,
//     so every gathered source row is read with coalesced LDG.128s;
//   * the row's neighbour indices are loaded 32 at a time with one coalesced
//     load per lane and broadcast with register shuffles; U edges' gathers are
//     issued before any is consumed (memory-level parallelism, Little's law:
//     SURVEY §8(d));
//   * rows are processed in degree-descending order (fg_graph rows_by_deg,
//     longest-processing-time first) and split into two modes by one launch:
//     rows with degree >= T run CTA-per-row (the CTA's groups take contiguous
//     edge ranges and combine partials in shared memory in a fixed order --
//     deterministic, no atomics; the GPU analogue of the paper's hybrid
//     degree split), the rest run group-per-row;
//   * max keeps (value, CSR position) per element; ties keep the lowest
//     position, the u_mul_e product is rounded once (__fmul_rn)
//     before the compare, matching the oracle's fp32-rounded key.
#include <algorithm>
#include <cstdlib>

#include "fg_internal.h"

namespace {

enum { OP_COPY = 0, OP_UMULE = 1, OP_UMULE_GEN = 2 };   // GEN: D % 4 != 0 (head varies inside a float4)
constexpr int THREADS = 256;

template <int G>
__device__ __forceinline__ unsigned group_mask(int lane) {
    if constexpr (G == 32) return 0xffffffffu;
    else return ((1u << G) - 1u) << (lane & ~(G - 1));
}

struct Args {
    const int32_t* rows;        // rows_by_deg
    int64_t n_heavy;            // rows[0, n_heavy) -> CTA-per-row mode
    int64_t n_rows;             // n_dst
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* eid;
    const float4* X;
    const float* E;
    int H, D, F4;
    float4* out;
    int4* arg_u;
    int4* arg_e;
};

__device__ __forceinline__ float4 f4(float a) { return make_float4(a, a, a, a); }
__device__ __forceinline__ float comp(const float4& v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
__device__ __forceinline__ void set_comp(float4& v, int k, float a) {
    if (k == 0) v.x = a; else if (k == 1) v.y = a; else if (k == 2) v.z = a; else v.w = a;
}

// Accumulate edges [s, e) of one row into (acc, pos) for this lane's NV chunks.
template <int G, int NV, int OP, bool MAX>
__device__ __forceinline__ void gather_range(const Args& A, int64_t s, int64_t e, int gl, unsigned mask,
                                             int c4base, float4 (&acc)[NV], int (&pos)[NV][4],
                                             float* __restrict__ etile) {
    constexpr int B = 32;                                   // edges per index batch
    constexpr int R = B / G;                                // indices per lane per batch
    constexpr int U = NV >= 4 ? 2 : (NV >= 2 ? 4 : 8);      // edges in flight per lane
    const int F4 = A.F4;
    for (int64_t p0 = s; p0 < e; p0 += B) {
        const int cnt = int(min((int64_t)B, e - p0));
        int uix[R];
        int eix[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t p = p0 + gl + r * G;
            uix[r] = (p < e) ? __ldg(A.col_idx + p) : 0;
            if constexpr (OP != OP_COPY) eix[r] = (p < e) ? (A.eid ? __ldg(A.eid + p) : int(p)) : 0;
        }
        // u_mul_e with identity edge ids: the batch's E rows are one contiguous span;
        // stage it in shared memory with coalesced loads instead of one dependent
        // scalar load per edge and chunk
        bool staged = false;
        if constexpr (OP == OP_UMULE && G == 32) {
            if (A.eid == nullptr && A.H <= 16) {
                staged = true;
                __syncwarp(mask);
                const float* Eb = A.E + p0 * A.H;
                for (int q = gl; q < cnt * A.H; q += G) etile[q] = __ldg(Eb + q);
                __syncwarp(mask);
            }
        }
#pragma unroll
        for (int t0 = 0; t0 < B; t0 += U) {
            if (t0 >= cnt) break;                           // uniform within the group
            float4 x[U][NV];
            float ev[U][NV][(OP == OP_UMULE_GEN) ? 4 : 1];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = t0 + uu;
                const int u = __shfl_sync(mask, uix[t / G], t % G, G);
                int ed = 0;
                if constexpr (OP != OP_COPY) ed = __shfl_sync(mask, eix[t / G], t % G, G);
                const float4* xr = A.X + int64_t(u) * F4;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int c = c4base + gl + G * j;
                    const bool ok = (t < cnt) && (c < F4);
                    x[uu][j] = ok ? __ldg(xr + c) : f4(0.f);
                    if constexpr (OP == OP_UMULE) {
                        const int h = (4 * c) / A.D;
                        ev[uu][j][0] = !ok ? 0.f : (staged ? etile[t * A.H + h] : __ldg(A.E + int64_t(ed) * A.H + h));
                    } else if constexpr (OP == OP_UMULE_GEN) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int h = (4 * c + k) / A.D;
                            ev[uu][j][k] = ok ? __ldg(A.E + int64_t(ed) * A.H + h) : 0.f;
                        }
                    }
                }
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = t0 + uu;
                if (t >= cnt) break;
                const int p = int(p0) + t;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    if constexpr (!MAX) {
                        if constexpr (OP == OP_COPY) {
                            acc[j].x += x[uu][j].x; acc[j].y += x[uu][j].y;
                            acc[j].z += x[uu][j].z; acc[j].w += x[uu][j].w;
                        } else if constexpr (OP == OP_UMULE) {
                            const float w = ev[uu][j][0];
                            acc[j].x = fmaf(x[uu][j].x, w, acc[j].x); acc[j].y = fmaf(x[uu][j].y, w, acc[j].y);
                            acc[j].z = fmaf(x[uu][j].z, w, acc[j].z); acc[j].w = fmaf(x[uu][j].w, w, acc[j].w);
                        } else {
                            acc[j].x = fmaf(x[uu][j].x, ev[uu][j][0], acc[j].x);
                            acc[j].y = fmaf(x[uu][j].y, ev[uu][j][1], acc[j].y);
                            acc[j].z = fmaf(x[uu][j].z, ev[uu][j][2], acc[j].z);
                            acc[j].w = fmaf(x[uu][j].w, ev[uu][j][3], acc[j].w);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            float m = comp(x[uu][j], k);
                            if constexpr (OP == OP_UMULE) m = __fmul_rn(m, ev[uu][j][0]);
                            else if constexpr (OP == OP_UMULE_GEN) m = __fmul_rn(m, ev[uu][j][k]);
                            if (m > comp(acc[j], k)) { set_comp(acc[j], k, m); pos[j][k] = p; }   // strict: first wins
                        }
                    }
                }
            }
        }
    }
}

template <int NV, bool MAX>
__device__ __forceinline__ void init_acc(float4 (&acc)[NV], int (&pos)[NV][4]) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        acc[j] = f4(MAX ? -INFINITY : 0.f);
#pragma unroll
        for (int k = 0; k < 4; ++k) pos[j][k] = -1;
    }
}

template <bool MAX>
__device__ __forceinline__ void store_elem(const Args& A, int64_t v, int c, float4 a, const int (&ps)[4], bool empty) {
    const int64_t o = v * A.F4 + c;
    if (!MAX) {
        A.out[o] = a;
        return;
    }
    if (empty) {
        A.out[o] = f4(0.f);
        if (A.arg_u) A.arg_u[o] = make_int4(-1, -1, -1, -1);
        if (A.arg_e) A.arg_e[o] = make_int4(-1, -1, -1, -1);
        return;
    }
    A.out[o] = a;
    if (A.arg_u) {
        int4 r;
        r.x = ps[0] < 0 ? -1 : __ldg(A.col_idx + ps[0]);
        r.y = ps[1] < 0 ? -1 : __ldg(A.col_idx + ps[1]);
        r.z = ps[2] < 0 ? -1 : __ldg(A.col_idx + ps[2]);
        r.w = ps[3] < 0 ? -1 : __ldg(A.col_idx + ps[3]);
        A.arg_u[o] = r;
    }
    if (A.arg_e) {
        int4 r;
        r.x = ps[0] < 0 ? -1 : (A.eid ? __ldg(A.eid + ps[0]) : ps[0]);
        r.y = ps[1] < 0 ? -1 : (A.eid ? __ldg(A.eid + ps[1]) : ps[1]);
        r.z = ps[2] < 0 ? -1 : (A.eid ? __ldg(A.eid + ps[2]) : ps[2]);
        r.w = ps[3] < 0 ? -1 : (A.eid ? __ldg(A.eid + ps[3]) : ps[3]);
        A.arg_e[o] = r;
    }
}

template <int G, int NV, int OP, bool MAX>
__global__ void __launch_bounds__(THREADS) spmm_gather_kernel(Args A) {
    constexpr int NG = THREADS / G;                 // groups per CTA
    constexpr int TW = G * NV;                      // float4 columns per tile
    __shared__ float4 s_acc[MAX ? 1 : NG][MAX ? 1 : TW];
    __shared__ float s_etile[(OP == OP_UMULE && G == 32) ? NG : 1][(OP == OP_UMULE && G == 32) ? 32 * 16 : 1];
    __shared__ float s_val[MAX ? NG : 1][MAX ? TW * 4 : 1];
    __shared__ int s_pos[MAX ? NG : 1][MAX ? TW * 4 : 1];

    const int lane = threadIdx.x & 31;
    const int gl = threadIdx.x & (G - 1);
    const int gi = threadIdx.x / G;
    const unsigned mask = group_mask<G>(lane);
    const int c4base = blockIdx.y * TW;

    float4 acc[NV];
    int pos[NV][4];
    init_acc<NV, MAX>(acc, pos);

    if (int64_t(blockIdx.x) < A.n_heavy) {
        // ---- CTA-per-row: contiguous edge ranges per group, fixed-order combine
        const int64_t v = A.rows[blockIdx.x];
        const int64_t s = A.row_ptr[v], e = A.row_ptr[v + 1];
        const int64_t len = (e - s + NG - 1) / NG;
        const int64_t gs = min(e, s + gi * len), ge = min(e, gs + len);
        gather_range<G, NV, OP, MAX>(A, gs, ge, gl, mask, c4base, acc, pos, s_etile[gi]);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int c = gl + G * j;
            if constexpr (!MAX) {
                s_acc[gi][c] = acc[j];
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) { s_val[gi][4 * c + k] = comp(acc[j], k); s_pos[gi][4 * c + k] = pos[j][k]; }
            }
        }
        __syncthreads();
        for (int c = threadIdx.x; c < TW; c += THREADS) {
            if (c4base + c >= A.F4) continue;
            float4 a;
            int ps[4] = {-1, -1, -1, -1};
            if constexpr (!MAX) {
                a = s_acc[0][c];
                for (int g2 = 1; g2 < NG; ++g2) {
                    const float4 b = s_acc[g2][c];
                    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
                }
            } else {
                a = f4(-INFINITY);
                for (int g2 = 0; g2 < NG; ++g2) {   // ascending ranges: strict > keeps the lowest position
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float b = s_val[g2][4 * c + k];
                        if (b > comp(a, k)) { set_comp(a, k, b); ps[k] = s_pos[g2][4 * c + k]; }
                    }
                }
            }
            store_elem<MAX>(A, v, c4base + c, a, ps, false);
        }
        return;
    }

    // ---- group-per-row
    const int64_t r = A.n_heavy + (int64_t(blockIdx.x) - A.n_heavy) * NG + gi;
    if (r >= A.n_rows) return;
    const int64_t v = A.rows[r];
    const int64_t s = A.row_ptr[v], e = A.row_ptr[v + 1];
    gather_range<G, NV, OP, MAX>(A, s, e, gl, mask, c4base, acc, pos, s_etile[gi]);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = c4base + gl + G * j;
        if (c < A.F4) store_elem<MAX>(A, v, c, acc[j], pos[j], e == s);
    }
}

template <int G, int NV, int OP, bool MAX>
fg_status launch_t(const Args& A0, cudaStream_t st) {
    Args A = A0;
    constexpr int NG = THREADS / G;
    constexpr int TW = G * NV;
    const int64_t light = A.n_rows - A.n_heavy;
    const int64_t blocks = A.n_heavy + (light + NG - 1) / NG;
    const int tiles = (A.F4 + TW - 1) / TW;
    if (blocks == 0) return FG_OK;
    const dim3 grid{unsigned(blocks), unsigned(tiles), 1u};
    spmm_gather_kernel<G, NV, OP, MAX><<<grid, THREADS, 0, st>>>(A);
    return fgk::check_launch("spmm_gather_kernel");
}

template <int G, int NV>
fg_status dispatch_op(const Args& A, int op, bool mx, cudaStream_t st) {
    if (op == OP_COPY) return mx ? launch_t<G, NV, OP_COPY, true>(A, st) : launch_t<G, NV, OP_COPY, false>(A, st);
    if (op == OP_UMULE) return mx ? launch_t<G, NV, OP_UMULE, true>(A, st) : launch_t<G, NV, OP_UMULE, false>(A, st);
    return mx ? launch_t<G, NV, OP_UMULE_GEN, true>(A, st) : launch_t<G, NV, OP_UMULE_GEN, false>(A, st);
}

}  // namespace

namespace fgk {

fg_status launch_spmm_gather(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D, const float* X,
                             const float* E, float* out, int32_t* arg_u, int32_t* arg_e, cudaStream_t st) {
    Args A;
    A.rows = g->rows_by_deg;
    A.n_rows = g->n_dst;
    A.row_ptr = g->row_ptr;
    A.col_idx = g->col_idx;
    A.eid = g->eid;
    A.X = reinterpret_cast<const float4*>(X);
    A.E = E;
    A.H = H;
    A.D = D;
    A.F4 = H * D / 4;
    A.out = reinterpret_cast<float4*>(out);
    A.arg_u = reinterpret_cast<int4*>(arg_u);
    A.arg_e = reinterpret_cast<int4*>(arg_e);
    const int op = (msg == FG_MSG_COPY_U) ? OP_COPY : (D % 4 == 0 ? OP_UMULE : OP_UMULE_GEN);
    const bool mx = (red == FG_REDUCE_MAX);
    // column mapping: G lanes x NV float4 per lane per tile.
    // Feature-dimension tiling for L2 (the paper's FDS tiling for cache, P:466-472,
    // retargeted from the CPU LLC to the B200 L2): when the source features do not
    // fit in the L2 budget, the columns are processed in tiles of T4 float4 such
    // that n_src * 16 * T4 <= budget.  Tiles are grid.y, and the block scheduler
    // issues all of tile 0 before tile 1, so each pass gathers from an L2-resident
    // slice of X; the extra cost is one re-read of col_idx per tile.
    int G = 32, NV = 4;
    int F4 = A.F4;
    {
        const int64_t budget = fgk::l2_tile_budget();
        // u_mul_e re-reads E (m x H floats) on every pass; measured not to pay off
        if (msg == FG_MSG_COPY_U && budget > 0 && g->n_src * int64_t(F4) * 16 > budget) {
            int64_t t4 = 32;
            while (t4 > 1 && g->n_src * t4 * 16 > budget) t4 /= 2;
            F4 = int(t4);            // tile width drives (G, NV) below; the kernel tiles A.F4 by G*NV
        }
    }
    if (F4 <= 32) {
        NV = 1;
        G = 1;
        while (G < F4) G *= 2;
    } else if (F4 <= 64) {
        NV = 2;
    } else if (F4 <= 96) {
        NV = 3;
    }
    const int64_t NG = THREADS / G;
    A.n_heavy = rows_with_degree_at_least(g, NG * 32);
    switch (G) {
        case 1: return dispatch_op<1, 1>(A, op, mx, st);
        case 2: return dispatch_op<2, 1>(A, op, mx, st);
        case 4: return dispatch_op<4, 1>(A, op, mx, st);
        case 8: return dispatch_op<8, 1>(A, op, mx, st);
        case 16: return dispatch_op<16, 1>(A, op, mx, st);
        default:
            if (NV == 1) return dispatch_op<32, 1>(A, op, mx, st);
            if (NV == 2) return dispatch_op<32, 2>(A, op, mx, st);
            if (NV == 3) return dispatch_op<32, 3>(A, op, mx, st);
            return dispatch_op<32, 4>(A, op, mx, st);
    }
}

}  // namespace fgk
