// sddmm.cu -- gSDDMM u_dot_v with H heads.
//
// Eq. (4) H_E = A . (X_V X_V^T) with the dot-product edge
// function of Fig. 5a and its multi-head form Fig. 5b:
//     out[eid(p)][h] = sum_{d<D} X[u][h][d] * Y[v][h][d],   p = (u -> v)
//
// The paper parallelises edges across a CUDA block and tree-reduces each dot
// product through shared memory (Fig. 7b; up to 2x).  On
// sm_100a the reduction is a register butterfly (__shfl_xor_sync) inside a
// group of G lanes, and the traversal is ROW-major in work units of <= 256
// edges of one destination row (fg_graph unit table): the group loads Y[v]
// into registers once per unit and then only gathers X[u] (coalesced
// LDG.128 per lane), so the kernel is bound by the gather bytes m*F*4.
// Heads are independent reductions: lanes that share a head
// (D/4 consecutive lanes) reduce together.
#include "fg_internal.h"

namespace {

constexpr int THREADS = 256;

template <int G>
__device__ __forceinline__ unsigned group_mask(int lane) {
    if constexpr (G == 32) return 0xffffffffu;
    else return ((1u << G) - 1u) << (lane & ~(G - 1));
}

struct Args {
    const int32_t* unit_row;
    const int64_t* unit_p0;
    int64_t n_units;
    int unit_chunk;
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* eid;
    const float4* X;
    const float4* Y;
    float* out;
    int H, D4, F4;
};

__device__ __forceinline__ float dot4(const float4& a, const float4& b) {
    return fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, a.w * b.w)));
}

// Butterfly sum over W consecutive lanes of the group (W a power of two <= G).
template <int G>
__device__ __forceinline__ float group_sum(float x, int W, unsigned mask) {
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1)
        if (o < W) x += __shfl_xor_sync(mask, x, o, G);
    return x;
}

// One group per work unit.  Mode A (H > 1, D4 <= G): every float4 chunk j of a
// lane belongs to head (c / D4); reduce over D4 lanes per chunk.  Mode B (H == 1
// or D4 > G): accumulate chunks in-lane, flush (reduce over all G lanes) at each
// head boundary.
template <int G, int NV>
__global__ void __launch_bounds__(THREADS) sddmm_kernel(Args A) {
    constexpr int TW = G * NV;
    constexpr int U = NV >= 4 ? 2 : (NV >= 2 ? 4 : 8);
    constexpr int B = 32, R = B / G;
    const int lane = threadIdx.x & 31;
    const int gl = threadIdx.x & (G - 1);
    const unsigned mask = group_mask<G>(lane);
    const int64_t unit = (int64_t(blockIdx.x) * THREADS + threadIdx.x) / G;
    if (unit >= A.n_units) return;
    const int64_t v = A.unit_row[unit];
    const int64_t s = A.unit_p0[unit];
    const int64_t e = min(s + A.unit_chunk, A.row_ptr[v + 1]);
    const int F4 = A.F4, H = A.H, D4 = A.D4;
    const bool modeA = (H > 1) && (D4 <= G);
    const int ntiles = (F4 + TW - 1) / TW;

    // Y[v] tile 0 stays in registers (single-tile case covers F <= 4*G*NV)
    float4 y0[NV];
    const float4* yr = A.Y + v * F4;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = gl + G * j;
        y0[j] = (c < F4) ? __ldg(yr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }

    for (int64_t p0 = s; p0 < e; p0 += B) {
        const int cnt = int(min((int64_t)B, e - p0));
        int uix[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t p = p0 + gl + r * G;
            uix[r] = (p < e) ? __ldg(A.col_idx + p) : 0;
        }
#pragma unroll
        for (int t0 = 0; t0 < B; t0 += U) {
            if (t0 >= cnt) break;
            float4 x[U][NV];
            int us[U];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = t0 + uu;
                us[uu] = __shfl_sync(mask, uix[t / G], t % G, G);
                const float4* xr = A.X + int64_t(us[uu]) * F4;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int c = gl + G * j;
                    x[uu][j] = (t < cnt && c < F4) ? __ldg(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = t0 + uu;
                if (t >= cnt) break;
                const int64_t p = p0 + t;
                const int64_t ed = A.eid ? int64_t(__ldg(A.eid + p)) : p;
                float* o = A.out + ed * H;
                if (modeA) {
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        const int c = gl + G * j;   // single tile: F4 <= TW when modeA (D4 <= G, checked at launch)
                        float part = dot4(x[uu][j], y0[j]);
                        part = group_sum<G>(part, D4, mask);
                        if (c < F4 && (gl & (D4 - 1)) == 0) o[c / D4] = part;
                    }
                } else {
                    float hs = 0.f;
                    int head = 0;
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        hs += dot4(x[uu][j], y0[j]);
                        const int cend = G * (j + 1);          // first chunk index after this j
                        if (j == NV - 1 || (H > 1 && cend % D4 == 0)) {
                            if (ntiles == 1 || H > 1) {
                                const float tot = group_sum<G>(hs, G, mask);
                                if (gl == 0 && head < H && G * j < F4) o[head] = tot;
                                hs = 0.f;
                                ++head;
                            }
                        }
                    }
                    if (ntiles > 1 && H == 1) {
                        // H == 1 with F > 4*G*NV: remaining tiles, Y re-read through L1
                        const float4* xr = A.X + int64_t(us[uu]) * F4;
                        for (int tile = 1; tile < ntiles; ++tile) {
                            for (int j = 0; j < NV; ++j) {
                                const int c = tile * TW + gl + G * j;
                                if (c < F4) hs += dot4(__ldg(xr + c), __ldg(yr + c));
                            }
                        }
                        const float tot = group_sum<G>(hs, G, mask);
                        if (gl == 0) o[0] = tot;
                    }
                }
            }
        }
    }
}

template <int G, int NV>
fg_status launch_t(const Args& A, cudaStream_t st) {
    const int64_t per_block = THREADS / G;
    const int64_t blocks = (A.n_units + per_block - 1) / per_block;
    if (blocks == 0) return FG_OK;
    sddmm_kernel<G, NV><<<unsigned(blocks), THREADS, 0, st>>>(A);
    return fgk::check_launch("sddmm_kernel");
}

}  // namespace

namespace fgk {

fg_status launch_sddmm(const fg_graph* g, int H, int D, const float* X, const float* Y, float* out,
                       cudaStream_t st) {
    Args A;
    A.unit_row = g->unit_row;
    A.unit_p0 = g->unit_p0;
    A.n_units = g->n_units;
    A.unit_chunk = g->unit_chunk;
    A.row_ptr = g->row_ptr;
    A.col_idx = g->col_idx;
    A.eid = g->eid;
    A.X = reinterpret_cast<const float4*>(X);
    A.Y = reinterpret_cast<const float4*>(Y);
    A.out = out;
    A.H = H;
    A.F4 = H * D / 4;
    A.D4 = (H > 1) ? D / 4 : A.F4;
    const int F4 = A.F4;
    int G = 32, NV = 4;
    if (F4 <= 32) {
        NV = 1;
        G = 1;
        while (G < F4) G *= 2;
    } else if (F4 <= 64) {
        NV = 2;
    } else if (F4 <= 96) {
        NV = 3;
    }
    // multi-head with F > 4*G*NV: heads larger than a tile are handled by mode B
    // only when a head boundary falls on a tile boundary of a single tile.
    if (H > 1 && F4 > G * NV)
        return set_error(FG_EUNSUPPORTED, "fg_sddmm: multi-head with H*D > 512 not implemented");
    switch (G) {
        case 1: return launch_t<1, 1>(A, st);
        case 2: return launch_t<2, 1>(A, st);
        case 4: return launch_t<4, 1>(A, st);
        case 8: return launch_t<8, 1>(A, st);
        case 16: return launch_t<16, 1>(A, st);
        default:
            if (NV == 1) return launch_t<32, 1>(A, st);
            if (NV == 2) return launch_t<32, 2>(A, st);
            if (NV == 3) return launch_t<32, 3>(A, st);
            return launch_t<32, 4>(A, st);
    }
}

}  // namespace fgk
