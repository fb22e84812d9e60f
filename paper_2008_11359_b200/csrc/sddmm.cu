// sddmm.cu -- gSDDMM u_dot_v with H heads.
//
// Eq. (4) H_E = A . (X_V X_V^T) with the dot-product edge
// function of Fig. 5a and its multi-head form Fig. 5b:
//     out[eid(p)][h] = sum_{d<D} X[u][h][d] * Y[v][h][d],   p = (u -> v)
//
// The paper parallelises edges across a CUDA block and tree-reduces each dot
// product through shared memory (Fig. 7b; up to 2x).  On
// sm_100a the reduction is a register butterfly (__shfl_xor_sync) inside a
// group of G lanes, and the traversal is ROW-major in work units of <= 64
// edges of one destination row (fg_graph unit table): the group loads Y[v]
// into registers once per unit and then only gathers X[u] (coalesced LDG.128
// per lane), so the kernel is bound by the gather bytes m*F*4.  Heads are
// independent reductions: lanes that share a head (D/4
// consecutive lanes) reduce together.
//
// Per batch of 32 edges the group stages the neighbour indices in shared
// memory (one coalesced load) and the results in shared memory (one coalesced
// store), so the loop body holds no global store and no unrolled-per-edge
// index bookkeeping: the compact body keeps the instruction stream in cache
// (the first version, fully unrolled, was instruction-fetch bound).
#include <algorithm>
#include <cstdlib>

#include "device_common.cuh"
#include "fg_internal.h"

namespace {
using namespace fgdev;

constexpr int THREADS = 256;

enum { MODE_H1 = 0, MODE_HEADS = 1, MODE_GENERAL = 2 };

struct Args {
    const int32_t* unit_row;
    const int64_t* unit_p0;
    const int64_t* unit_p1;   // explicit unit ends (source-segmented tables); NULL: min(p0 + chunk, row end)
    int64_t n_units;
    int unit_chunk;
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* eid;
    int H, D4, F4;
    int D;            // features per head (the generic multi-head kernel)
    int c4base;       // first float4 column of this pass (feature-dimension tiling, H == 1)
    int accumulate;   // pass > 0: out += partial
    int tile4;        // float4 columns per pass (0: one pass over all F4)
    int persistent;   // != 0: persistent grid (resident CTAs per SM x #SMs; > 0 caps the CTAs per SM)
    const float* E;   // u_dot_v-then-e_mul (fg_sddmm_emul): scores scaled by E[eid][h] at the write-back
    int pipe;         // H == 1 wide rows: 0 sddmm_kernel, 1..3 sddmm_h1_pipe_kernel, 4..6 sddmm_pf_kernel variants, -1 auto (FG_TUNE_SDDMM_PIPE)
};

// smallest power of two >= x: reduce_scatter halves its value count per level,
// so U*NV partial dots with NV = 3 are zero-padded to the next power of two
constexpr int pow2ceil(int x) { return x <= 1 ? 1 : 2 * pow2ceil((x + 1) / 2); }

// chunk c (4 features) of row r of a feature matrix with F4 chunks per row;
// XB: bf16 storage (the float4 pointer then addresses 8-byte chunks)
template <bool XB>
__device__ __forceinline__ float4 ld_chunk(const float4* __restrict__ M, int64_t r, int F4, int c) {
    if constexpr (XB) return bf16x4(__ldg(reinterpret_cast<const uint2*>(M) + r * F4 + c));
    else return __ldg(M + r * F4 + c);
}

// the chunk at byte address p (fp32: 16 bytes; bf16 storage: 8 bytes decoded)
template <bool XB>
__device__ __forceinline__ float4 ld_at(const char* p) {
    if constexpr (XB) return bf16x4(__ldg(reinterpret_cast<const uint2*>(p)));
    else return __ldg(reinterpret_cast<const float4*>(p));
}

// MODE_H1      : H == 1 and F <= 4*G*NV: one dot per edge, reduce over all G lanes.
// MODE_HEADS   : H > 1, D4 = D/4 <= G (power of two), F <= 4*G*NV: chunk j of a
//                lane belongs to head c / D4; reduce over D4 lanes per chunk.
// MODE_GENERAL : H == 1 with F > 4*G*NV (column tiles; Y re-read through L1), or
//                H > 1 with D4 > G (a head spans several chunks of a lane).
// FULLW: F4 == G*NV exactly (every lane's every chunk is inside the row): no
// per-chunk column predicate.
template <int G, int NV, int MODE, int DW, bool XB, bool EM = false, bool FULLW = false>
__global__ void __launch_bounds__(THREADS, 3) sddmm_kernel(const Args A, const float4* __restrict__ X,
                                                           const float4* __restrict__ Y, float* __restrict__ out) {
    constexpr int TW = G * NV;
    constexpr int B = G >= 4 ? 32 : 8;              // edges per batch
    constexpr int U = NV >= 3 ? 2 : (NV == 2 ? 4 : 8);   // edges in flight per lane
    constexpr int NGRP = THREADS / G;
    constexpr int CAP = 32 * G;                           // staged results per group
    __shared__ int s_idx[NGRP][B];
    __shared__ float s_res[NGRP][CAP];
    const int lane = threadIdx.x & 31;
    const int gl = threadIdx.x & (G - 1);
    const int gi = threadIdx.x / G;
    const unsigned mask = group_mask<G>(lane);
    // grid-stride over the work units: one unit per group when the grid covers them
    // all, or a persistent grid (A.persistent) whose groups walk the unit list in
    // order -- concurrent groups then stay inside one source segment, and no CTA
    // launch is paid per short unit
    const int64_t stride = int64_t(gridDim.x) * (THREADS / G);
    for (int64_t unit = (int64_t(blockIdx.x) * THREADS + threadIdx.x) / G; unit < A.n_units; unit += stride) {
    const int64_t v = A.unit_row[unit];
    const int64_t s = A.unit_p0[unit];
    const int64_t e = A.unit_p1 ? A.unit_p1[unit] : min(s + A.unit_chunk, A.row_ptr[v + 1]);
    const int F4 = A.F4, H = A.H, D4 = A.D4;
    const bool stage = (H * B <= CAP);
    constexpr int CB = XB ? 8 : 16;                                        // bytes per 4-feature chunk
    const char* xl = reinterpret_cast<const char*>(X) + int64_t(A.c4base + gl) * CB;   // this lane's column
    const uint32_t rowb = uint32_t(F4) * CB;                              // bytes per X row
    int* idx = s_idx[gi];
    float* res = s_res[gi];

    float4 y0[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = A.c4base + gl + G * j;
        y0[j] = (c < F4) ? ld_chunk<XB>(Y, v, F4, c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }

    constexpr int PF = (B + G - 1) / G;   // running sums per lane in a tiled pass (H == 1)
    for (int64_t p0 = s; p0 < e; p0 += B) {
        const int cnt = int(min((int64_t)B, e - p0));
        __syncwarp(mask);
        for (int t = gl; t < cnt; t += G) idx[t] = __ldg(A.col_idx + p0 + t);
        // column-tiled pass k > 0 (H == 1): fetch the batch's running sums now, so the
        // read-modify-write at the end of the batch does not wait a DRAM round trip
        float prev[PF];
        if (A.accumulate) {
#pragma unroll
            for (int k = 0; k < PF; ++k) {
                const int q = gl + G * k;
                prev[k] = (q < cnt) ? out[A.eid ? int64_t(__ldg(A.eid + p0 + q)) : p0 + q] : 0.f;
            }
        }
        __syncwarp(mask);
        for (int t0 = 0; t0 < cnt; t0 += U) {
            float4 x[U][NV];
            int us[U];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                // past the batch end: re-read the last edge's row (an L1 hit) instead of
                // predicating every load -- its result is never stored (staged slots
                // beyond cnt are not written back; the unstaged path breaks at cnt)
                const int t = min(t0 + uu, cnt - 1);
                us[uu] = idx[t];
                const char* xr = xl + uint64_t(uint32_t(us[uu])) * rowb;   // one IMAD.WIDE.U32
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int c = A.c4base + gl + G * j;
                    x[uu][j] = (FULLW || c < F4) ? ld_at<XB>(xr + j * G * CB) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            if constexpr (MODE == MODE_H1 || MODE == MODE_HEADS) {
                if (stage) {
                    // reduce-scatter of the U edges' (x NV chunk) partial dots over the DW
                    // lanes that share a head: ~log2(DW) + (K-1)/... shuffles per U edges
                    // instead of log2(DW) per edge and chunk
                    constexpr int KR = (MODE == MODE_H1) ? U : U * NV;   // real partial dots
                    constexpr int K = pow2ceil(KR);
                    float pv[K];
#pragma unroll
                    for (int k = KR; k < K; ++k) pv[k] = 0.f;
#pragma unroll
                    for (int uu = 0; uu < U; ++uu) {
                        if constexpr (MODE == MODE_H1) {
                            float hs = 0.f;
#pragma unroll
                            for (int j = 0; j < NV; ++j) hs += dot4(x[uu][j], y0[j]);
                            pv[uu] = hs;
                        } else {
#pragma unroll
                            for (int j = 0; j < NV; ++j) pv[uu * NV + j] = dot4(x[uu][j], y0[j]);
                        }
                    }
                    reduce_scatter<K, DW, G>(pv, gl, mask);
                    constexpr int L = ilog2(K) < ilog2(DW) ? ilog2(K) : ilog2(DW);
                    constexpr int KEEP = K >> L;                       // values held per lane
                    const int sub = gl & (DW - 1);
                    const int bits = sub >> (ilog2(DW) - L);
                    if ((sub & ((DW >> L) - 1)) == 0) {
#pragma unroll
                        for (int i = 0; i < KEEP; ++i) {
                            const int id = bits * KEEP + i;
                            if constexpr (MODE == MODE_H1) {
                                res[t0 + id] = pv[i];
                            } else {
                                const int uu = id / NV, j = id % NV;
                                const int head = gl / DW + j * (G / DW);
                                if (id < KR && head < H) res[(t0 + uu) * H + head] = pv[i];
                            }
                        }
                    }
                    continue;
                }
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = t0 + uu;
                if (t >= cnt) break;
                float* rr = stage ? res + t * H
                                  : out + (A.eid ? int64_t(__ldg(A.eid + p0 + t)) : (p0 + t)) * H;
                if constexpr (MODE == MODE_H1) {
                    float hs = 0.f;
#pragma unroll
                    for (int j = 0; j < NV; ++j) hs += dot4(x[uu][j], y0[j]);
                    hs = group_sum<G>(hs, G, mask);
                    if (gl == 0) rr[0] = hs;
                } else if constexpr (MODE == MODE_HEADS) {
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        const int c = gl + G * j;
                        const float part = group_sum<G>(dot4(x[uu][j], y0[j]), D4, mask);
                        if (c < F4 && (gl & (D4 - 1)) == 0) rr[c / D4] = part;
                    }
                } else {
                    const int ntiles = (F4 + TW - 1) / TW;
                    float hs = 0.f;
                    int head = 0;
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        hs += dot4(x[uu][j], y0[j]);
                        const int cend = G * (j + 1);
                        if (H > 1 && (j == NV - 1 || cend % D4 == 0)) {
                            const float tot = group_sum<G>(hs, G, mask);
                            if (gl == 0 && head < H) rr[head] = tot;
                            hs = 0.f;
                            ++head;
                        }
                    }
                    if (H == 1) {
                        for (int tile = 1; tile < ntiles; ++tile)
                            for (int j = 0; j < NV; ++j) {
                                const int c = tile * TW + gl + G * j;
                                if (c < F4) hs += dot4(ld_chunk<XB>(X, us[uu], F4, c), ld_chunk<XB>(Y, v, F4, c));
                            }
                        const float tot = group_sum<G>(hs, G, mask);
                        if (gl == 0) rr[0] = tot;
                    }
                }
            }
        }
        if (stage) {   // coalesced write-back of the batch's results
            __syncwarp(mask);
            const int tot = cnt * H;
            if (A.accumulate) {   // H == 1: q == t
#pragma unroll
                for (int k = 0; k < PF; ++k) {
                    const int q = gl + G * k;
                    if (q < cnt) out[A.eid ? int64_t(__ldg(A.eid + p0 + q)) : p0 + q] = prev[k] + res[q];
                }
            } else if (A.eid == nullptr) {
                float* o = out + p0 * H;
                if constexpr (EM) {   // u_dot_v then e_mul: scale at the write-back
                    const float* ew = A.E + p0 * H;
                    for (int q = gl; q < tot; q += G) o[q] = res[q] * __ldg(ew + q);
                } else {
                    for (int q = gl; q < tot; q += G) o[q] = res[q];
                }
            } else {
                for (int q = gl; q < tot; q += G) {
                    const int t = q / H, h = q - t * H;
                    const int64_t oi = int64_t(__ldg(A.eid + p0 + t)) * H + h;
                    if constexpr (EM) out[oi] = res[q] * __ldg(A.E + oi);
                    else out[oi] = res[q];
                }
            }
        }
    }
    }   // units
}

// bf16 storage (fg_sddmm_x16): each lane reads PAIRS of 4-feature chunks (8
// bf16) with one 16-byte load and keeps them raw until the dot, so U = 4 / 8
// edges stay in flight -- the same bytes in flight per warp as the fp32
// mapping, half the gathered bytes.  Lane gl owns pairs gl + G*j (j < NP).
//   DWP == G (H == 1): one dot per edge over all G lanes;
//   DWP <  G (H > 1): a head spans D/8 = DWP consecutive pairs, i.e. DWP lanes;
//                     pair j of lane gl belongs to head gl/DWP + j*(G/DWP).
// Same unit walk, batching, reduce-scatter and coalesced result write-back as
// sddmm_kernel (MODE_H1 / MODE_HEADS).
template <int G, int NP, int DWP>
__global__ void __launch_bounds__(THREADS, 3) sddmm_pair_kernel(const Args A, const uint4* __restrict__ X,
                                                                const uint4* __restrict__ Y,
                                                                float* __restrict__ out) {
    constexpr bool H1 = (DWP == G);
    constexpr int B = G >= 4 ? 32 : 8;      // edges per batch
    constexpr int U = NP >= 2 ? 4 : 8;      // edges in flight per lane (4 for NP = 1 measured 2 % slower)
    constexpr int NGRP = THREADS / G;
    constexpr int CAP = 32 * G;             // staged results per group (B * H <= CAP, checked by the host)
    __shared__ int s_idx[NGRP][B];
    __shared__ float s_res[NGRP][CAP];
    const int lane = threadIdx.x & 31;
    const int gl = threadIdx.x & (G - 1);
    const int gi = threadIdx.x / G;
    const unsigned mask = group_mask<G>(lane);
    const int P8 = A.F4 / 2;                 // 8-feature pairs per row
    const int H = A.H;
    const int64_t stride = int64_t(gridDim.x) * (THREADS / G);
    for (int64_t unit = (int64_t(blockIdx.x) * THREADS + threadIdx.x) / G; unit < A.n_units; unit += stride) {
        const int64_t v = A.unit_row[unit];
        const int64_t s = A.unit_p0[unit];
        const int64_t e = A.unit_p1 ? A.unit_p1[unit] : min(s + A.unit_chunk, A.row_ptr[v + 1]);
        int* idx = s_idx[gi];
        float* res = s_res[gi];
        float4 ylo[NP], yhi[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int c = gl + G * j;
            const uint4 w = (c < P8) ? __ldg(Y + v * P8 + c) : make_uint4(0, 0, 0, 0);
            ylo[j] = bf16x4(make_uint2(w.x, w.y));
            yhi[j] = bf16x4(make_uint2(w.z, w.w));
        }
        for (int64_t p0 = s; p0 < e; p0 += B) {
            const int cnt = int(min((int64_t)B, e - p0));
            __syncwarp(mask);
            for (int t = gl; t < cnt; t += G) idx[t] = __ldg(A.col_idx + p0 + t);
            __syncwarp(mask);
            for (int t0 = 0; t0 < cnt; t0 += U) {
                uint4 xw[U][NP];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int t = t0 + uu;
                    const int64_t u = (t < cnt) ? idx[t] : 0;
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        const int c = gl + G * j;
                        xw[uu][j] = (t < cnt && c < P8) ? __ldg(X + u * P8 + c) : make_uint4(0, 0, 0, 0);
                    }
                }
                constexpr int K = H1 ? U : U * NP;
                float pv[K];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    float hs = 0.f;
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        const float d = dot4(bf16x4(make_uint2(xw[uu][j].x, xw[uu][j].y)), ylo[j]) +
                                        dot4(bf16x4(make_uint2(xw[uu][j].z, xw[uu][j].w)), yhi[j]);
                        if constexpr (H1) hs += d;
                        else pv[uu * NP + j] = d;
                    }
                    if constexpr (H1) pv[uu] = hs;
                }
                reduce_scatter<K, DWP, G>(pv, gl, mask);
                constexpr int L = ilog2(K) < ilog2(DWP) ? ilog2(K) : ilog2(DWP);
                constexpr int KEEP = K >> L;
                const int sub = gl & (DWP - 1);
                const int bits = sub >> (ilog2(DWP) - L);
                if ((sub & ((DWP >> L) - 1)) == 0) {
#pragma unroll
                    for (int i = 0; i < KEEP; ++i) {
                        const int id = bits * KEEP + i;
                        if constexpr (H1) {
                            res[t0 + id] = pv[i];
                        } else {
                            const int uu = id / NP, j = id % NP;
                            const int head = gl / DWP + j * (G / DWP);
                            if (head < H) res[(t0 + uu) * H + head] = pv[i];
                        }
                    }
                }
            }
            __syncwarp(mask);   // coalesced write-back of the batch's results
            const int tot = cnt * H;
            if (A.eid == nullptr) {
                float* o = out + p0 * H;
                for (int q = gl; q < tot; q += G) o[q] = res[q];
            } else {
                for (int q = gl; q < tot; q += G) {
                    const int t = q / H, h = q - t * H;
                    out[int64_t(__ldg(A.eid + p0 + t)) * H + h] = res[q];
                }
            }
        }
    }
}

// Ablation E6: the per-edge dot product computed by ONE
// thread, walking the whole feature row (the "thread-per-edge" alternative the
// paper's tree reduction is measured against: "consume too many registers" at
// large F).  A warp takes one work unit (<= unit_chunk edges of one destination
// row), lane l the edges p0 + l, p0 + l + 32, ...; Y[v] is shared by the warp
// (L1).  Same unit tables, same outputs; the per-edge summation order differs
// from the lane-partitioned kernels (within tolerance, not bit-identical).
__global__ void __launch_bounds__(THREADS) sddmm_thread_kernel(const Args A, const float4* __restrict__ X,
                                                               const float4* __restrict__ Y, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = int64_t(gridDim.x) * (THREADS / 32);
    const int F4 = A.F4, D4 = A.D4, H = A.H;
    for (int64_t unit = (int64_t(blockIdx.x) * THREADS + threadIdx.x) / 32; unit < A.n_units; unit += nwarps) {
        const int64_t v = A.unit_row[unit];
        const int64_t s = A.unit_p0[unit];
        const int64_t e = A.unit_p1 ? A.unit_p1[unit] : min(s + A.unit_chunk, A.row_ptr[v + 1]);
        for (int64_t p = s + lane; p < e; p += 32) {
            const int64_t u = __ldg(A.col_idx + p);
            const int64_t eo = (A.eid ? int64_t(__ldg(A.eid + p)) : p) * H;
            const float4* xr = X + u * F4;
            const float4* yr = Y + v * F4;
            float acc = 0.f;
            int h = 0;
            for (int c = 0; c < F4; ++c) {
                acc += dot4(__ldg(xr + c), __ldg(yr + c));
                if ((c + 1) % D4 == 0) {   // end of head h
                    out[eo + h] = A.E ? acc * __ldg(A.E + eo + h) : acc;
                    acc = 0.f;
                    ++h;
                }
            }
        }
    }
}

// Software-pipelined H == 1 gather for wide rows (G = 32 lanes, NV float4 per
// lane; F = 132..512): a work unit's (<= 64) neighbour indices are staged in
// shared memory once, then the loop keeps the NEXT U edges' X rows in flight
// while it reduces the current U (two register buffers, ping-pong by manual
// unrolling, so no register copy waits on a load).  The non-pipelined kernel
// drains its loads every U edges: its warps hold 0 bytes in flight while they
// reduce.  Same per-lane partial dots and the same reduce-scatter tree as
// sddmm_kernel<32, NV, MODE_H1>: bit-identical results.
template <int NV, int U, int MINB, bool EM>
__global__ void __launch_bounds__(THREADS, MINB) sddmm_h1_pipe_kernel(const Args A, const float4* __restrict__ X,
                                                                      const float4* __restrict__ Y,
                                                                      float* __restrict__ out) {
    constexpr int NGRP = THREADS / 32;
    constexpr int CH = 64;   // max edges per work unit (host-checked: unit_chunk <= 64)
    __shared__ int s_idx[NGRP][CH];
    __shared__ float s_res[NGRP][CH];
    const int gl = threadIdx.x & 31;
    const int gi = threadIdx.x >> 5;
    constexpr unsigned mask = 0xffffffffu;
    int* idx = s_idx[gi];
    float* res = s_res[gi];
    const int F4 = A.F4;
    const char* xl = reinterpret_cast<const char*>(X + gl);   // this lane's first column
    const uint32_t rowb = uint32_t(F4) * 16u;
    bool cin[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) cin[j] = gl + 32 * j < F4;
    const int64_t stride = int64_t(gridDim.x) * NGRP;
    for (int64_t unit = int64_t(blockIdx.x) * NGRP + gi; unit < A.n_units; unit += stride) {
        const int64_t v = A.unit_row[unit];
        const int64_t s = A.unit_p0[unit];
        const int64_t e = A.unit_p1 ? A.unit_p1[unit] : min(s + A.unit_chunk, A.row_ptr[v + 1]);
        const int cnt = int(e - s);
        __syncwarp();
        for (int t = gl; t < cnt; t += 32) idx[t] = __ldg(A.col_idx + s + t);
        float4 y0[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int c = gl + 32 * j;
            y0[j] = (c < F4) ? __ldg(Y + v * F4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncwarp();
        auto load = [&](float4 (&x)[U][NV], int t0) {   // past cnt: the last row again, never stored
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const char* xr = xl + uint64_t(uint32_t(idx[min(t0 + uu, cnt - 1)])) * rowb;
#pragma unroll
                for (int j = 0; j < NV; ++j)
                    x[uu][j] = cin[j] ? __ldg(reinterpret_cast<const float4*>(xr) + 32 * j)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        auto reduce = [&](const float4 (&x)[U][NV], int t0) {
            float pv[U];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                float hs = 0.f;
#pragma unroll
                for (int j = 0; j < NV; ++j) hs += dot4(x[uu][j], y0[j]);
                pv[uu] = hs;
            }
            reduce_scatter<U, 32, 32>(pv, gl, mask);
            constexpr int L = ilog2(U) < 5 ? ilog2(U) : 5;
            constexpr int KEEP = U >> L;
            const int bits = gl >> (5 - L);
            if ((gl & ((32 >> L) - 1)) == 0) {
#pragma unroll
                for (int i = 0; i < KEEP; ++i) {
                    const int t = t0 + bits * KEEP + i;
                    if (t < cnt) res[t] = pv[i];
                }
            }
        };
        float4 xa[U][NV], xb[U][NV];
        load(xa, 0);
        for (int t0 = 0; t0 < cnt; t0 += 2 * U) {
            if (t0 + U < cnt) load(xb, t0 + U);       // uniform: next U edges in flight ...
            reduce(xa, t0);                          // ... while this U reduce
            if (t0 + U >= cnt) break;
            if (t0 + 2 * U < cnt) load(xa, t0 + 2 * U);
            reduce(xb, t0 + U);
        }
        __syncwarp();
        if (A.eid == nullptr) {
            for (int q = gl; q < cnt; q += 32) {
                if constexpr (EM) out[s + q] = res[q] * __ldg(A.E + s + q);
                else out[s + q] = res[q];
            }
        } else {
            for (int q = gl; q < cnt; q += 32) {
                const int64_t oi = __ldg(A.eid + s + q);
                if constexpr (EM) out[oi] = res[q] * __ldg(A.E + oi);
                else out[oi] = res[q];
            }
        }
    }
}

// shared-memory float4 read that the compiler may not hoist out of a loop (keeps
// the Y chunks of sddmm_pf_kernel<YS = true> out of registers)
__device__ __forceinline__ float4 lds_f4(const float4* p) {
    float4 r;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
    return r;
}

// Unit-prefetching gather (G = 32 lanes, NV float4 per lane; H == 1 with DW =
// 32, or H heads of D = 4*DW features).  A work unit (<= 64 edges of one row
// inside one source segment; 35 on average on the reddit-shaped graph) starts
// with two dependent global round trips before its first X gather: the unit
// table, then the row's neighbour indices and Y[v].  Here each warp stages the
// NEXT unit's indices and Y row into a second shared-memory buffer with cp.async
// (LDGSTS: no registers held) and loads the unit table entry of the one after,
// while it gathers the current unit; so a unit's X gathers start as soon as the
// previous unit ends.
//   YS == false: Y[v] copied into registers at the unit start (as sddmm_kernel);
//   YS == true : Y read from shared memory chunk by chunk inside the edge loop.
// Same per-lane partial dots, same U edges per reduce-scatter and the same tree
// as sddmm_kernel<32, NV, MODE_H1 / MODE_HEADS, DW>: bit-identical results.
template <int NV, int DW, bool YS, int MINB, bool EM, int UO = 0>
__global__ void __launch_bounds__(THREADS, MINB) sddmm_pf_kernel(const Args A, const float4* __restrict__ X,
                                                                 const float4* __restrict__ Y,
                                                                 float* __restrict__ out) {
    constexpr int NGRP = THREADS / 32;
    constexpr int CH = 64;                                   // max edges per work unit (host-checked)
    constexpr bool H1 = (DW == 32);
    // edges per reduce-scatter: as sddmm_kernel (UO != 0: an override, same tree only
    // for the same U)
    constexpr int U = UO ? UO : (NV >= 3 ? 2 : (NV == 2 ? 4 : 8));
    constexpr int HMAX = H1 ? 1 : 32 * NV / DW;              // heads per row
    // dynamic shared memory (pf_smem_bytes): per warp two Y buffers, two index
    // buffers and the unit's staged results
    extern __shared__ __align__(16) unsigned char pf_smem[];
    auto s_y = reinterpret_cast<float4 (*)[2][32 * NV]>(pf_smem);
    auto s_idx = reinterpret_cast<int (*)[2][CH]>(pf_smem + NGRP * 2 * 32 * NV * 16);
    auto s_res = reinterpret_cast<float (*)[CH * HMAX]>(pf_smem + NGRP * (2 * 32 * NV * 16 + 2 * CH * 4));
    const int gl = threadIdx.x & 31;
    const int gi = threadIdx.x >> 5;
    constexpr unsigned mask = 0xffffffffu;
    float* res = s_res[gi];
    const int F4 = A.F4, H = H1 ? 1 : A.H;
    const char* xl = reinterpret_cast<const char*>(X + gl);   // this lane's first column
    const uint32_t rowb = uint32_t(F4) * 16u;
    bool cin[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) cin[j] = gl + 32 * j < F4;
    const int64_t stride = int64_t(gridDim.x) * NGRP;
    const int64_t n_units = A.n_units;
    auto meta = [&](int64_t u, int64_t& v, int64_t& s, int& cnt) {
        v = A.unit_row[u];
        s = A.unit_p0[u];
        const int64_t e = A.unit_p1 ? A.unit_p1[u] : min(s + A.unit_chunk, A.row_ptr[v + 1]);
        cnt = int(e - s);
    };
    auto stage = [&](int buf, int64_t v, int64_t s, int cnt) {   // one commit group per unit
        int* idx = s_idx[gi][buf];
        for (int t = gl; t < cnt; t += 32) cp_async4_ca(idx + t, A.col_idx + s + t);
        float4* yb = s_y[gi][buf];
#pragma unroll
        for (int j = 0; j < NV; ++j)
            if (cin[j]) cp_async16_cg(yb + gl + 32 * j, Y + v * F4 + gl + 32 * j);
        cp_async_commit();
    };
    int64_t unit = int64_t(blockIdx.x) * NGRP + gi;
    if (unit >= n_units) return;
    int64_t v0, s0, v1 = 0, s1 = 0;
    int c0, c1 = 0;
    meta(unit, v0, s0, c0);
    stage(0, v0, s0, c0);
    if (unit + stride < n_units) meta(unit + stride, v1, s1, c1);
    int buf = 0;
    for (; unit < n_units; unit += stride) {
        // the next unit's indices and Y row into the other buffer (an empty group at
        // the end keeps the wait count uniform), then the unit table entry after it
        if (unit + stride < n_units) stage(buf ^ 1, v1, s1, c1);
        else cp_async_commit();
        int64_t v2 = 0, s2 = 0;
        int c2 = 0;
        if (unit + 2 * stride < n_units) meta(unit + 2 * stride, v2, s2, c2);
        cp_async_wait<1>();   // this unit's group has landed (this lane's copies) ...
        __syncwarp();         // ... and every lane's
        const int* idx = s_idx[gi][buf];
        const float4* yb = s_y[gi][buf];
        const int cnt = c0;
        float4 y0[YS ? 1 : NV];
        if constexpr (!YS) {
#pragma unroll
            for (int j = 0; j < NV; ++j) y0[j] = cin[j] ? yb[gl + 32 * j] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll 1
        for (int t0 = 0; t0 < cnt; t0 += U) {
            float4 x[U][NV];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {   // past cnt: the last row again, never stored
                const char* xr = xl + uint64_t(uint32_t(idx[min(t0 + uu, cnt - 1)])) * rowb;
#pragma unroll
                for (int j = 0; j < NV; ++j)
                    x[uu][j] = cin[j] ? __ldg(reinterpret_cast<const float4*>(xr) + 32 * j)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            constexpr int KR = H1 ? U : U * NV;   // real partial dots (zero-padded to a power of two)
            constexpr int K = pow2ceil(KR);
            float pv[K];
#pragma unroll
            for (int k = 0; k < K; ++k) pv[k] = 0.f;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                float4 yj;
                if constexpr (YS) yj = cin[j] ? lds_f4(yb + gl + 32 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
                else yj = y0[j];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    if constexpr (H1) pv[uu] += dot4(x[uu][j], yj);
                    else pv[uu * NV + j] = dot4(x[uu][j], yj);
                }
            }
            reduce_scatter<K, DW, 32>(pv, gl, mask);
            constexpr int L = ilog2(K) < ilog2(DW) ? ilog2(K) : ilog2(DW);
            constexpr int KEEP = K >> L;                       // values held per lane
            const int sub = gl & (DW - 1);
            const int bits = sub >> (ilog2(DW) - L);
            if ((sub & ((DW >> L) - 1)) == 0) {
#pragma unroll
                for (int i = 0; i < KEEP; ++i) {
                    const int id = bits * KEEP + i;
                    if constexpr (H1) {
                        if (t0 + id < cnt) res[t0 + id] = pv[i];
                    } else {
                        const int uu = id / NV, j = id % NV;
                        const int head = gl / DW + j * (32 / DW);
                        if (id < KR && head < H && t0 + uu < cnt) res[(t0 + uu) * H + head] = pv[i];
                    }
                }
            }
        }
        __syncwarp();
        const int tot = cnt * H;
        if (A.eid == nullptr) {
            float* o = out + s0 * H;
            for (int q = gl; q < tot; q += 32) {
                if constexpr (EM) o[q] = res[q] * __ldg(A.E + s0 * H + q);
                else o[q] = res[q];
            }
        } else {
            for (int q = gl; q < tot; q += 32) {
                const int t = H1 ? q : q / H, h = q - t * H;
                const int64_t oi = int64_t(__ldg(A.eid + s0 + t)) * H + h;
                if constexpr (EM) out[oi] = res[q] * __ldg(A.E + oi);
                else out[oi] = res[q];
            }
        }
        __syncwarp();   // res / idx / y of this buffer are free before they are refilled
        v0 = v1; s0 = s1; c0 = c1;
        v1 = v2; s1 = s2; c1 = c2;
        buf ^= 1;
    }
}

// Generic multi-head u_dot_v for shapes the lane-partitioned kernels do not
// cover (D not a multiple of 4 or D/4 not a power of two, or H*D > 512): a warp
// per work unit, a thread per edge walking the feature row in float4 chunks and
// closing head h after its D-th product (heads may start inside a chunk).  Each
// head's dot is one sequential fp32 FMA chain in feature order.  The support
// path for unusual head shapes (thread-per-edge gathers are 2.5-4.3x slower
// than the lane-partitioned kernels at the shapes both run, ablation E6).
__global__ void __launch_bounds__(THREADS) sddmm_heads_generic_kernel(const Args A, const float4* __restrict__ X,
                                                                      const float4* __restrict__ Y,
                                                                      float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = int64_t(gridDim.x) * (THREADS / 32);
    const int F4 = A.F4, H = A.H, D = A.D;
    for (int64_t unit = (int64_t(blockIdx.x) * THREADS + threadIdx.x) / 32; unit < A.n_units; unit += nwarps) {
        const int64_t v = A.unit_row[unit];
        const int64_t s = A.unit_p0[unit];
        const int64_t e = A.unit_p1 ? A.unit_p1[unit] : min(s + A.unit_chunk, A.row_ptr[v + 1]);
        for (int64_t p = s + lane; p < e; p += 32) {
            const int64_t u = __ldg(A.col_idx + p);
            const int64_t eo = (A.eid ? int64_t(__ldg(A.eid + p)) : p) * H;
            const float4* xr = X + u * F4;
            const float4* yr = Y + v * F4;
            float acc = 0.f;
            int h = 0, k = 0;
            for (int c = 0; c < F4; ++c) {
                const float4 x = __ldg(xr + c), y = __ldg(yr + c);
                const float xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc = fmaf(xs[q], ys[q], acc);
                    if (++k == D) {   // head h complete
                        out[eo + h] = A.E ? acc * __ldg(A.E + eo + h) : acc;
                        acc = 0.f;
                        k = 0;
                        ++h;
                    }
                }
            }
        }
    }
}

// FG_TUNE_SDDMM_PIPE = 7: the unit-prefetching kernel with twice the plain kernel's
// edges per lane in flight at 2 CTAs per SM (NV = 2: 8, NV = 3 / 4: 4)
template <int NV>
constexpr int PF2U = NV >= 3 ? 4 : (NV == 2 ? 8 : 16);

// shared-memory bytes of sddmm_pf_kernel<NV, DW>
constexpr int pf_smem_bytes(int NV, int DW) {
    return (THREADS / 32) * (2 * 32 * NV * 16 + 2 * 64 * 4 + 64 * (DW == 32 ? 1 : 32 * NV / DW) * 4);
}

template <int G, int NV, bool XB = false>
fg_status launch_t(const Args& A, const float4* X, const float4* Y, float* out, cudaStream_t st) {
    using K = void (*)(const Args, const float4*, const float4*, float*);
    const int TW = G * NV;
    K k;
    int dsmem = 0;   // dynamic shared memory of the chosen kernel (sddmm_pf_kernel only)
    // full-width rows (F4 == G*NV, one pass): the variant without per-chunk column predicates
    const bool fullw = !XB && A.tile4 == 0 && A.c4base == 0 && A.F4 == TW;
    if (A.H == 1 && (A.tile4 ? A.tile4 : A.F4) <= TW) {
        k = fullw ? sddmm_kernel<G, NV, MODE_H1, G, XB, false, true> : sddmm_kernel<G, NV, MODE_H1, G, XB>;
    } else if (A.H > 1 && A.D4 <= G && A.F4 <= TW) {
        switch (A.D4) {   // heads of D = 4*D4 floats reduce over D4 lanes
            case 1: k = sddmm_kernel<G, NV, MODE_HEADS, 1, XB>; break;
            case 2: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 2 ? 2 : 1), XB>; break;
            case 4: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 4 ? 4 : 1), XB>; break;
            case 8:
                k = fullw ? sddmm_kernel<G, NV, MODE_HEADS, (G >= 8 ? 8 : 1), XB, false, true>
                          : sddmm_kernel<G, NV, MODE_HEADS, (G >= 8 ? 8 : 1), XB>;
                break;
            case 16: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 16 ? 16 : 1), XB>; break;
            default: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 32 ? 32 : 1), XB>; break;
        }
    } else {
        k = sddmm_kernel<G, NV, MODE_GENERAL, 1, XB>;
    }
    if constexpr (!XB) {   // u_dot_v then e_mul (fg_sddmm_emul, fp32 only): the staged modes
        if (A.E) {
            if (A.H == 1 && (A.tile4 ? A.tile4 : A.F4) <= TW) {
                k = sddmm_kernel<G, NV, MODE_H1, G, false, true>;
            } else if (A.H > 1 && A.D4 <= G && A.F4 <= TW) {
                switch (A.D4) {
                    case 1: k = sddmm_kernel<G, NV, MODE_HEADS, 1, false, true>; break;
                    case 2: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 2 ? 2 : 1), false, true>; break;
                    case 4: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 4 ? 4 : 1), false, true>; break;
                    case 8: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 8 ? 8 : 1), false, true>; break;
                    case 16: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 16 ? 16 : 1), false, true>; break;
                    default: k = sddmm_kernel<G, NV, MODE_HEADS, (G >= 32 ? 32 : 1), false, true>; break;
                }
            } else {
                k = sddmm_kernel<G, NV, MODE_GENERAL, 1, false, true>;
            }
        }
    }
    if constexpr (G == 32 && NV >= 2 && !XB) {   // software-pipelined wide-row H == 1 kernel (FG_TUNE_SDDMM_PIPE)
        // auto (-1), measured on reddit (tools/sddmm_ab.py): the software-pipelined U=2
        // kernel for NV = 3 (F=384: 12.21 plain -> 10.27 ms; unit-prefetching 11.2-11.7);
        // the unit-prefetching kernel for NV = 2 (F=256: 7.07 -> 6.72 ms) and, with 4
        // edges in flight per lane at 2 CTAs per SM, for NV = 4 (F=512: 14.79 plain,
        // 14.38 at U = 2 / 3 CTAs, 14.20 at U = 4 / 2 CTAs; on another box 14.55 /
        // 14.15 / 13.84); the software-pipelined variants 8.26-9.12 / 15.41-30.5
        const int pipe = A.pipe < 0 ? (NV == 3 ? 3 : (NV == 4 ? 7 : 4)) : A.pipe;
        if (pipe && A.H == 1 && A.tile4 == 0 && A.F4 <= TW && A.unit_chunk <= 64) {
            if (pipe == 1) k = A.E ? sddmm_h1_pipe_kernel<NV, 1, 3, true> : sddmm_h1_pipe_kernel<NV, 1, 3, false>;
            else if (pipe == 2) k = A.E ? sddmm_h1_pipe_kernel<NV, 2, 2, true> : sddmm_h1_pipe_kernel<NV, 2, 2, false>;
            else if (pipe == 3) k = A.E ? sddmm_h1_pipe_kernel<NV, 2, 3, true> : sddmm_h1_pipe_kernel<NV, 2, 3, false>;
            // 4..6: unit-prefetching kernel (next unit's indices + Y row staged by cp.async)
            else if (pipe == 4) k = A.E ? sddmm_pf_kernel<NV, 32, false, 3, true> : sddmm_pf_kernel<NV, 32, false, 3, false>;
            else if (pipe == 5) k = A.E ? sddmm_pf_kernel<NV, 32, true, 4, true> : sddmm_pf_kernel<NV, 32, true, 4, false>;
            else if (pipe == 6) k = A.E ? sddmm_pf_kernel<NV, 32, true, 3, true> : sddmm_pf_kernel<NV, 32, true, 3, false>;
            else k = A.E ? sddmm_pf_kernel<NV, 32, false, 2, true, PF2U<NV>> : sddmm_pf_kernel<NV, 32, false, 2, false, PF2U<NV>>;
            if (pipe >= 4) dsmem = pf_smem_bytes(NV, 32);
        }
    }
    if constexpr (G == 32 && NV == 1 && !XB) {   // H == 1, 17..32 float4 per row: unit prefetch
        // auto (-1) = 4: reddit F=128 4.36 -> 4.03 ms, proteins 3.10 -> 2.91 (7: 4.17 / 3.14)
        const int pipe = A.pipe < 0 ? 4 : A.pipe;
        if (A.H == 1 && A.tile4 == 0 && A.F4 <= TW && A.unit_chunk <= 64 && (pipe == 4 || pipe == 7)) {
            if (pipe == 4) k = A.E ? sddmm_pf_kernel<1, 32, false, 3, true> : sddmm_pf_kernel<1, 32, false, 3, false>;
            else k = A.E ? sddmm_pf_kernel<1, 32, false, 2, true, PF2U<1>> : sddmm_pf_kernel<1, 32, false, 2, false, PF2U<1>>;
            dsmem = pf_smem_bytes(1, 32);
        }
    }
    if constexpr (G == 32 && NV >= 2 && !XB) {   // unit-prefetching multi-head kernel (FG_TUNE_SDDMM_PIPE = 4)
        // heads of D = 32 / 64 (D4 = 8 / 16 lanes per head); other head widths run sddmm_kernel.
        // auto (-1): on for H*D <= 384 (reddit H=8 D=32 7.63 -> 7.30 ms, H=4 D=64 8.20 -> 7.36,
        // H=6 D=32 7.82 -> 6.43, H=12 D=32 13.96 -> 13.14, H=6 D=64 14.98 -> 13.25) and for
        // H*D = 512 with D = 64 (H=8: 18.16 -> 16.03); off for H*D = 512 with D = 32 (H=16:
        // 16.30 plain vs 20.12 -- 70 KB of staged results per CTA)
        // with 2 CTAs per SM and twice the edges in flight (pipe 7): H=12 D=32 12.96 -> 12.74,
        // H=8 D=64 16.04 -> 15.28, but H=8 D=32 7.32 -> 7.67: 7 for NV = 3 / 4, 4 for NV = 2
        const bool dflt = NV <= 3 || (NV == 4 && A.D4 == 16);
        const int pipe = A.pipe < 0 ? (dflt ? (NV == 2 ? 4 : 7) : 0) : A.pipe;
        if (pipe == 4 && A.H > 1 && A.F4 <= TW && A.unit_chunk <= 64 && (A.D4 == 8 || A.D4 == 16)) {
            if (A.D4 == 8) k = A.E ? sddmm_pf_kernel<NV, 8, false, 3, true> : sddmm_pf_kernel<NV, 8, false, 3, false>;
            else k = A.E ? sddmm_pf_kernel<NV, 16, false, 3, true> : sddmm_pf_kernel<NV, 16, false, 3, false>;
            dsmem = pf_smem_bytes(NV, A.D4 == 8 ? 8 : 16);
        } else if (pipe == 7 && A.H > 1 && A.F4 <= TW && A.unit_chunk <= 64 && (A.D4 == 8 || A.D4 == 16)) {
            if (A.D4 == 8) k = A.E ? sddmm_pf_kernel<NV, 8, false, 2, true, PF2U<NV>> : sddmm_pf_kernel<NV, 8, false, 2, false, PF2U<NV>>;
            else k = A.E ? sddmm_pf_kernel<NV, 16, false, 2, true, PF2U<NV>> : sddmm_pf_kernel<NV, 16, false, 2, false, PF2U<NV>>;
            dsmem = pf_smem_bytes(NV, A.D4 == 8 ? 8 : 16);
        }
    }
    if (dsmem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
        if (e != cudaSuccess) return fgk::set_error(FG_ECUDA, "sddmm: smem attribute: %s", cudaGetErrorString(e));
    }
    const int64_t per_block = THREADS / G;
    int64_t blocks = (A.n_units + per_block - 1) / per_block;
    if (blocks == 0) return FG_OK;
    if (A.persistent) {   // exactly the resident CTAs: the groups then walk the unit list together
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, dsmem) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        if (A.persistent > 0 && A.persistent < per_sm) per_sm = A.persistent;
        blocks = std::min<int64_t>(blocks, int64_t(fgk::num_sms()) * per_sm);
    }
    k<<<unsigned(blocks), THREADS, dsmem, st>>>(A, X, Y, out);
    return fgk::check_launch("sddmm_kernel");
}

template <int G, int NP, int DWP = G>
fg_status launch_pair(const Args& A, const uint4* X, const uint4* Y, float* out, cudaStream_t st) {
    auto k = sddmm_pair_kernel<G, NP, DWP>;
    const int64_t per_block = THREADS / G;
    int64_t blocks = (A.n_units + per_block - 1) / per_block;
    if (blocks == 0) return FG_OK;
    if (A.persistent) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, 0) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        if (A.persistent > 0 && A.persistent < per_sm) per_sm = A.persistent;
        blocks = std::min<int64_t>(blocks, int64_t(fgk::num_sms()) * per_sm);
    }
    k<<<unsigned(blocks), THREADS, 0, st>>>(A, X, Y, out);
    return fgk::check_launch("sddmm_pair_kernel");
}

}  // namespace

namespace fgk {

__global__ void scale_by_kernel(float* __restrict__ out, const float* __restrict__ E, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
    if (i < n) out[i] *= E[i];
}

static fg_status launch_sddmm_core(const fg_graph* g, int H, int D, const float* X, const float* Y, float* out,
                                   cudaStream_t st, const uint16_t* Xbf16, const uint16_t* Ybf16, const float* E) {
    const bool xb = Xbf16 != nullptr;   // bf16 storage of X and Y (fg_sddmm_x16)
    Args A;
    A.E = E;
    A.unit_row = g->unit_row;
    A.unit_p0 = g->unit_p0;
    A.n_units = g->n_units;
    A.unit_chunk = g->unit_chunk;
    A.unit_p1 = nullptr;
    A.row_ptr = g->row_ptr;
    A.col_idx = g->col_idx;
    A.eid = g->eid;
    A.H = H;
    A.F4 = H * D / 4;
    A.D4 = (H > 1) ? D / 4 : A.F4;
    A.D = D;
    A.c4base = 0;
    A.accumulate = 0;
    A.tile4 = 0;
    A.persistent = 0;
    A.pipe = int(g->tune.sddmm_pipe);
    int F4 = A.F4;
    const float4* X4 = reinterpret_cast<const float4*>(xb ? static_cast<const void*>(Xbf16) : X);
    const float4* Y4 = reinterpret_cast<const float4*>(xb ? static_cast<const void*>(Ybf16) : Y);
    // Feature-dimension tiling for L2 (as in spmm.cu): for H == 1 and
    // X larger than the L2 budget, pass k computes the partial dot over float4
    // columns [k*T4, (k+1)*T4) and accumulates into out (fixed pass order:
    // deterministic).  Each pass gathers from an L2-resident slice of X.
    {
        const int64_t budget = fgk::l2_tile_budget(g);
        // opt-in (FG_TUNE_SDDMM_L2_TILE): measured slower than one pass on reddit F=512
        // (25.8 ms at 64 MB vs 21.3 untiled, even with the running sums prefetched;
        // the narrow-group per-edge reduction, not the traffic, is the limit)
        if (!xb && g->tune.sddmm_l2_tile && H == 1 && budget > 0 && g->n_src * int64_t(F4) * 16 > budget) {
            int t4 = 32;
            while (t4 > 1 && g->n_src * int64_t(t4) * 16 > budget) t4 /= 2;
            A.tile4 = t4;
            for (int c4 = 0; c4 < F4; c4 += t4) {
                A.c4base = c4;
                A.accumulate = c4 > 0;
                fg_status r;
                switch (t4) {
                    case 1: r = launch_t<1, 1>(A, X4, Y4, out, st); break;
                    case 2: r = launch_t<2, 1>(A, X4, Y4, out, st); break;
                    case 4: r = launch_t<4, 1>(A, X4, Y4, out, st); break;
                    case 8: r = launch_t<8, 1>(A, X4, Y4, out, st); break;
                    case 16: r = launch_t<16, 1>(A, X4, Y4, out, st); break;
                    default: r = launch_t<32, 1>(A, X4, Y4, out, st); break;
                }
                if (r != FG_OK) return r;
            }
            return FG_OK;
        }
    }
    // Source-segmented traversal (the paper's 1D graph partitioning by source
    // segments, retargeted from the CPU LLC to the B200 L2): when X does
    // not fit the segment budget, the work units are ordered segment by segment of
    // seg_rows source vertices (each unit = a contiguous run of one row's edges
    // inside one segment, since rows are sorted by source).  SDDMM has no
    // cross-edge reduction, so no merge is needed.  The launch is persistent
    // (resident CTAs only, groups stride through the unit list together), so the
    // concurrently active units stay inside one or two segments and their X
    // slice stays L2-resident.  Measured on reddit u_dot_v F = 512: 19.7 ms -> 16.4
    // ms (DRAM 115 -> 29 GB); non-persistent segmentation was slower (23.8 ms: one
    // CTA launch per 8 short units caps the active warps at 15 %).
    // FG_SDDMM_SEG_MB: segment size (default 48; 0 disables); segmentation only when X
    // exceeds FG_SDDMM_SEG_MIN_MB (default 96).  Swept on reddit / proteins
    // (tools/seg_sweep.py, tools/var_exp.py): X of 60 MB (F = 64) runs 3.00 ms
    // unsegmented vs 3.61 ms in 48 MB segments, 119 MB (F = 128) ties, and the
    // 238 / 477 MB cases (H = 8 D = 32, H = 1 F = 512) prefer 48 MB segments over
    // 96 MB ones (9.39 vs 9.79 ms, 16.46 vs 16.72 ms).
    // The tables are built by fg_graph_prepare(g, row_bytes) (synchronous, per
    // topology); a width that was not prepared runs the unsegmented traversal --
    // this launch path never allocates or synchronises.
    if (A.tile4 == 0) {
        const int64_t seg_rows = fgk::sddmm_seg_rows(g, int64_t(F4) * (xb ? 8 : 16));
        const int64_t rb_rows = fgk::sddmm_rb_rows(g, int64_t(F4) * (xb ? 8 : 16));
        const fg_graph::SegUnits* su = seg_rows ? fgk::find_seg_units(g, seg_rows, rb_rows) : nullptr;
        if (su) {
            A.unit_row = su->row;
            A.unit_p0 = su->p0;
            A.unit_p1 = su->p1;
            A.n_units = su->n_units;
            A.persistent = int(g->tune.sddmm_persist);   // CTAs per SM (-1: the occupancy)
        }
    }
    // multi-head shapes outside the lane-partitioned kernels (D not 4 * 2^k, or
    // H*D > 512): the generic thread-per-edge kernel, any D (fp32 storage)
    if (!xb && H > 1 && (D % 4 != 0 || ((D / 4) & (D / 4 - 1)) != 0 || F4 > 128)) {
        const int64_t per_block = THREADS / 32;
        int64_t blocks = (A.n_units + per_block - 1) / per_block;
        if (A.persistent) blocks = std::min<int64_t>(blocks, int64_t(fgk::num_sms()) * 8);
        if (blocks == 0) return FG_OK;
        sddmm_heads_generic_kernel<<<unsigned(blocks), THREADS, 0, st>>>(A, X4, Y4, out);
        return fgk::check_launch("sddmm_heads_generic_kernel");
    }
    if (g->tune.sddmm_dot == 1 && !xb && A.tile4 == 0) {   // ablation E6: thread-per-edge dot products
        const int64_t per_block = THREADS / 32;
        int64_t blocks = (A.n_units + per_block - 1) / per_block;
        if (A.persistent) blocks = std::min<int64_t>(blocks, int64_t(fgk::num_sms()) * 8);
        if (blocks == 0) return FG_OK;
        sddmm_thread_kernel<<<unsigned(blocks), THREADS, 0, st>>>(A, X4, Y4, out);
        return fgk::check_launch("sddmm_thread_kernel");
    }
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
    if (H > 1 && F4 > G * NV)
        return set_error(FG_EUNSUPPORTED, "fg_sddmm: multi-head with H*D > 512 not implemented");
    // bf16 storage, 16-byte aligned X / Y, whole 8-feature pairs: 16-byte loads of
    // pairs (sddmm_pair_kernel; G lanes x NP pairs).  H == 1: any even F4 <= 256;
    // H > 1: D = 8 * 2^k with D/8 <= 32 lanes per head, H*D <= 512 and the batch's
    // H results per edge fitting the group's staging buffer (H * 32 <= 32 * G).
    if (xb && ((reinterpret_cast<uintptr_t>(Xbf16) | reinterpret_cast<uintptr_t>(Ybf16)) & 15u) == 0) {
        const uint4* Xp = reinterpret_cast<const uint4*>(Xbf16);
        const uint4* Yp = reinterpret_cast<const uint4*>(Ybf16);
        const int P8 = F4 / 2;
        if (H == 1 && F4 % 2 == 0 && F4 <= 256) {
            if (P8 <= 32) {
                int G2 = 1;
                while (G2 < P8) G2 *= 2;
                switch (G2) {
                    case 1: return launch_pair<1, 1>(A, Xp, Yp, out, st);
                    case 2: return launch_pair<2, 1>(A, Xp, Yp, out, st);
                    case 4: return launch_pair<4, 1>(A, Xp, Yp, out, st);
                    case 8: return launch_pair<8, 1>(A, Xp, Yp, out, st);
                    case 16: return launch_pair<16, 1>(A, Xp, Yp, out, st);
                    default: return launch_pair<32, 1>(A, Xp, Yp, out, st);
                }
            }
            if (P8 <= 64) return launch_pair<32, 2>(A, Xp, Yp, out, st);
            if (P8 <= 96) return launch_pair<32, 3>(A, Xp, Yp, out, st);
            return launch_pair<32, 4>(A, Xp, Yp, out, st);
        }
        const int DP = D / 8;   // pairs (= lanes) per head
        if (H > 1 && D % 8 == 0 && (DP & (DP - 1)) == 0 && DP <= 32 && F4 <= 128) {
            // G = 32 lanes x NP pairs covers P8 <= 32 * NP; heads need H * 32 <= 32 * 32
            const int NP = P8 <= 32 ? 1 : 2;
            if (H <= 32) {
                switch (DP) {
                    case 1: return NP == 1 ? launch_pair<32, 1, 1>(A, Xp, Yp, out, st) : launch_pair<32, 2, 1>(A, Xp, Yp, out, st);
                    case 2: return NP == 1 ? launch_pair<32, 1, 2>(A, Xp, Yp, out, st) : launch_pair<32, 2, 2>(A, Xp, Yp, out, st);
                    case 4: return NP == 1 ? launch_pair<32, 1, 4>(A, Xp, Yp, out, st) : launch_pair<32, 2, 4>(A, Xp, Yp, out, st);
                    case 8: return NP == 1 ? launch_pair<32, 1, 8>(A, Xp, Yp, out, st) : launch_pair<32, 2, 8>(A, Xp, Yp, out, st);
                    case 16: return NP == 1 ? launch_pair<32, 1, 16>(A, Xp, Yp, out, st) : launch_pair<32, 2, 16>(A, Xp, Yp, out, st);
                    default: break;   // DP == 32: one head per 32 lanes = the H1 reduction per head; use the chunk path
                }
            }
        }
    }
    if (xb) {
        switch (G) {
            case 1: return launch_t<1, 1, true>(A, X4, Y4, out, st);
            case 2: return launch_t<2, 1, true>(A, X4, Y4, out, st);
            case 4: return launch_t<4, 1, true>(A, X4, Y4, out, st);
            case 8: return launch_t<8, 1, true>(A, X4, Y4, out, st);
            case 16: return launch_t<16, 1, true>(A, X4, Y4, out, st);
            default:
                if (NV == 1) return launch_t<32, 1, true>(A, X4, Y4, out, st);
                if (NV == 2) return launch_t<32, 2, true>(A, X4, Y4, out, st);
                if (NV == 3) return launch_t<32, 3, true>(A, X4, Y4, out, st);
                return launch_t<32, 4, true>(A, X4, Y4, out, st);
        }
    }
    switch (G) {
        case 1: return launch_t<1, 1>(A, X4, Y4, out, st);
        case 2: return launch_t<2, 1>(A, X4, Y4, out, st);
        case 4: return launch_t<4, 1>(A, X4, Y4, out, st);
        case 8: return launch_t<8, 1>(A, X4, Y4, out, st);
        case 16: return launch_t<16, 1>(A, X4, Y4, out, st);
        default:
            if (NV == 1) return launch_t<32, 1>(A, X4, Y4, out, st);
            if (NV == 2) return launch_t<32, 2>(A, X4, Y4, out, st);
            if (NV == 3) return launch_t<32, 3>(A, X4, Y4, out, st);
            return launch_t<32, 4>(A, X4, Y4, out, st);
    }
}

// u_dot_v, optionally followed by e_mul (E != NULL: out[e][h] = score * E[e][h]).
// The scale is fused into the kernels' staged result write-back; configurations
// that write results directly (more heads than a group stages: H > G, or the
// opt-in column-tiled pass) scale in a second, elementwise pass instead.
fg_status launch_sddmm(const fg_graph* g, int H, int D, const float* X, const float* Y, float* out,
                       cudaStream_t st, const uint16_t* Xbf16, const uint16_t* Ybf16, const float* E) {
    if (E) {
        const int F4 = H * D / 4;
        int G = 32;
        if (F4 <= 32) {
            G = 1;
            while (G < F4) G *= 2;
        }
        const int B = G >= 4 ? 32 : 8;
        const bool tiled = !Xbf16 && g->tune.sddmm_l2_tile && H == 1;
        if (H * B > 32 * G || tiled) {   // (the bf16 pair kernels stage whenever this holds)
            fg_status s = launch_sddmm_core(g, H, D, X, Y, out, st, Xbf16, Ybf16, nullptr);
            if (s != FG_OK) return s;
            const int64_t n = g->nnz * H;
            scale_by_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(out, E, n);
            return check_launch("scale_by_kernel");
        }
    }
    return launch_sddmm_core(g, H, D, X, Y, out, st, Xbf16, Ybf16, E);
}

}  // namespace fgk
