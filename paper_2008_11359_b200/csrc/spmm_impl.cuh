// spmm_impl.cuh -- the gathered-message gSpMM kernel template (design notes in
// spmm.cu), instantiated per (reducer, op set) by spmm_inst_*.cu.
#pragma once
#include <algorithm>
#include <type_traits>

#ifndef FG_SPMM_FULLB
#define FG_SPMM_FULLB 0   // full-batch fast path: 0 select reducers only (default), 1 all, 2 none
#endif
#ifndef FG_SPMM_IDXPF
// next-batch index prefetch in the gather loop (development variant, -DFG_SPMM_IDXPF=1):
// measured slower on reddit -- copy_u-sum F=512 12.1 -> 12.9 ms (the two extra index
// registers per lane spill at the 64-register cap), u_mul_e H=8 7.6 -> 7.8, copy_u-max
// F=128 unchanged (48 -> 64 registers); the product loads a batch's indices at its start
#define FG_SPMM_IDXPF 0
#endif

#include "device_common.cuh"
#include "fg_internal.h"

namespace fgspmm {
using fgdev::bf16x4;
using fgdev::group_mask;


// OP_UMULE_GEN: u_mul_e with D % 4 != 0 (the head varies inside a float4);
// OP_UADDE: u_add_e (per-component head lookup, any D); OP_COPYE: copy_e (the
// message row is E[eid] itself, E is [nnz][F]).
enum { OP_COPY = 0, OP_UMULE = 1, OP_UMULE_GEN = 2, OP_UADDE = 3, OP_COPYE = 4 };
enum { R_SUM = 0, R_MAX = 1, R_MIN = 2, R_MEAN = 3 };
constexpr int THREADS = 256;

struct Args {
    const int32_t* rows;        // rows_by_deg
    int64_t n_heavy;            // rows[0, n_heavy) -> CTA-per-row mode
    int64_t n_rows;             // n_dst
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* eid;
    const float4* X;
    const uint2* Xh;            // bf16 storage of X (fg_spmm_x16): 4 features per 8-byte chunk
    const float* E;
    int H, D, F4;
    float4* out;
    int4* arg_u;
    int4* arg_e;
    // hybrid partitioning (HYB kernels only): per-edge source codes (u, or
    // -(slot+1) for a source staged in shared memory) and the staged sources
    const int32_t* hyb_code;
    const int32_t* hyb_hot;
    int hyb_k;
    int64_t n_vblocks;          // virtual blocks of the launch (HYB: persistent grid-stride)
    // source-segmented pass (SEG kernels only; u_mul_e / copy_u sum): row v's edges
    // with sources in this pass's segment are [seg_lo[v], seg_hi[v]); seg_acc != 0:
    // the pass adds onto out (passes run in segment order, so a group-per-row sum
    // keeps the CSR order of the unsegmented kernel)
    const int64_t* seg_lo;
    const int64_t* seg_hi;
    int seg_acc;
};

__device__ __forceinline__ float4 f4(float a) { return make_float4(a, a, a, a); }
// 32 bytes (two adjacent float4) with one 256-bit load (sm_100: LDG.E.256)
__device__ __forceinline__ void ldg256(const char* p, float4& a, float4& b) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p));
}
__device__ __forceinline__ float comp(const float4& v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
__device__ __forceinline__ void set_comp(float4& v, int k, float a) {
    if (k == 0) v.x = a; else if (k == 1) v.y = a; else if (k == 2) v.z = a; else v.w = a;
}

// Column (float4 index within the tile) of a lane's chunk j.  PAIR (NV even): a
// lane owns pairs of adjacent chunks, read with ONE load -- 16 bytes for bf16
// storage (8 features), 32 bytes (LDG.256, ld.global.nc.v8.f32) for fp32;
// otherwise chunk j of lane gl is column gl + G*j.
template <int G, bool PAIR>
__device__ __forceinline__ int colj(int gl, int j) {
    if constexpr (PAIR) return 2 * (gl + G * (j >> 1)) + (j & 1);
    else return gl + G * j;
}

// u_mul_e stages each 32-edge batch's E rows in shared memory (NG x 512 floats)
// when a whole warp owns the row (G == 32)
template <int G, int OP, int RED>
constexpr bool stage_e() {
    return OP == OP_UMULE && G == 32;
}

// Accumulate edges [s, e) of one row into (acc, pos) for this lane's NV chunks.
template <int G, int NV, int OP, int RED, bool XB, bool PAIR, bool HYB = false>
__device__ __forceinline__ void gather_range(const Args& A, int64_t s, int64_t e, int gl, unsigned mask,
                                             int c4base, float4 (&acc)[NV], int (&pos)[NV][4],
                                             float* __restrict__ etile, const float4* __restrict__ hot = nullptr) {
    constexpr int B = 32;                                   // edges per index batch
    constexpr int R = B / G;                                // indices per lane per batch
    // edges in flight per lane; PAIR (raw bf16 pairs): 4 -- 8 measured slower
    // (reddit bf16 copy_u-sum F=512 9.37 vs 8.49 ms, u_mul_e H=8 10.1 vs 7.5 ms);
    // one chunk per lane: 8 for sum, 4 for the select reducers (reddit copy_u-max
    // F=128 + args 4.84 -> 4.63 ms; sum F=512 unchanged)
    // fp32 pairs (32-byte loads): the same bytes in flight per lane as the 16-byte
    // mapping with twice the chunks, i.e. U of the NV / 2 = 1 / 2 pair cases 4 / 2
    constexpr int U = PAIR ? ((XB || NV < 4) ? 4 : 2)
                           : (NV >= 4 ? 2 : (NV >= 2 ? 4 : ((RED == R_MAX || RED == R_MIN) ? 4 : 8)));
    constexpr bool P16 = PAIR && XB;                         // bf16 pairs: raw 16-byte words
    constexpr bool MAX = (RED == R_MAX || RED == R_MIN);     // select-type reducers
    const int F4 = A.F4;
    constexpr int CB = XB ? 8 : 16;                          // bytes of X per 4-feature chunk
    const char* xl = (OP == OP_COPYE) ? reinterpret_cast<const char*>(A.E)
                                      : XB ? reinterpret_cast<const char*>(A.Xh)
                                                     : reinterpret_cast<const char*>(A.X);
    xl += int64_t(c4base + colj<G, PAIR>(gl, 0)) * CB;       // this lane's first column
    const uint32_t rowb = uint32_t(F4) * CB;                 // bytes per source row
    bool cin[NV];                                            // chunk j inside the row (edge-invariant)
#pragma unroll
    for (int j = 0; j < NV; ++j) cin[j] = c4base + colj<G, PAIR>(gl, j) < F4;
    // the batch's neighbour indices (and edge ids), one per lane and R per lane
    auto load_idx = [&](int64_t q0, int (&ui)[R], int (&ei)[R]) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t p = q0 + gl + r * G;
            if constexpr (HYB) ui[r] = (p < e) ? __ldg(A.hyb_code + p) : 0;   // u, or -(slot+1): staged
            else ui[r] = (OP != OP_COPYE && p < e) ? __ldg(A.col_idx + p) : 0;   // copy_e reads no source row
            if constexpr (OP != OP_COPY) ei[r] = (p < e) ? (A.eid ? __ldg(A.eid + p) : int(p)) : 0;
        }
    };
    // FG_SPMM_IDXPF: the next batch's indices are loaded while this batch gathers, so
    // a batch's first X gathers do not wait an index round trip
    int uixn[R], eixn[R];
    if constexpr (FG_SPMM_IDXPF) {
        if (s < e) load_idx(s, uixn, eixn);
    }
    for (int64_t p0 = s; p0 < e; p0 += B) {
        const int cnt = int(min((int64_t)B, e - p0));
        int uix[R];
        int eix[R];
        if constexpr (FG_SPMM_IDXPF) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                uix[r] = uixn[r];
                eix[r] = eixn[r];
            }
            if (p0 + B < e) load_idx(p0 + B, uixn, eixn);
        } else {
            load_idx(p0, uix, eix);
        }
        // u_mul_e with identity edge ids: the batch's E rows are one contiguous span;
        // stage it in shared memory with coalesced loads instead of one dependent
        // scalar load per edge and chunk
        bool staged = false;
        if constexpr (stage_e<G, OP, RED>()) {
            if (A.eid == nullptr && A.H <= 16) {
                staged = true;
                __syncwarp(mask);
                const float* Eb = A.E + p0 * A.H;
                for (int q = gl; q < cnt * A.H; q += G) etile[q] = __ldg(Eb + q);
                __syncwarp(mask);
            }
        }
        // one step of U edges (t0 a compile-time constant after unrolling); FULL (all
        // U edges inside the batch) drops the per-edge bounds predicates.
        // Source rows are addressed from this lane's column base with one
        // 32x32 -> 64-bit multiply-add per edge (IMAD.WIDE.U32) and immediate
        // chunk offsets.
        auto step = [&](int t0, auto full_c) {
            constexpr bool FULL = decltype(full_c)::value;
            float4 x[P16 ? 1 : U][P16 ? 1 : NV];
            uint4 xw[P16 ? U : 1][P16 ? NV / 2 : 1];     // bf16 pairs: raw words, converted at use
            constexpr bool PERK = (OP == OP_UMULE_GEN || OP == OP_UADDE);   // head per component
            float ev[U][NV][PERK ? 4 : 1];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int t = t0 + uu;
                const int u = __shfl_sync(mask, uix[t / G], t % G, G);
                int ed = 0;
                if constexpr (OP != OP_COPY) ed = __shfl_sync(mask, eix[t / G], t % G, G);
                // u_mul_e keeps the element-indexed form: with the lane-base form the
                // compiler re-loads kernel parameters per edge (reddit H=8: 7.8 -> 8.3 ms)
                const int64_t ce = int64_t(u) * F4 + c4base + colj<G, PAIR>(gl, 0);   // element-indexed chunk
                const char* xr = (OP == OP_UMULE || OP == OP_UMULE_GEN)
                                     ? (XB ? reinterpret_cast<const char*>(A.Xh + ce)
                                                     : reinterpret_cast<const char*>(A.X + ce))
                                     : xl + uint64_t(uint32_t(OP == OP_COPYE ? ed : u)) * rowb;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int c = c4base + colj<G, PAIR>(gl, j);
                    const bool ok = (FULL || t < cnt) && cin[j];
                    if constexpr (P16) {   // F4 even: c even, c + 1 < F4 with c
                        if ((j & 1) == 0)
                            xw[uu][j / 2] = ok ? __ldg(reinterpret_cast<const uint4*>(xr + (2 * G * (j >> 1)) * CB))
                                               : make_uint4(0, 0, 0, 0);
                    } else if constexpr (PAIR) {   // fp32 pair: one 32-byte load (32-byte aligned, checked by the host)
                        if ((j & 1) == 0) {
                            if (ok) {
                                ldg256(xr + (2 * G * (j >> 1)) * CB, x[uu][j], x[uu][j + 1]);
                            } else {
                                x[uu][j] = f4(0.f);
                                x[uu][j + 1] = f4(0.f);
                            }
                        }
                    } else if constexpr (XB) {
                        x[uu][j] = ok ? bf16x4(__ldg(reinterpret_cast<const uint2*>(xr + j * G * CB))) : f4(0.f);
                    } else if constexpr (HYB) {   // hot sources from shared memory, the rest from L2 / HBM
                        x[uu][j] = !ok ? f4(0.f) : (u < 0 ? hot[int64_t(-1 - u) * F4 + c] : __ldg(A.X + int64_t(u) * F4 + c));
                    } else {
                        x[uu][j] = ok ? __ldg(reinterpret_cast<const float4*>(xr + j * G * CB)) : f4(0.f);
                    }
                    if constexpr (OP == OP_UMULE) {
                        const int h = (4 * c) / A.D;
                        ev[uu][j][0] = !ok ? 0.f : (staged ? etile[t * A.H + h] : __ldg(A.E + int64_t(ed) * A.H + h));
                    } else if constexpr (PERK) {
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
                if (!FULL && t >= cnt) break;
                const int p = int(p0) + t;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    float4 xv;
                    if constexpr (P16) {
                        const uint4 w = xw[uu][j / 2];
                        xv = (j & 1) ? bf16x4(make_uint2(w.z, w.w)) : bf16x4(make_uint2(w.x, w.y));
                    } else {
                        xv = x[uu][j];
                    }
                    if constexpr (!MAX) {
                        if constexpr (OP == OP_COPY) {
                            acc[j].x += xv.x; acc[j].y += xv.y;
                            acc[j].z += xv.z; acc[j].w += xv.w;
                        } else if constexpr (OP == OP_UMULE) {
                            const float w = ev[uu][j][0];
                            acc[j].x = fmaf(xv.x, w, acc[j].x); acc[j].y = fmaf(xv.y, w, acc[j].y);
                            acc[j].z = fmaf(xv.z, w, acc[j].z); acc[j].w = fmaf(xv.w, w, acc[j].w);
                        } else if constexpr (OP == OP_UADDE) {
                            acc[j].x += __fadd_rn(xv.x, ev[uu][j][0]);
                            acc[j].y += __fadd_rn(xv.y, ev[uu][j][1]);
                            acc[j].z += __fadd_rn(xv.z, ev[uu][j][2]);
                            acc[j].w += __fadd_rn(xv.w, ev[uu][j][3]);
                        } else if constexpr (OP == OP_COPYE) {
                            acc[j].x += xv.x; acc[j].y += xv.y;
                            acc[j].z += xv.z; acc[j].w += xv.w;
                        } else {
                            acc[j].x = fmaf(xv.x, ev[uu][j][0], acc[j].x);
                            acc[j].y = fmaf(xv.y, ev[uu][j][1], acc[j].y);
                            acc[j].z = fmaf(xv.z, ev[uu][j][2], acc[j].z);
                            acc[j].w = fmaf(xv.w, ev[uu][j][3], acc[j].w);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            float m = comp(xv, k);
                            if constexpr (OP == OP_UMULE) m = __fmul_rn(m, ev[uu][j][0]);
                            else if constexpr (OP == OP_UMULE_GEN) m = __fmul_rn(m, ev[uu][j][k]);
                            else if constexpr (OP == OP_UADDE) m = __fadd_rn(m, ev[uu][j][k]);
                            const bool better = (RED == R_MIN) ? (m < comp(acc[j], k)) : (m > comp(acc[j], k));
                            if (better) { set_comp(acc[j], k, m); pos[j][k] = p; }   // strict: first wins
                        }
                    }
                }
            }
        };
        // full 32-edge batches of the select reducers take a predicate-free unrolled
        // copy of the loop (reddit copy_u-max F=128 + args 4.28 -> 3.65 ms); for the
        // sums the larger code measured equal (copy_u) or slower (u_mul_e 8.2 -> 10.7 ms)
        if (FG_SPMM_FULLB == 1 || (FG_SPMM_FULLB == 0 && MAX)) {
          if (cnt == B) {
#pragma unroll
            for (int t0 = 0; t0 < B; t0 += U) step(t0, std::true_type{});
            continue;
          }
        }
#pragma unroll
        for (int t0 = 0; t0 < B; t0 += U) {
            if (t0 >= cnt) break;                           // uniform within the group
            step(t0, std::false_type{});
        }
    }
}

template <int NV, int RED>
__device__ __forceinline__ void init_acc(float4 (&acc)[NV], int (&pos)[NV][4]) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        acc[j] = f4(RED == R_MAX ? -INFINITY : (RED == R_MIN ? INFINITY : 0.f));
#pragma unroll
        for (int k = 0; k < 4; ++k) pos[j][k] = -1;
    }
}

template <int RED>
__device__ __forceinline__ void store_elem(const Args& A, int64_t v, int c, float4 a, const int (&ps)[4], int64_t deg) {
    const int64_t o = v * A.F4 + c;
    const bool empty = deg == 0;
    if (RED == R_SUM) {
        A.out[o] = a;
        return;
    }
    if (RED == R_MEAN) {   // sum / in-degree (IEEE division); empty rows -> 0
        const float d = float(deg);
        A.out[o] = empty ? f4(0.f) : make_float4(a.x / d, a.y / d, a.z / d, a.w / d);
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

// One virtual block of the gather launch: CTA-per-row (vb < n_heavy) or a group
// of rows per CTA.  The shared buffers belong to the calling kernel.
template <int G, int NV, int OP, int RED, bool XB, bool PAIR, bool HYB, bool SEG, typename SAcc, typename SEt,
          typename SVal, typename SPos>
__device__ __forceinline__ void spmm_vblock(const Args& A, int64_t vb, int gl, int gi, unsigned mask, int c4base,
                                            SAcc& s_acc, SEt& s_etile, SVal& s_val, SPos& s_pos,
                                            const float4* __restrict__ s_hot) {
    constexpr bool MAX = (RED == R_MAX || RED == R_MIN);
    constexpr int NG = THREADS / G;                 // groups per CTA
    constexpr int TW = G * NV;                      // float4 columns per tile
    float4 acc[NV];
    int pos[NV][4];
    init_acc<NV, RED>(acc, pos);

    if (vb < A.n_heavy) {
        // ---- CTA-per-row: contiguous edge ranges per group, fixed-order combine
        const int64_t v = A.rows[vb];
        const int64_t s = SEG ? A.seg_lo[v] : A.row_ptr[v], e = SEG ? A.seg_hi[v] : A.row_ptr[v + 1];
        if (SEG && A.seg_acc && s == e) return;   // nothing to add (uniform across the CTA)
        const int64_t len = (e - s + NG - 1) / NG;
        const int64_t gs = min(e, s + gi * len), ge = min(e, gs + len);
        gather_range<G, NV, OP, RED, XB, PAIR, HYB>(A, gs, ge, gl, mask, c4base, acc, pos, s_etile[gi], s_hot);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int c = colj<G, PAIR>(gl, j);
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
                if (SEG && A.seg_acc) {   // earlier segments' sum + this pass's partials, fixed order
                    const float4 b = a;
                    a = A.out[v * A.F4 + c4base + c];
                    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
                }
                for (int g2 = 1; g2 < NG; ++g2) {
                    const float4 b = s_acc[g2][c];
                    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
                }
            } else {
                a = f4(RED == R_MIN ? INFINITY : -INFINITY);
                for (int g2 = 0; g2 < NG; ++g2) {   // ascending ranges: strict compare keeps the lowest position
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float b = s_val[g2][4 * c + k];
                        const bool better = (RED == R_MIN) ? (b < comp(a, k)) : (b > comp(a, k));
                        if (better) { set_comp(a, k, b); ps[k] = s_pos[g2][4 * c + k]; }
                    }
                }
            }
            store_elem<RED>(A, v, c4base + c, a, ps, e - s);
        }
        if constexpr (HYB) __syncthreads();   // the combine buffers are reused by this CTA's next virtual block
        return;
    }

    // ---- group-per-row
    const int64_t r = A.n_heavy + (vb - A.n_heavy) * NG + gi;
    if (r >= A.n_rows) return;
    const int64_t v = A.rows[r];
    const int64_t s = SEG ? A.seg_lo[v] : A.row_ptr[v], e = SEG ? A.seg_hi[v] : A.row_ptr[v + 1];
    if constexpr (SEG) {
        if (A.seg_acc) {
            if (s == e) return;
#pragma unroll
            for (int j = 0; j < NV; ++j) {   // continue the running sum of the earlier segments
                const int c = c4base + colj<G, PAIR>(gl, j);
                if (c < A.F4) acc[j] = A.out[v * A.F4 + c];
            }
        }
    }
    gather_range<G, NV, OP, RED, XB, PAIR, HYB>(A, s, e, gl, mask, c4base, acc, pos, s_etile[gi], s_hot);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = c4base + colj<G, PAIR>(gl, j);
        if (c < A.F4) store_elem<RED>(A, v, c, acc[j], pos[j], e - s);
    }
}

// HYB: the paper's hybrid partitioning on the GPU: the hyb_k sources
// of highest out-degree are staged in shared memory once per CTA (persistent
// grid-stride over the virtual blocks) and read from there; the others from
// L2 / HBM.  Same values in the same order as the plain kernel: bit-identical.
template <int G, int NV, int OP, int RED, bool XB, bool PAIR, bool HYB = false, bool SEG = false>
__global__ void __launch_bounds__(THREADS) spmm_gather_kernel(Args A) {
    constexpr bool MAX = (RED == R_MAX || RED == R_MIN);
    constexpr int NG = THREADS / G;                 // groups per CTA
    constexpr int TW = G * NV;                      // float4 columns per tile
    __shared__ float4 s_acc[MAX ? 1 : NG][MAX ? 1 : TW];
    __shared__ float s_etile[stage_e<G, OP, RED>() ? NG : 1][stage_e<G, OP, RED>() ? 32 * 16 : 1];
    __shared__ float s_val[MAX ? NG : 1][MAX ? TW * 4 : 1];
    __shared__ int s_pos[MAX ? NG : 1][MAX ? TW * 4 : 1];

    extern __shared__ float4 s_hot[];   // HYB: hyb_k staged source rows of F4 float4
    const int lane = threadIdx.x & 31;
    const int gl = threadIdx.x & (G - 1);
    const int gi = threadIdx.x / G;
    const unsigned mask = group_mask<G>(lane);
    const int c4base = blockIdx.y * TW;
    if constexpr (HYB) {
        for (int i = threadIdx.x; i < A.hyb_k * A.F4; i += THREADS) {
            const int k = i / A.F4, c = i - k * A.F4;
            s_hot[i] = __ldg(A.X + int64_t(__ldg(A.hyb_hot + k)) * A.F4 + c);
        }
        __syncthreads();
    }

    if constexpr (HYB) {
        for (int64_t vb = blockIdx.x; vb < A.n_vblocks; vb += gridDim.x)
            spmm_vblock<G, NV, OP, RED, XB, PAIR, HYB, SEG>(A, vb, gl, gi, mask, c4base, s_acc, s_etile, s_val, s_pos,
                                                            s_hot);
    } else {   // one virtual block per CTA: the plain launch (no loop, no extra registers)
        spmm_vblock<G, NV, OP, RED, XB, PAIR, HYB, SEG>(A, blockIdx.x, gl, gi, mask, c4base, s_acc, s_etile, s_val,
                                                        s_pos, s_hot);
    }
}

template <int G, int NV, int OP, int RED, bool XB = false, bool PAIR = false, bool HYB = false, bool SEG = false>
fg_status launch_t(const Args& A0, cudaStream_t st) {
    Args A = A0;
    constexpr int NG = THREADS / G;
    constexpr int TW = G * NV;
    const int64_t light = A.n_rows - A.n_heavy;
    const int64_t blocks = A.n_heavy + (light + NG - 1) / NG;
    const int tiles = (A.F4 + TW - 1) / TW;
    if (blocks == 0) return FG_OK;
    A.n_vblocks = blocks;
    int64_t grid_x = blocks;
    size_t smem = 0;
    auto k = spmm_gather_kernel<G, NV, OP, RED, XB, PAIR, HYB, SEG>;
    if constexpr (HYB) {   // persistent: the resident CTAs stage the hot rows once each
        smem = size_t(A.hyb_k) * A.F4 * 16;   // (plus the kernel's static combine buffers)
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
            return fgk::set_error(FG_ECUDA, "spmm hybrid: %zu bytes of shared memory", smem);
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        grid_x = std::min<int64_t>(blocks, int64_t(fgk::num_sms()) * per_sm);
    }
    const dim3 grid{unsigned(grid_x), unsigned(tiles), 1u};
    k<<<grid, THREADS, smem, st>>>(A);
    return fgk::check_launch("spmm_gather_kernel");
}

// hybrid partitioning (copy_u-sum, one float4 per lane, untiled): spmm_inst_sum_base.cu
fg_status launch_hybrid(const Args& A, int G, cudaStream_t st);
// one source-segmented pass of u_mul_e-sum (A.seg_lo / seg_hi / seg_acc set): spmm_inst_sum_base.cu
fg_status launch_seg_pass(const Args& A, int G, int NV, cudaStream_t st);

// One explicit specialisation per (reducer, op set) -- op set 0 = copy_u /
// u_mul_e, 1 = u_add_e / copy_e -- each compiled in its own translation unit
// (spmm_inst_*.cu via spmm_inst.cuh) so the instantiations build in parallel.
template <int RED, int OPSET>
fg_status dispatch_inst(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_SUM, 0>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_SUM, 1>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_MAX, 0>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_MAX, 1>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_MIN, 0>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_MIN, 1>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_MEAN, 0>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_inst<R_MEAN, 1>(const Args& A, int G, int NV, int op, cudaStream_t st);
// fp32 X read as 32-byte chunk pairs (copy_u; every reducer): spmm_inst_*_base.cu
template <int RED>
fg_status dispatch_pair32(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_pair32<R_SUM>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_pair32<R_MAX>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_pair32<R_MIN>(const Args& A, int G, int NV, int op, cudaStream_t st);
template <>
fg_status dispatch_pair32<R_MEAN>(const Args& A, int G, int NV, int op, cudaStream_t st);
// bf16 storage of X (copy_u, u_mul_e; sum and max): spmm_inst_x16.cu
// pair: 16-byte loads of adjacent chunk pairs (F4 even; NV even)
template <int RED>
fg_status dispatch_x16(const Args& A, int G, int NV, int op, bool pair, cudaStream_t st);
template <>
fg_status dispatch_x16<R_SUM>(const Args& A, int G, int NV, int op, bool pair, cudaStream_t st);
template <>
fg_status dispatch_x16<R_MAX>(const Args& A, int G, int NV, int op, bool pair, cudaStream_t st);
template <>
fg_status dispatch_x16<R_MIN>(const Args& A, int G, int NV, int op, bool pair, cudaStream_t st);
template <>
fg_status dispatch_x16<R_MEAN>(const Args& A, int G, int NV, int op, bool pair, cudaStream_t st);

}  // namespace fgspmm
