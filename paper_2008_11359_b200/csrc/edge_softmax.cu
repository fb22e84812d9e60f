// edge_softmax.cu -- per-destination, per-head softmax over in-edges (SURVEY
// §8(a) row a5).  Not in the paper: the GAT layer it evaluates uses
// dot-product attention whose scores are normalised over the
// in-edges of each destination (standard GAT / DGL edge_softmax):
//     alpha[e][h] = exp(s[e][h] - m_v,h) / sum_{e' in row v} exp(s[e'][h] - m_v,h)
//
// HBM-bound streaming kernel: one warp per destination row (degree-descending
// order).  When H divides 32 and edge ids are the identity, a row's scores are
// the contiguous span s[row_ptr[v]*H .. row_ptr[v+1]*H) and lane l always sees
// head l % H: pass 1 keeps an online (max, sum) per lane and merges lanes of
// equal head with a butterfly; pass 2 re-reads (L2-resident for all but the
// longest rows) and writes alpha.  Algorithmic bytes: 2*m*H*4 (+ the re-read).
// expf / IEEE division, no fast-math.
#include "fg_internal.h"

namespace {

constexpr int THREADS = 256;

__device__ __forceinline__ void merge(float& m, float& s, float m2, float s2) {
    const float mn = fmaxf(m, m2);
    if (mn == -INFINITY) return;
    s = s * expf(m - mn) + s2 * expf(m2 - mn);
    m = mn;
}

__device__ __forceinline__ void online(float& m, float& s, float x) {
    if (x > m) {
        s = s * expf(m - x) + 1.f;
        m = x;
    } else {
        s += expf(x - m);
    }
}

// H % 4 == 0, (H/4) | 32, identity edge ids: the row's scores are the
// contiguous, 16-byte aligned span S[s0*H, s1*H); lane l reads float4 i = l +
// 32k, whose 4 heads are 4*(l % (H/4)) .. +3 for every k.  4 float4 loads in
// flight per lane; lanes with equal l % (H/4) merge with a butterfly.
__global__ void __launch_bounds__(THREADS) softmax_vec_kernel(const int32_t* __restrict__ rows, int64_t n_rows,
                                                              const int64_t* __restrict__ rp, int H,
                                                              const float* S, float* out) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    if (r >= n_rows) return;
    const int64_t v = rows[r];
    const int64_t s0 = rp[v], s1 = rp[v + 1];
    const int64_t n4 = (s1 - s0) * H / 4;
    const float4* S4 = reinterpret_cast<const float4*>(S + s0 * H);
    float4* O4 = reinterpret_cast<float4*>(out + s0 * H);
    float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, sm[4] = {0.f, 0.f, 0.f, 0.f};
    constexpr int UN = 4;
    for (int64_t i0 = lane; i0 < n4; i0 += 32 * UN) {
        float4 x[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const int64_t i = i0 + 32 * k;
            x[k] = (i < n4) ? S4[i] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            if (i0 + 32 * k < n4) {
                online(m[0], sm[0], x[k].x); online(m[1], sm[1], x[k].y);
                online(m[2], sm[2], x[k].z); online(m[3], sm[3], x[k].w);
            }
        }
    }
    const int hq = H / 4;
    for (int o = 16; o >= hq; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m[c], o);
            const float s2 = __shfl_xor_sync(0xffffffffu, sm[c], o);
            merge(m[c], sm[c], m2, s2);
        }
    }
    // alpha = e * (1 / S): one correctly rounded reciprocal per (row, head) and a
    // correctly rounded multiply per element (<= 1.5 ulp vs 0.5 for the division,
    // ~8 fewer instructions per element -- this kernel is issue-heavy)
    float rs[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) rs[c] = __frcp_rn(sm[c]);
    for (int64_t i0 = lane; i0 < n4; i0 += 32 * UN) {
        float4 x[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const int64_t i = i0 + 32 * k;
            if (i < n4) x[k] = S4[i];
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const int64_t i = i0 + 32 * k;
            if (i < n4) {
                float4 a;
                a.x = __fmul_rn(expf(x[k].x - m[0]), rs[0]);
                a.y = __fmul_rn(expf(x[k].y - m[1]), rs[1]);
                a.z = __fmul_rn(expf(x[k].z - m[2]), rs[2]);
                a.w = __fmul_rn(expf(x[k].w - m[3]), rs[3]);
                O4[i] = a;
            }
        }
    }
}

// H divides 32: warp per row, lane-strided over the row's (edge, head) elements.
__global__ void __launch_bounds__(THREADS) softmax_warp_kernel(const int32_t* __restrict__ rows, int64_t n_rows,
                                                               const int64_t* __restrict__ rp,
                                                               const int32_t* __restrict__ eid, int H,
                                                               const float* S, float* out) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    if (r >= n_rows) return;
    const int64_t v = rows[r];
    const int64_t s0 = rp[v], s1 = rp[v + 1];
    const int64_t n = (s1 - s0) * H;
    if (n == 0) return;
    const int h = lane % H;
    float m = -INFINITY, sum = 0.f;
    constexpr int UN = 4;
    for (int64_t q0 = lane; q0 < n; q0 += 32 * UN) {
        float x[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            const int64_t q = q0 + 32 * k;
            if (q < n) {
                const int64_t idx = eid ? int64_t(__ldg(eid + s0 + q / H)) * H + h : s0 * H + q;
                x[k] = S[idx];
            } else {
                x[k] = -INFINITY;
            }
        }
#pragma unroll
        for (int k = 0; k < UN; ++k)
            if (q0 + 32 * k < n) online(m, sum, x[k]);
    }
    for (int o = 16; o >= H; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
        merge(m, sum, m2, s2);
    }
    for (int64_t q = lane; q < n; q += 32) {
        const int64_t p = s0 + q / H;
        const int64_t idx = eid ? int64_t(__ldg(eid + p)) * H + h : s0 * H + q;
        out[idx] = expf(S[idx] - m) / sum;
    }
}

// Generic H: one thread per (row, head), sequential passes.
__global__ void __launch_bounds__(THREADS) softmax_thread_kernel(const int32_t* __restrict__ rows, int64_t n_rows,
                                                                 const int64_t* __restrict__ rp,
                                                                 const int32_t* __restrict__ eid, int H,
                                                                 const float* S, float* out) {
    const int64_t t = int64_t(blockIdx.x) * THREADS + threadIdx.x;
    if (t >= n_rows * H) return;
    const int64_t v = rows[t / H];
    const int h = int(t % H);
    const int64_t s0 = rp[v], s1 = rp[v + 1];
    float m = -INFINITY, sum = 0.f;
    for (int64_t p = s0; p < s1; ++p) {
        const float x = S[(eid ? int64_t(eid[p]) : p) * H + h];
        if (x > m) { sum = sum * expf(m - x) + 1.f; m = x; }
        else sum += expf(x - m);
    }
    for (int64_t p = s0; p < s1; ++p) {
        const int64_t idx = (eid ? int64_t(eid[p]) : p) * H + h;
        out[idx] = expf(S[idx] - m) / sum;
    }
}

}  // namespace

namespace fgk {

fg_status launch_edge_softmax(const fg_graph* g, int H, const float* S, float* out, cudaStream_t st) {
    const int64_t n_rows = g->n_nonempty;   // empty rows have no edges to normalise
    if (n_rows == 0) return FG_OK;
    if (H % 4 == 0 && 32 % (H / 4) == 0 && g->eid == nullptr) {
        const int64_t blocks = (n_rows * 32 + THREADS - 1) / THREADS;
        softmax_vec_kernel<<<unsigned(blocks), THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr, H, S, out);
    } else if (32 % H == 0) {
        const int64_t blocks = (n_rows * 32 + THREADS - 1) / THREADS;
        softmax_warp_kernel<<<unsigned(blocks), THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr, g->eid, H, S,
                                                                  out);
    } else {
        const int64_t blocks = (n_rows * H + THREADS - 1) / THREADS;
        softmax_thread_kernel<<<unsigned(blocks), THREADS, 0, st>>>(g->rows_by_deg, n_rows, g->row_ptr, g->eid, H, S,
                                                                    out);
    }
    return check_launch("edge_softmax");
}

}  // namespace fgk
