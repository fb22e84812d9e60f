// device_common.cuh -- device helpers shared by the gather kernels of libfg.so
// (gSpMM spmm_impl.cuh, gSDDMM sddmm.cu, fused GAT gat_fused.cu).  Internal:
// not part of the ABI.
#pragma once
#include <cstdint>

namespace fgdev {

// Lane mask of the aligned group of G lanes (G a power of two <= 32) holding `lane`.
template <int G>
__device__ __forceinline__ unsigned group_mask(int lane) {
    if constexpr (G == 32) return 0xffffffffu;
    else return ((1u << G) - 1u) << (lane & ~(G - 1));
}

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// 4 bf16 (one 8-byte chunk, feature 0 in the low half of .x) -> 4 fp32, exact
__device__ __forceinline__ float4 bf16x4(uint2 w) {
    return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y << 16),
                       __uint_as_float(w.y & 0xffff0000u));
}

// 4-term dot product, FMA chain (summation order fixed: w, z, y, x)
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

// Recursive-halving reduce-scatter of K values over W aligned lanes of a group:
// at offset o the lane keeps the half of its values selected by (gl & o) and adds
// the partner's copy of that half.  Afterwards lane gl holds, in v[0 .. K/2^L),
// the W-lane sums of original indices bits*K/2^L + i (bits = the top L bits of
// gl mod W, L = min(log2 K, log2 W)); remaining levels are a plain butterfly.
// Every value is summed over the same lane tree (pairs by XOR offset W/2, ...,
// 1), whichever slot it occupies.
template <int K, int W, int G>
__device__ __forceinline__ void reduce_scatter(float (&v)[K], int gl, unsigned mask) {
    if constexpr (W > 1) {
        constexpr int o = W / 2;
        if constexpr (K > 1) {
            const bool up = (gl & o) != 0;
#pragma unroll
            for (int i = 0; i < K / 2; ++i) {
                const float send = up ? v[i] : v[i + K / 2];
                const float keep = up ? v[i + K / 2] : v[i];
                v[i] = keep + __shfl_xor_sync(mask, send, o, G);
            }
            float (&h)[K / 2] = *reinterpret_cast<float(*)[K / 2]>(&v[0]);
            reduce_scatter<K / 2, W / 2, G>(h, gl, mask);
        } else {
#pragma unroll
            for (int oo = o; oo >= 1; oo >>= 1) v[0] += __shfl_xor_sync(mask, v[0], oo, G);
        }
    }
}

// cp.async (LDGSTS) into shared memory without registers in flight: 16 bytes
// bypassing L1 (.cg), or 4 bytes (.ca; .cg takes 16 only); one commit group per
// call of cp_async_commit, cp_async_wait<N> = at most N groups still pending.
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* g) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4_ca(void* smem, const void* g) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace fgdev
