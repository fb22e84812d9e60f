// ldpol.cuh -- L2 eviction-priority loads for the source-row gathers.
//
// The paper stages high-degree source vertices in fast memory (hybrid
// partitioning).  On the B200 the fast memory shared by all
// SMs is the 126 MB L2; when X does not fit, gathers of the rows of the
// hottest sources (by out-degree, fg_graph::src_deg; at most FG_HOT_MB of rows)
// are issued with an L2 evict_last policy and all other source rows with
// evict_first, so the streaming cold rows do not evict the reused hot ones.
// createpolicy builds the 64-bit policy once per thread; the policy operand
// must be warp-uniform, so callers only pass per-edge policies where a whole
// warp loads the same source row (G == 32).
#pragma once
#include <cstdint>

namespace fgpol {

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_unchanged() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// policy for the cold (non-hot) source rows: 0 evict_normal, 1 evict_first,
// 2 evict_unchanged (FG_HOT_COLD, development knob)
__device__ __forceinline__ uint64_t policy_cold(int kind) {
    return kind == 1 ? policy_evict_first() : kind == 2 ? policy_evict_unchanged() : policy_evict_normal();
}

__device__ __forceinline__ float4 ldg_policy(const float4* ptr, uint64_t pol) {
    float4 r;
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(ptr), "l"(pol));
    return r;
}

constexpr int HOT_BIT = int(0x80000000u);   // hot flag carried in a staged source index
constexpr int IDX_MASK = 0x7fffffff;

}  // namespace fgpol
