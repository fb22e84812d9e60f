// l2_probe.cu -- libfgprobe.so: measure, live on the bench's GPU, the bandwidth
// at which L2 serves the gather pattern of the gSpMM / gSDDMM kernels.  This is a
// MEASUREMENT utility for bench.py's roofline (not part of the method, not in
// include/fg.h): on the reddit-shaped graph ~half to ~95 % of the per-edge
// source-row gathers hit L2, so those kernels are bound by L2 gather throughput,
// which no datasheet states -- it is measured here instead.
//
//   gather: groups of G lanes read whole random rows (F floats, one float4 per
//           lane per 16 B column chunk, NV chunks per lane) of an L2-resident X,
//           U rows in flight per group -- the kernels' access pattern without the
//           arithmetic or the index loads;
//   stream: coalesced re-reads of an L2-resident buffer (the L2's sequential
//           read ceiling, for context).
//
// extern "C" int fgprobe_l2(void* buf, int64_t buf_bytes, double* out5)
//   buf: caller-owned device buffer of >= 96 MiB (contents irrelevant);
//   out5[0] = best gather GB/s, 2 KiB rows (F = 512) over a 64 MiB X
//   out5[1] = best gather GB/s, 512 B rows (F = 128) over a 64 MiB X
//   out5[2] = best gather GB/s, 128 B rows (F = 32) over a 64 MiB X
//   out5[3] = best stream GB/s over a 32 MiB buffer
//   out5[4] = the best of [0..2] (the gather ceiling)
//   returns 0 on success, else a cudaError_t; synchronises the device.
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

namespace {

__global__ void stream_kernel(const float4* __restrict__ b, int64_t n4, int reps, float* sink) {
    float4 acc = make_float4(0, 0, 0, 0);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride * 4) {
            float4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = (i + k * stride < n4) ? __ldg(b + i + k * stride) : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int k = 0; k < 4; ++k) { acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w; }
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[0] = acc.x;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <int G, int NV, int U>
__global__ void gather_kernel(const float4* __restrict__ X, int nrows, int F4, int64_t rows_per_group, float* sink) {
    const int gl = threadIdx.x & (G - 1);
    const int64_t grp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t t = 0; t < rows_per_group; t += U) {
        float4 x[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t r = hash32(uint32_t(grp * 7919 + t + u)) % uint32_t(nrows);
#pragma unroll
            for (int j = 0; j < NV; ++j) x[u][j] = __ldg(X + int64_t(r) * F4 + gl + G * j);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < NV; ++j) { acc.x += x[u][j].x; acc.y += x[u][j].y; acc.z += x[u][j].z; acc.w += x[u][j].w; }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[0] = acc.x;
}

template <typename K>
float best_ms(K launch, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();   // warm: pulls the buffer into L2
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int i = 0; i < iters; ++i) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int g_sms = 148;

template <int G, int NV, int U>
double gather_gbs(const float4* X, int64_t x_bytes, int F, int blocks_per_sm, float* sink, bool verbose) {
    const int F4 = F / 4;
    const int nrows = int(x_bytes / (int64_t(F) * 4));
    const int threads = 256;
    const int blocks = g_sms * blocks_per_sm;
    const int64_t groups = int64_t(blocks) * threads / G;
    const int64_t total_rows = (6400LL << 20) / (int64_t(F) * 4);   // ~6.4 GB of row reads per launch (long enough that ramp-up does not cap the rate)
    const int64_t rpg = (total_rows / groups + U - 1) / U * U;
    const float ms = best_ms([&] { gather_kernel<G, NV, U><<<blocks, threads>>>(X, nrows, F4, rpg, sink); }, 5);
    const double gbs = double(groups) * rpg * F * 4 / (ms * 1e-3) / 1e9;
    if (verbose)
        printf("gather F=%4d X=%4lld MiB G=%2d NV=%d U=%d blocks/SM=%d: %.3f ms %.1f GB/s\n", F,
               (long long)(x_bytes >> 20), G, NV, U, blocks_per_sm, ms, gbs);
    return gbs;
}

double maxd(double a, double b) { return a > b ? a : b; }

// ---------------------------------------------------------------- TMA bulk row gather
// The same random whole-row gathers, moved by the TMA engine instead of LDG:
// lanes of one producer warp each issue cp.async.bulk (one 16-byte-aligned row
// per instruction) into a STAGES-deep shared-memory ring of RPS rows per stage,
// completing on an mbarrier (expect_tx); NC consumer warps wait for each stage,
// optionally read it from shared memory (READ: LDS.128 + add, as a gSDDMM /
// gSpMM consumer would), and release it.  Measures whether TMA row gathers
// beat the register-bound LDG gathers above.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}"
                 ::"r"(smem_u32(b)), "r"(ph) : "memory");
}

template <int ROWB, int STAGES, int RPS, int NC, bool READ>
__global__ void __launch_bounds__((NC + 1) * 32) tma_gather_kernel(const char* __restrict__ X, int nrows,
                                                                   int iters, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* buf = sm;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * RPS * ROWB);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC * 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    if (warp == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                             "r"(RPS * ROWB) : "memory");
            __syncwarp();
            for (int r = lane; r < RPS; r += 32) {
                const uint32_t row = hash32(uint32_t(blockIdx.x * 1000003u + it * RPS + r)) % uint32_t(nrows);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                    ::"r"(smem_u32(buf + (s * RPS + r) * ROWB)), "l"(X + int64_t(row) * ROWB), "r"(ROWB),
                    "r"(smem_u32(&full[s])) : "memory");
            }
        }
    } else {
        const int ct = threadIdx.x - 32;
        for (int it = 0; it < iters; ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            if (READ) {
                const float4* b4 = reinterpret_cast<const float4*>(buf + s * RPS * ROWB);
                for (int i = ct; i < RPS * ROWB / 16; i += NC * 32) {
                    const float4 v = b4[i];
                    acc += v.x + v.y + v.z + v.w;
                }
            }
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

template <int ROWB, int STAGES, int RPS, int NC, bool READ>
double tma_gbs(const char* X, int64_t x_bytes, int ctas_per_sm, float* sink, bool verbose) {
    const int nrows = int(x_bytes / ROWB);
    const int smem = STAGES * RPS * ROWB + 2 * STAGES * 8;
    auto k = tma_gather_kernel<ROWB, STAGES, RPS, NC, READ>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 0;
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int blocks = g_sms * ctas_per_sm;
    const int64_t total = (1600LL << 20) / ROWB;
    const int iters = int((total / blocks + RPS - 1) / RPS);
    const float ms = best_ms([&] { k<<<blocks, (NC + 1) * 32, smem>>>(X, nrows, iters, sink); }, 5);
    const double gbs = double(blocks) * iters * RPS * ROWB / (ms * 1e-3) / 1e9;
    if (verbose)
        printf("tma-bulk rowB=%4d X=%4lld MiB stages=%d rows/stage=%d consumers=%d ctas/SM=%d read=%d: %.3f ms %.1f GB/s\n",
               ROWB, (long long)(x_bytes >> 20), STAGES, RPS, NC, ctas_per_sm, int(READ), ms, gbs);
    return gbs;
}

// The same gathers with the Blackwell TMA row gather (cp.async.bulk.tensor.2d
// ... tile::gather4): ONE request moves 4 arbitrary rows x BOXC columns of a 2D
// tensor map over X (rows x F fp32), so the per-request cost is amortised over
// 4 rows -- the bulk-copy sweep above shows ~1 request per ~32 clk per SM.
template <int F, int BOXC, int STAGES, int RPS, int NC, bool READ>
__global__ void __launch_bounds__((NC + 1) * 32) tma_gather4_kernel(const __grid_constant__ CUtensorMap map,
                                                                    int nrows, int iters, float* sink) {
    constexpr int ROWB = F * 4;
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* buf = sm;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * RPS * ROWB);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC * 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    if (warp == 0) {
        constexpr int NCH = F / BOXC;          // column chunks per row
        constexpr int NREQ = (RPS / 4) * NCH;  // gather4 requests per stage
        for (int it = 0; it < iters; ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                             "r"(RPS * ROWB) : "memory");
            __syncwarp();
            for (int q = lane; q < NREQ; q += 32) {
                const int g4 = q / NCH, ch = q % NCH;
                int r[4];
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    r[k] = int(hash32(uint32_t(blockIdx.x * 1000003u + it * RPS + g4 * 4 + k)) % uint32_t(nrows));
                // smem: the 4 rows' column chunk ch, [4][BOXC] fp32, chunk-major inside the stage
                unsigned char* dst = buf + s * RPS * ROWB + (g4 * NCH + ch) * 4 * BOXC * 4;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                    ::"r"(smem_u32(dst)), "l"(&map), "r"(ch * BOXC), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
                    "r"(smem_u32(&full[s])) : "memory");
            }
        }
    } else {
        const int ct = threadIdx.x - 32;
        for (int it = 0; it < iters; ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            if (READ) {
                const float4* b4 = reinterpret_cast<const float4*>(buf + s * RPS * ROWB);
                for (int i = ct; i < RPS * ROWB / 16; i += NC * 32) {
                    const float4 v = b4[i];
                    acc += v.x + v.y + v.z + v.w;
                }
            }
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <int F, int BOXC, int STAGES, int RPS, int NC, bool READ>
double gather4_gbs(const char* X, int64_t x_bytes, int ctas_per_sm, float* sink, bool verbose) {
    constexpr int ROWB = F * 4;
    const int nrows = int(x_bytes / ROWB);
    CUtensorMap map;
    cuuint64_t gdim[2] = {cuuint64_t(F), cuuint64_t(nrows)};
    cuuint64_t gstride[1] = {cuuint64_t(ROWB)};
    cuuint32_t box[2] = {cuuint32_t(BOXC), 1u};
    cuuint32_t estr[2] = {1u, 1u};
    auto enc = encode_fn();
    if (!enc) return -1;
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<char*>(X), gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        if (verbose) printf("gather4 F=%d BOXC=%d: cuTensorMapEncodeTiled error %d\n", F, BOXC, int(r));
        return -2;
    }
    const int smem = STAGES * RPS * ROWB + 2 * STAGES * 8;
    auto k = tma_gather4_kernel<F, BOXC, STAGES, RPS, NC, READ>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 0;
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int blocks = g_sms * ctas_per_sm;
    const int64_t total = (1600LL << 20) / ROWB;
    const int iters = int((total / blocks + RPS - 1) / RPS);
    const float ms = best_ms([&] { k<<<blocks, (NC + 1) * 32, smem>>>(map, nrows, iters, sink); }, 5);
    cudaError_t e = cudaGetLastError();
    const double gbs = double(blocks) * iters * RPS * ROWB / (ms * 1e-3) / 1e9;
    if (verbose)
        printf("tma-gather4 F=%4d box=%3d X=%4lld MiB stages=%d rows/stage=%d consumers=%d ctas/SM=%d read=%d: "
               "%.3f ms %.1f GB/s %s\n", F, BOXC, (long long)(x_bytes >> 20), STAGES, RPS, NC, ctas_per_sm,
               int(READ), ms, gbs, e == cudaSuccess ? "" : cudaGetErrorString(e));
    return gbs;
}

}  // namespace

// TMA gather4 sweep (tooling only): out4 = best GB/s for F = 128 (512 B rows)
// without / with the shared-memory read, and F = 256 (1 KiB rows) without / with.
extern "C" int fgprobe_gather4(void* buf, int64_t buf_bytes, double* out4, int verbose) {
    if (!buf || !out4 || buf_bytes < (96LL << 20)) return int(cudaErrorInvalidValue);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    const char* X = static_cast<const char*>(buf);
    float* sink = reinterpret_cast<float*>(static_cast<char*>(buf) + buf_bytes - 64);
    const int64_t xb = 64LL << 20;
    double a = 0, b = 0, c = 0, d = 0;
    a = maxd(a, gather4_gbs<128, 128, 8, 16, 4, false>(X, xb, 2, sink, verbose));
    a = maxd(a, gather4_gbs<128, 128, 4, 32, 4, false>(X, xb, 3, sink, verbose));
    a = maxd(a, gather4_gbs<128, 128, 8, 8, 4, false>(X, xb, 4, sink, verbose));
    b = maxd(b, gather4_gbs<128, 128, 8, 16, 4, true>(X, xb, 2, sink, verbose));
    b = maxd(b, gather4_gbs<128, 128, 4, 32, 8, true>(X, xb, 3, sink, verbose));
    b = maxd(b, gather4_gbs<128, 128, 8, 8, 4, true>(X, xb, 4, sink, verbose));
    c = maxd(c, gather4_gbs<256, 256, 8, 8, 4, false>(X, xb, 2, sink, verbose));
    c = maxd(c, gather4_gbs<256, 256, 4, 16, 4, false>(X, xb, 3, sink, verbose));
    d = maxd(d, gather4_gbs<256, 256, 8, 8, 4, true>(X, xb, 2, sink, verbose));
    d = maxd(d, gather4_gbs<256, 256, 4, 16, 8, true>(X, xb, 3, sink, verbose));
    gather4_gbs<512, 256, 4, 8, 8, true>(X, xb, 3, sink, verbose);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    out4[0] = a; out4[1] = b; out4[2] = c; out4[3] = d;
    return int(e);
}

// TMA bulk-copy row gathers vs the LDG gathers (verbose sweep; tooling only).
// out4: best GB/s for 2 KiB rows without / with the shared-memory read, and for
// 512 B rows without / with it, all over a 64 MiB (L2-resident) X.
extern "C" int fgprobe_tma(void* buf, int64_t buf_bytes, double* out4, int verbose) {
    if (!buf || !out4 || buf_bytes < (96LL << 20)) return int(cudaErrorInvalidValue);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    const char* X = static_cast<const char*>(buf);
    float* sink = reinterpret_cast<float*>(static_cast<char*>(buf) + buf_bytes - 64);
    const int64_t xb = 64LL << 20;
    double a = 0, b = 0, c = 0, d = 0;
    a = maxd(a, tma_gbs<2048, 8, 4, 4, false>(X, xb, 2, sink, verbose));
    a = maxd(a, tma_gbs<2048, 8, 4, 4, false>(X, xb, 3, sink, verbose));
    a = maxd(a, tma_gbs<2048, 4, 8, 4, false>(X, xb, 3, sink, verbose));
    a = maxd(a, tma_gbs<2048, 12, 4, 2, false>(X, xb, 2, sink, verbose));
    b = maxd(b, tma_gbs<2048, 8, 4, 4, true>(X, xb, 2, sink, verbose));
    b = maxd(b, tma_gbs<2048, 8, 4, 4, true>(X, xb, 3, sink, verbose));
    b = maxd(b, tma_gbs<2048, 4, 8, 8, true>(X, xb, 3, sink, verbose));
    b = maxd(b, tma_gbs<2048, 6, 4, 8, true>(X, xb, 4, sink, verbose));
    c = maxd(c, tma_gbs<512, 8, 16, 4, false>(X, xb, 2, sink, verbose));
    c = maxd(c, tma_gbs<512, 8, 32, 4, false>(X, xb, 3, sink, verbose));
    d = maxd(d, tma_gbs<512, 8, 16, 4, true>(X, xb, 2, sink, verbose));
    d = maxd(d, tma_gbs<512, 8, 32, 8, true>(X, xb, 3, sink, verbose));
    // DRAM-resident X (503 MB) for the 2 KiB rows
    if (buf_bytes >= (512LL << 20)) {
        tma_gbs<2048, 8, 4, 4, false>(X, 503LL << 20, 3, sink, verbose);
        tma_gbs<2048, 8, 4, 4, true>(X, 503LL << 20, 3, sink, verbose);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    out4[0] = a; out4[1] = b; out4[2] = c; out4[3] = d;
    return int(e);
}

namespace {
}  // namespace

extern "C" int fgprobe_l2_verbose(void* buf, int64_t buf_bytes, double* out5, int verbose) {
    if (!buf || !out5 || buf_bytes < (96LL << 20)) return int(cudaErrorInvalidValue);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    const float4* X = reinterpret_cast<const float4*>(buf);
    float* sink = reinterpret_cast<float*>(static_cast<char*>(buf) + buf_bytes - 64);
    const int64_t xb = 64LL << 20;
    double r512 = 0, r128 = 0, r32 = 0, st = 0;
    r512 = maxd(r512, gather_gbs<32, 4, 2>(X, xb, 512, 3, sink, verbose));
    r512 = maxd(r512, gather_gbs<32, 4, 4>(X, xb, 512, 4, sink, verbose));
    r512 = maxd(r512, gather_gbs<32, 4, 2>(X, xb, 512, 8, sink, verbose));
    r128 = maxd(r128, gather_gbs<32, 1, 4>(X, xb, 128, 4, sink, verbose));
    r128 = maxd(r128, gather_gbs<32, 1, 8>(X, xb, 128, 8, sink, verbose));
    r32 = maxd(r32, gather_gbs<8, 1, 8>(X, xb, 32, 4, sink, verbose));
    r32 = maxd(r32, gather_gbs<8, 1, 8>(X, xb, 32, 8, sink, verbose));
    {
        const int64_t mb = 32;
        const int64_t n4 = (mb << 20) / 16;
        const int reps = 128;
        const float ms = best_ms([&] { stream_kernel<<<g_sms * 8, 256>>>(X, n4, reps, sink); }, 5);
        st = double(reps) * (mb << 20) / (ms * 1e-3) / 1e9;
        if (verbose) printf("stream 32 MiB: %.3f ms %.1f GB/s\n", ms, st);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    out5[0] = r512;
    out5[1] = r128;
    out5[2] = r32;
    out5[3] = st;
    out5[4] = maxd(r512, maxd(r128, r32));
    return int(e);
}


// X-size sweep (tooling only): random 2 KiB-row LDG gathers and sequential
// re-reads over an X of 4..160 MiB, ~6.4 GB moved per launch.  Tests whether
// the gather ceiling depends on how much of the L2 the working set occupies
// (B200's L2 is two halves, one per die).  out[2*i], out[2*i+1] = gather,
// stream GB/s for the i-th size in sizes_mb (n sizes).
extern "C" int fgprobe_xsweep(void* buf, int64_t buf_bytes, const int* sizes_mb, int n, double* out, int verbose) {
    if (!buf || !out || !sizes_mb) return int(cudaErrorInvalidValue);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    const float4* X = reinterpret_cast<const float4*>(buf);
    float* sink = reinterpret_cast<float*>(static_cast<char*>(buf) + buf_bytes - 64);
    for (int i = 0; i < n; ++i) {
        const int64_t xb = int64_t(sizes_mb[i]) << 20;
        if (xb + 4096 > buf_bytes) { out[2 * i] = out[2 * i + 1] = 0; continue; }
        const int F = 512, F4 = 128, G = 32, U = 4;
        const int nrows = int(xb / (F * 4));
        const int blocks = g_sms * 4;
        const int64_t groups = int64_t(blocks) * 256 / G;
        const int64_t total_rows = (6400LL << 20) / (F * 4);
        const int64_t rpg = (total_rows / groups + U - 1) / U * U;
        float ms = best_ms([&] { gather_kernel<32, 4, 4><<<blocks, 256>>>(X, nrows, F4, rpg, sink); }, 3);
        out[2 * i] = double(groups) * rpg * F * 4 / (ms * 1e-3) / 1e9;
        const int64_t n4 = xb / 16;
        const int reps = int((6400LL << 20) / xb);
        ms = best_ms([&] { stream_kernel<<<g_sms * 8, 256>>>(X, n4, reps, sink); }, 3);
        out[2 * i + 1] = double(reps) * xb / (ms * 1e-3) / 1e9;
        if (verbose) printf("xsweep X=%4d MiB: gather 2KiB rows %.1f GB/s, stream %.1f GB/s\n", sizes_mb[i], out[2 * i], out[2 * i + 1]);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    return int(e);
}


// ---------------------------------------------------------------- load-flavour sweep
// The same random whole-row gathers with other LDG flavours: LD = 0 __ldg
// (LDG.128, L1-allocating), 1 ld.global.nc.L1::no_allocate.v4, 2 the same with
// the L2::256B prefetch hint, 3 Blackwell 256-bit loads (ld.global.nc.
// L1::no_allocate.v8.f32 -> LDG.256: half the load instructions per row).
template <int LD>
__device__ __forceinline__ void ld_row_piece(const float4* p, float4& a, float4& b) {
    if constexpr (LD == 0) {
        a = __ldg(p);
    } else if constexpr (LD == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p));
    } else if constexpr (LD == 2) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p));
    } else {
        asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                     : "l"(p));
    }
}

// G lanes per row; each lane NV pieces of 16 B (LD < 3) or 32 B (LD == 3)
template <int G, int NV, int U, int LD>
__global__ void gather_ld_kernel(const float4* __restrict__ X, int nrows, int F4, int64_t rows_per_group, float* sink) {
    constexpr int W = LD == 3 ? 2 : 1;   // float4 per piece
    const int gl = threadIdx.x & (G - 1);
    const int64_t grp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t t = 0; t < rows_per_group; t += U) {
        float4 x[U][NV], y[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t r = hash32(uint32_t(grp * 7919 + t + u)) % uint32_t(nrows);
#pragma unroll
            for (int j = 0; j < NV; ++j) ld_row_piece<LD>(X + int64_t(r) * F4 + W * (gl + G * j), x[u][j], y[u][j]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                acc.x += x[u][j].x; acc.y += x[u][j].y; acc.z += x[u][j].z; acc.w += x[u][j].w;
                if (LD == 3) { acc.x += y[u][j].x; acc.y += y[u][j].y; acc.z += y[u][j].z; acc.w += y[u][j].w; }
            }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) sink[0] = acc.x;
}

template <int G, int NV, int U, int LD>
double gather_ld_gbs(const float4* X, int64_t x_bytes, int F, int blocks_per_sm, float* sink, bool verbose) {
    const int F4 = F / 4;
    const int nrows = int(x_bytes / (int64_t(F) * 4));
    const int blocks = g_sms * blocks_per_sm;
    const int64_t groups = int64_t(blocks) * 256 / G;
    const int64_t total_rows = (6400LL << 20) / (int64_t(F) * 4);
    const int64_t rpg = (total_rows / groups + U - 1) / U * U;
    const float ms = best_ms([&] { gather_ld_kernel<G, NV, U, LD><<<blocks, 256>>>(X, nrows, F4, rpg, sink); }, 3);
    const double gbs = double(groups) * rpg * F * 4 / (ms * 1e-3) / 1e9;
    if (verbose)
        printf("gather-ld LD=%d F=%4d X=%4lld MiB G=%2d NV=%d U=%d blocks/SM=%d: %.3f ms %.1f GB/s\n", LD, F,
               (long long)(x_bytes >> 20), G, NV, U, blocks_per_sm, ms, gbs);
    return gbs;
}

extern "C" int fgprobe_ldmodes(void* buf, int64_t buf_bytes, int verbose) {
    if (!buf || buf_bytes < (64LL << 20)) return int(cudaErrorInvalidValue);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    const float4* X = reinterpret_cast<const float4*>(buf);
    float* sink = reinterpret_cast<float*>(static_cast<char*>(buf) + buf_bytes - 64);
    const int64_t xb = 48LL << 20;
    // F = 512 (2 KiB rows): 16-byte pieces 32 lanes x 4; 32-byte pieces 32 lanes x 2
    gather_ld_gbs<32, 4, 2, 0>(X, xb, 512, 3, sink, verbose);
    gather_ld_gbs<32, 4, 4, 0>(X, xb, 512, 4, sink, verbose);
    gather_ld_gbs<32, 4, 2, 1>(X, xb, 512, 3, sink, verbose);
    gather_ld_gbs<32, 4, 4, 1>(X, xb, 512, 4, sink, verbose);
    gather_ld_gbs<32, 4, 2, 2>(X, xb, 512, 3, sink, verbose);
    gather_ld_gbs<32, 4, 4, 2>(X, xb, 512, 4, sink, verbose);
    gather_ld_gbs<32, 2, 2, 3>(X, xb, 512, 3, sink, verbose);
    gather_ld_gbs<32, 2, 4, 3>(X, xb, 512, 4, sink, verbose);
    gather_ld_gbs<32, 2, 4, 3>(X, xb, 512, 3, sink, verbose);
    gather_ld_gbs<32, 2, 8, 3>(X, xb, 512, 3, sink, verbose);
    // F = 256 (1 KiB rows)
    gather_ld_gbs<32, 2, 4, 0>(X, xb, 256, 4, sink, verbose);
    gather_ld_gbs<32, 2, 4, 1>(X, xb, 256, 4, sink, verbose);
    gather_ld_gbs<32, 1, 4, 3>(X, xb, 256, 4, sink, verbose);
    gather_ld_gbs<32, 1, 8, 3>(X, xb, 256, 4, sink, verbose);
    // F = 128 (512 B rows)
    gather_ld_gbs<32, 1, 8, 0>(X, xb, 128, 8, sink, verbose);
    gather_ld_gbs<32, 1, 8, 1>(X, xb, 128, 8, sink, verbose);
    gather_ld_gbs<16, 1, 8, 3>(X, xb, 128, 8, sink, verbose);
    gather_ld_gbs<16, 1, 4, 3>(X, xb, 128, 8, sink, verbose);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    return int(e);
}

extern "C" int fgprobe_l2(void* buf, int64_t buf_bytes, double* out5) {
    return fgprobe_l2_verbose(buf, buf_bytes, out5, 0);
}
