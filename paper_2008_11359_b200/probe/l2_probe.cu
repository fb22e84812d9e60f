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
    const int64_t total_rows = (1600LL << 20) / (int64_t(F) * 4);   // ~1.6 GB of row reads per launch
    const int64_t rpg = (total_rows / groups + U - 1) / U * U;
    const float ms = best_ms([&] { gather_kernel<G, NV, U><<<blocks, threads>>>(X, nrows, F4, rpg, sink); }, 5);
    const double gbs = double(groups) * rpg * F * 4 / (ms * 1e-3) / 1e9;
    if (verbose)
        printf("gather F=%4d X=%4lld MiB G=%2d NV=%d U=%d blocks/SM=%d: %.3f ms %.1f GB/s\n", F,
               (long long)(x_bytes >> 20), G, NV, U, blocks_per_sm, ms, gbs);
    return gbs;
}

double maxd(double a, double b) { return a > b ? a : b; }

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

extern "C" int fgprobe_l2(void* buf, int64_t buf_bytes, double* out5) {
    return fgprobe_l2_verbose(buf, buf_bytes, out5, 0);
}
