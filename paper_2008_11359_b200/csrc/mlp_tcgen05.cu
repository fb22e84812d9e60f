// mlp_tcgen05.cu -- gSpMM with the MLP message on the 5th-generation tensor
// cores.
//
// Fig. 3b: phi(u, v) = ReLU(sum_k (x_u[k] + x_v[k]) W[k, i]),
// aggregated by max (Fig. 1 "picking the maximum"; MLP aggregation of
// Table tab:gpu-kernel(b), d1 = 8) or sum.  Evaluated in the paper's
// order: s_e = x_u + x_v (one fp32 add per input dimension, as Fig. 3b line
// 1), then z_e = s_e W (the contraction), then ReLU and the aggregation:
//     max: out[v][i] = ReLU(max_e z_e[i]); argmax = first e attaining the max
//          if that is > 0, else the row's first edge (all messages are +0);
//     sum: out[v][i] = sum_e ReLU(z_e[i]).
// Forming s_e before the contraction keeps the error relative to
// sum_k |s_e[k] W[k,i]| -- the oracle's tolerance scale -- also when x_v nearly
// cancels x_u (the earlier x_u W + x_v W split carried an error relative to
// |x_u W| + |x_v W|).
//
// The paper's V100 schedule bound d2 to blocks and tree-reduced d1 over threads
// (listing fig:schedule-mlp-conv-gpu).  Here, per CTA (persistent,
// 4 per SM -- four independent pipelines hide the MMA/commit latency -- each
// owning a contiguous range of destination rows and therefore of CSR edges):
//   * a producer warp walks NT = 64 edges per tile: it finds each edge's
//     destination row in a 32-row window of row_ptr (register binary search),
//     loads x_u and x_v (L2-resident: n x d1 x 4 B), forms s_e, splits it into
//     tensor-core operands and stores them into the B operand (K-major,
//     no-swizzle canonical layout) of a 6-stage shared-memory ring;
//   * one thread issues the MMAs, M = 128 features (W^T, staged once), N = 64
//     edges, accumulating in TMEM (2 x 64 columns, double-buffered):
//       3xTF32 (default): tcgen05.mma.kind::tf32, K = 8, hi*hi + hi*lo + lo*hi
//         (error ~2^-21 relative: fp32-grade; one TF32 pass cannot meet the
//         1e-4 bound);
//       bf16 2-split (FG_TUNE_MLP_IMPL = 2): tcgen05.mma.kind::f16 with bf16
//         operands, K = 16, [s_hi | s_hi] . [w_hi | w_lo] + [s_lo | s_lo] .
//         [w_hi | w_lo] = (s_hi + s_lo)(w_hi + w_lo) (error ~2^-17 relative);
//   * 4 epilogue warps read the accumulator with tcgen05.ld (thread = feature,
//     walking edge columns, so the per-row segmented max needs no cross-lane
//     reduction), keep the running winner as a CSR position, and write each
//     finished row.
// Bound: reading every accumulator element out of TMEM (m x d2 x 4 B; the
// guide's LDTM throughput is 64 B/clk/SM, B300_MICROARCH.md "TMEM") -- on
// reddit d2 = 128 the epilogue's TMEM reads alone take ~2.8 ms of ~4 ms
// (DESIGN.md §6).
#include <cstdint>
#include <cstdlib>

#include "fg_internal.h"

namespace {

constexpr int NT = 64;                    // edges per tile (MMA N; 32 with 4 buffers: 4.7 vs 4.04 ms)
constexpr int NBUF = 2;                   // TMEM accumulator buffers (double buffer)
#ifndef FG_MLP_CTAS
#define FG_MLP_CTAS 4
#endif
#ifndef FG_MLP_LA
#define FG_MLP_LA 4
#endif
#ifndef FG_MLP_LDW
#define FG_MLP_LDW 0    // TMEM read granularity of the epilogue: 0 by reducer (max 16, sum 32), 16, 32
#endif
#ifndef FG_MLP_NPROD
#define FG_MLP_NPROD 2
#endif
constexpr int CTAS_PER_SM = FG_MLP_CTAS;  // 4 independent pipelines per SM hide the MMA/commit latency
constexpr int MT = 128;                   // features per CTA (MMA M)
constexpr int STAGES = 6;                 // B-operand ring (6 x 4 KB: four CTAs per SM fit with the producer staging)
constexpr int NEPI = 4;                   // epilogue warps 0..3 (TMEM lane quarters)
constexpr int MMA_WARP = 4;
constexpr int NPROD = FG_MLP_NPROD;       // producer warps 5, 6 (on two SM sub-partitions)
constexpr int THREADS = (NEPI + 1 + NPROD) * 32;
constexpr int TMEM_COLS = NBUF * NT;      // 128: four CTAs per SM share the 512 columns

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// wait with back-off, for the producer and MMA warps: they run ahead of the
// epilogue and would otherwise spin on try_wait, taking issue slots from the
// epilogue warps that share their SM sub-partition (measured: 27 % of all issued
// instructions were SYNCS / YIELD / BRA spin iterations)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, int ns) {
    uint32_t ok = 0;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (ok) break;
        __nanosleep(ns);
    }
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_NONE canonical layout,
// core matrix = 8 rows x 16 B; LBO = 128 B (next 16-byte K chunk), SBO = 256 B
// (next 8-row group); version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
           (uint64_t(1) << 46);
}
// byte offset of element (row r, k in [0,8)) inside a 128 x 8 tf32 operand tile
__device__ __forceinline__ uint32_t tile_off(int r, int k) {
    return uint32_t((r >> 3) * 256 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
// instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, N = NT, M = MT
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(NT >> 3) << 17) | (uint32_t(MT >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
// wait for the outstanding tcgen05.ld of BOTH 16-column buffers (wait::ld covers all of
// this thread's loads): a is consumed next, b may still be the one in flight
__device__ __forceinline__ void tmem_wait_ld2(uint32_t (&a)[16], uint32_t (&b)[16]) {
    asm volatile(
        "tcgen05.wait::ld.sync.aligned;"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
          "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]), "+r"(a[15]),
          "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]),
          "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]), "+r"(b[14]), "+r"(b[15])
        :
        : "memory");
}
// wait for this thread's outstanding tcgen05.ld; v is threaded through the asm so no use of
// the loaded registers can be scheduled before the wait
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.wait::ld.sync.aligned;"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
          "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
          "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
          "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
        :
        : "memory");
}

// cp.async of `bytes` (0 or 16) bytes into a 16-byte shared slot, zero-filling the
// rest: .ca keeps the line in L1 (x_v: consecutive edges share the row), .cg not.
__device__ __forceinline__ void cp_async16_zfill(uint32_t saddr, const void* g, int bytes, bool l1) {
    if (l1) asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
    else asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ int64_t lower_bound_rp(const int64_t* rp, int64_t n1, int64_t target) {
    int64_t lo = 0, hi = n1;   // first i in [0, n1) with rp[i] >= target
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(rp + mid) < target) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// bf16 (round to nearest even) bits of x, and its value as fp32 (exact)
__device__ __forceinline__ uint32_t bf16_bits(float x) {
    uint16_t r;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float bf16_val(uint32_t b) { return __uint_as_float(b << 16); }

struct Args {
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* eid;
    const float* X;       // [n_src][d_in]
    const float* Xd;      // [n_dst][d_in]
    const float* W;       // [d_in][d2]
    float* out;           // [n_dst][d2]
    int32_t* arg_u;
    int32_t* arg_e;
    int64_t n_dst, nnz, n_src;
    int d_in, d2;
};

constexpr int BACKOFF_NS = 128;   // producer / MMA wait back-off (the epilogue spins)

// Shared memory of one CTA.  Every operand tile is 32 bytes per row per MMA
// (tf32 K = 8 or bf16 K = 16): A tiles 128 rows (4 KB), B tiles NT rows (2 KB).
// 3xTF32: a_hi / a_lo = tf32 hi / lo of W^T, b_hi / b_lo = of s_e (per K step ks).
// bf16:   a_hi = [w_hi | w_lo] (bf16), b_hi = [s_hi | s_hi], b_lo = [s_lo | s_lo].
template <int KS>
struct Smem {
    static constexpr int LA = KS <= 2 ? FG_MLP_LA : 2;   // tiles of x rows in flight per producer lane
    float a_hi[KS][MT * 8];
    float a_lo[KS][MT * 8];
    float b_hi[STAGES][KS][NT * 8];
    float b_lo[STAGES][KS][NT * 8];
    float raw_u[LA][NT][KS * 8];                 // producer staging: x_u, x_v rows (fp32, zero-padded)
    float raw_v[LA][NT][KS * 8];
    int32_t idx[2 * LA][NT];                     // producer staging: neighbour indices
    int32_t rowtag[FG_MLP_NPROD][LA];            // the row of a single-row tile (per producer warp), else -1
    uint64_t full[STAGES], empty[STAGES], tfull[NBUF], tempty[NBUF];
    uint32_t tmem_base;
    int64_t r_lo, r_hi;
};

// Epilogue state of one thread (= one feature column i of the CTA's M tile).
// Edge positions are 32-bit offsets from the CTA's first edge E0 (a CTA owns a
// contiguous CSR range).  The running winner is kept as a position only; its
// source / edge id are read from col_idx / eid once per finished row.
template <bool MAX>
struct Epi {
    const Args* A;
    int r, r_hi;      // current row, end of the CTA's rows
    int64_t E0;       // CSR position of the CTA's first edge
    int rs, re;       // current row's edge range, relative to E0
    int nre;          // prefetched end of row r + 1 (relative)
    float best;
    int bpos;         // relative position of the current winner
    int i;            // global feature index
    bool active;      // i < d2

    // prefetch the next row's end pointer so that the per-row bookkeeping never
    // waits on a global load
    __device__ __forceinline__ void prefetch(int rn) {
        if (rn < r_hi) nre = int(__ldg(A->row_ptr + rn + 1) - E0);
    }
    __device__ __forceinline__ void start_row() {
        best = MAX ? -INFINITY : 0.f;
        bpos = 0;
        prefetch(r + 1);
    }
    __device__ __forceinline__ void finish_row() {
        if (!active) return;
        const int64_t o = int64_t(r) * A->d2 + i;
        if (!MAX) {
            A->out[o] = best;
            return;
        }
        if (re == rs) {
            A->out[o] = 0.f;
            if (A->arg_u) A->arg_u[o] = -1;
            if (A->arg_e) A->arg_e[o] = -1;
            return;
        }
        const bool pos = best > 0.f;
        A->out[o] = pos ? best : 0.f;
        // every message is +0 when max z <= 0: the row's first edge wins
        const int64_t p = E0 + (pos ? bpos : rs);
        if (A->arg_u) A->arg_u[o] = __ldg(A->col_idx + p);
        if (A->arg_e) A->arg_e[o] = A->eid ? __ldg(A->eid + p) : int(p);
    }
    // finish row r and move to r+1 (uniform across the epilogue threads)
    __device__ __forceinline__ void advance() {
        finish_row();
        ++r;
        if (r < r_hi) {
            rs = re;
            re = nre;
            start_row();
        }
    }
    // the W columns of a chunk that lies inside the current row (the common case)
    template <int W>
    __device__ __forceinline__ void consume_full(const uint32_t (&v)[W], int pc) {
        if (MAX) {
            // the chunk maximum by a 3-input max tree (FMNMX3); the first column
            // attaining it is searched only when it beats the running best (strict:
            // ties keep the earlier winner), skipped when no feature of the warp improves
            constexpr int N3 = (W + 2) / 3;
            float t[N3];
#pragma unroll
            for (int j = 0; j < N3; ++j) {
                const float a = __uint_as_float(v[3 * j]);
                const float b = 3 * j + 1 < W ? __uint_as_float(v[(3 * j + 1) % W]) : a;
                const float c = 3 * j + 2 < W ? __uint_as_float(v[(3 * j + 2) % W]) : a;
                t[j] = fmaxf(fmaxf(a, b), c);
            }
#pragma unroll
            for (int st = 1; st < N3; st *= 2)
#pragma unroll
                for (int j = 0; j + st < N3; j += 2 * st) t[j] = fmaxf(t[j], t[j + st]);
            const float m = t[0];
            const bool imp = m > best;
            if (__any_sync(0xffffffffu, imp)) {
                if (imp) {
                    int k = W - 1;
#pragma unroll
                    for (int c = W - 2; c >= 0; --c) k = (__uint_as_float(v[c]) == m) ? c : k;
                    best = m;
                    bpos = pc + k;
                }
            }
        } else {
            float sm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < W; c += 4)
#pragma unroll
                for (int k = 0; k < 4; ++k) sm[k] += fmaxf(__uint_as_float(v[c + k]), 0.f);
            best += (sm[0] + sm[1]) + (sm[2] + sm[3]);
        }
    }
    // general case: chunk at relative position pc with nvalid valid columns,
    // possibly spanning row boundaries
    template <int W>
    __device__ __forceinline__ void consume_split(const uint32_t (&v)[W], int pc, int nvalid) {
        int c0 = 0;
        while (c0 < nvalid) {
            while (pc + c0 >= re) advance();
            const int c1 = min(nvalid, re - pc);
            if (MAX) {
                float b0 = -INFINITY;   // ties -> lowest column
                int k0 = 0;
#pragma unroll
                for (int c = 0; c < W; ++c) {
                    const float x = __uint_as_float(v[c]);
                    if (c >= c0 && c < c1 && x > b0) { b0 = x; k0 = c; }
                }
                if (b0 > best) { best = b0; bpos = pc + k0; }
            } else {
                // columns [c0, c1) belong to row r (bit mask: measured faster than two compares for sum)
                const uint32_t cm = (c1 >= 32 ? 0xffffffffu : ((1u << c1) - 1u)) & ~((1u << c0) - 1u);
                float sm = 0.f;
#pragma unroll
                for (int c = 0; c < W; ++c)
                    if ((cm >> c) & 1u) sm += fmaxf(__uint_as_float(v[c]), 0.f);
                best += sm;
            }
            c0 = c1;
        }
    }
    template <int W>
    __device__ __forceinline__ void consume(const uint32_t (&v)[W], int pc, int nvalid) {
        if (nvalid == W && pc >= rs && pc + W <= re) consume_full<W>(v, pc);   // warp-uniform
        else if (nvalid > 0) consume_split<W>(v, pc, nvalid);
    }
};

__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// The B-operand rows of edge slot e (tile row e) for s = x_u + x_v, dimensions
// [ks*8, ks*8 + 8): 3xTF32 -> tf32 hi / lo (RNA); bf16 -> bf16 hi / lo (RN),
// each written twice (K positions 0-7 and 8-15 of the K = 16 step).
template <bool BF>
__device__ __forceinline__ void store_split(uint32_t bh, uint32_t bl, int e, const float4& s0, const float4& s1) {
    const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    if constexpr (!BF) {
        // hi = s with the low 13 mantissa bits cleared (a tf32 value), lo = s - hi
        // (exact, <= 13 significant bits), fed as raw fp32: the tensor core reads
        // its top 19 bits, so |s - hi - tf32(lo)| <= 2^-20 |s| -- two ALU ops per
        // value instead of two conversions and a subtraction (the producer shares
        // an SM sub-partition with an epilogue warp)
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            hi[k] = __float_as_uint(sv[k]) & 0xffffe000u;
            lo[k] = __float_as_uint(sv[k] - __uint_as_float(hi[k]));
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            sts128(bh + tile_off(e, 4 * c), hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
            sts128(bl + tile_off(e, 4 * c), lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
        }
    } else {
        uint32_t hp[4], lp[4];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const uint32_t h0 = bf16_bits(sv[k]), h1 = bf16_bits(sv[k + 1]);
            const uint32_t l0 = bf16_bits(sv[k] - bf16_val(h0)), l1 = bf16_bits(sv[k + 1] - bf16_val(h1));
            hp[k / 2] = h0 | (h1 << 16);
            lp[k / 2] = l0 | (l1 << 16);
        }
        // K-major bf16: 8 elements per 16-byte core-matrix row; K chunk 1 at +128 B
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            sts128(bh + tile_off(e, 4 * c), hp[0], hp[1], hp[2], hp[3]);
            sts128(bl + tile_off(e, 4 * c), lp[0], lp[1], lp[2], lp[3]);
        }
    }
}

// instruction descriptor: kind::f16 with bf16 A/B, D f32, K-major, N = NT, M = MT
constexpr uint32_t IDESC_BF16 = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(NT >> 3) << 17) |
                                (uint32_t(MT >> 4) << 24);
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC_BF16), "r"(accumulate));
}

template <int KS, bool MAX, bool BF>
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM) mlp_tcgen05_kernel(const __grid_constant__ Args A) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem<KS>& S = *reinterpret_cast<Smem<KS>*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int mbase = blockIdx.y * MT;

    if (tid == 0) {
        const int64_t nb = gridDim.x, b = blockIdx.x;
        const int64_t t_lo = (A.nnz * b) / nb, t_hi = (A.nnz * (b + 1)) / nb;
        S.r_lo = (b == 0) ? 0 : lower_bound_rp(A.row_ptr, A.n_dst + 1, t_lo);
        S.r_hi = (b == nb - 1) ? A.n_dst : lower_bound_rp(A.row_ptr, A.n_dst + 1, t_hi);
        if (S.r_hi < S.r_lo) S.r_hi = S.r_lo;
        for (int s = 0; s < STAGES; ++s) { mbar_init(&S.full[s], NPROD * 32); mbar_init(&S.empty[s], 1); }
        for (int b2 = 0; b2 < NBUF; ++b2) { mbar_init(&S.tfull[b2], 1); mbar_init(&S.tempty[b2], NEPI * 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // stage the A operand (W^T: row = feature, k = input dim), once
    for (int idx = tid; idx < KS * MT * 8; idx += THREADS) {
        const int ks = idx / (MT * 8), rem = idx % (MT * 8), r = rem / 8, k = rem % 8;
        const int kk = ks * 8 + k, col = mbase + r;
        const float w = (kk < A.d_in && col < A.d2) ? A.W[int64_t(kk) * A.d2 + col] : 0.f;
        if constexpr (!BF) {
            const float hi = tf32_rna(w);
            *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(S.a_hi[ks]) + tile_off(r, k)) = hi;
            *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(S.a_lo[ks]) + tile_off(r, k)) = tf32_rna(w - hi);
        } else {
            // [w_hi | w_lo]: element (r, k) of the K = 16 bf16 tile sits at byte
            // (r>>3)*256 + (k>>3)*128 + (r&7)*16 + (k&7)*2
            const uint32_t hb = bf16_bits(w), lb = bf16_bits(w - bf16_val(hb));
            unsigned char* base = reinterpret_cast<unsigned char*>(S.a_hi[ks]);
            const uint32_t o = uint32_t((r >> 3) * 256 + (r & 7) * 16 + k * 2);
            *reinterpret_cast<uint16_t*>(base + o) = uint16_t(hb);
            *reinterpret_cast<uint16_t*>(base + o + 128) = uint16_t(lb);
        }
    }
    fence_async_smem();
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;
    const int64_t r_lo = S.r_lo, r_hi = S.r_hi;
    const int64_t E0 = __ldg(A.row_ptr + r_lo), E1 = __ldg(A.row_ptr + r_hi);
    const int ntiles = int((E1 - E0 + NT - 1) / NT);
    const int nnz_cta = int(E1 - E0);

    if (warp >= MMA_WARP + 1) {
        // ------------------------------------------------ producer: s_e = x_u + x_v -> B operand
        // Three-stage software pipeline per lane (cp.async groups, one per tile):
        //   tile t + 2*LA: this lane's neighbour indices -> S.idx (4-byte cp.async);
        //   tile t + LA  : destination rows of its edges (window search below), then
        //                  x_u (and, for tiles that span rows, x_v) -> S.raw_u / S.raw_v
        //                  (16-byte cp.async, zero-filled beyond d_in);
        //   tile t       : s = x_u + x_v, split, stored into the B operand.
        // Every lane reads back only what it copied itself, so a per-thread
        // cp.async.wait_group is the only synchronisation; no register waits on a
        // gather round trip (the first register-loaded version ran at 5.6 ms vs 4.0).
        // Fast path (most tiles of long rows): all of a warp's edges of the tile lie
        // in one row -- found with two ballots -- whose x_v stays in registers.
        constexpr int EPT = NT / (NPROD * 32);          // edge slots per lane per tile
        constexpr int LA = Smem<KS>::LA;
        const int pw = warp - (MMA_WARP + 1);           // producer warp 0 .. NPROD-1
        const int pt = tid - (MMA_WARP + 1) * 32;       // 0 .. NPROD*32-1
        const bool vec = (A.d_in % 4) == 0;
        // destination rows: a window of 32 consecutive rows [wb, wb + 32) whose
        // ends (relative to E0) lane j holds in wend; rows >= r_hi end at INT_MAX
        int wb = int(r_lo);
        auto load_window = [&](int base) {
            const int64_t rr = int64_t(base) + lane;
            return rr < r_hi ? int(__ldg(A.row_ptr + rr + 1) - E0) : 0x7fffffff;
        };
        int wend = load_window(wb);
        auto issue_idx = [&](int t) {
            if (t >= ntiles) return;
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int e = pt + i * NPROD * 32;
                const int64_t p = E0 + int64_t(t) * NT + e;
                cp_async4(smem_u32(&S.idx[t % (2 * LA)][e]), A.col_idx + (p < E1 ? p : E0), p < E1 ? 4 : 0);
            }
        };
        auto copy_row = [&](float* dst, const float* src, bool l1) {
#pragma unroll
            for (int k0 = 0; k0 < KS * 8; k0 += 4) {
                if (vec) {
                    const int nb = k0 < A.d_in ? 16 : 0;   // zero-fill beyond d_in
                    cp_async16_zfill(smem_u32(dst + k0), src + (nb ? k0 : 0), nb, l1);
                } else {
#pragma unroll
                    for (int k = k0; k < k0 + 4; ++k) {
                        const int nb = k < A.d_in ? 4 : 0;
                        cp_async4(smem_u32(dst + k), src + (nb ? k : 0), nb);
                    }
                }
            }
        };
        auto issue_raw = [&](int t) {
            if (t >= ntiles) return;
            const int slot = t % LA;
            // this warp's edges of tile t: pe = t*NT + pw*32 + lane + i*NPROD*32
            const int pfirst = t * NT + pw * 32;
            const int plast = min(t * NT + pw * 32 + (EPT - 1) * NPROD * 32 + 31, nnz_cta - 1);
            int c0 = __popc(__ballot_sync(0xffffffffu, wend <= pfirst));
            while (c0 == 32) {   // the window ends before this tile: slide it
                wb += 32;
                wend = load_window(wb);
                c0 = __popc(__ballot_sync(0xffffffffu, wend <= pfirst));
            }
            const int c1 = __popc(__ballot_sync(0xffffffffu, wend <= plast));
            int vrow[EPT];
            int tag = -1;
            if (c1 == c0) {
                tag = wb + c0;                     // every edge of this warp's tile lies in row wb + c0
#pragma unroll
                for (int i = 0; i < EPT; ++i) vrow[i] = tag;
            } else {
                bool done[EPT];
#pragma unroll
                for (int i = 0; i < EPT; ++i) {
                    vrow[i] = int(r_hi) - 1;       // padded slots: the CTA's last row
                    done[i] = t * NT + pt + i * NPROD * 32 >= nnz_cta;
                }
                for (;;) {
                    const int last = __shfl_sync(0xffffffffu, wend, 31);
#pragma unroll
                    for (int i = 0; i < EPT; ++i) {
                        const int pe = t * NT + pt + i * NPROD * 32;
                        int lo = 0;   // number of window rows ending at or before pe (ends ascend)
#pragma unroll
                        for (int step = 16; step >= 1; step >>= 1)
                            if (__shfl_sync(0xffffffffu, wend, lo + step - 1) <= pe) lo += step;
                        if (!done[i] && pe < last) {
                            vrow[i] = wb + lo;
                            done[i] = true;
                        }
                    }
                    bool all = true;
#pragma unroll
                    for (int i = 0; i < EPT; ++i) all = all && done[i];
                    if (__all_sync(0xffffffffu, all)) break;
                    wb += 32;   // some edge lies beyond the window: slide it
                    wend = load_window(wb);
                }
            }
            if (lane == 0) S.rowtag[pw][slot] = tag;
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int e = pt + i * NPROD * 32;
                copy_row(S.raw_u[slot][e], A.X + int64_t(S.idx[t % (2 * LA)][e]) * A.d_in, false);
                if (tag < 0) copy_row(S.raw_v[slot][e], A.Xd + int64_t(vrow[i]) * A.d_in, true);
            }
            // keep the window at the row of this tile's last edge (rows only move forward)
            const int wlast = __shfl_sync(0xffffffffu, vrow[EPT - 1], 31);
            if (wlast >= wb + 32 - 1 && wlast < r_hi) {   // the next tile starts at or beyond the window's end
                wb = wlast;
                wend = load_window(wb);
            }
        };
        // x_v of the fast path's row, in registers (reloaded when the row changes)
        int xrow = -1;
        float4 xv[KS][2];
        auto load_xv = [&](int row) {
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int k0 = ks * 8 + c * 4;
                    const float* p = A.Xd + int64_t(row) * A.d_in + k0;
                    if (vec) {
                        xv[ks][c] = k0 < A.d_in ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
                    } else {
                        xv[ks][c] = make_float4(k0 < A.d_in ? __ldg(p) : 0.f, k0 + 1 < A.d_in ? __ldg(p + 1) : 0.f,
                                                k0 + 2 < A.d_in ? __ldg(p + 2) : 0.f, k0 + 3 < A.d_in ? __ldg(p + 3) : 0.f);
                    }
                }
            xrow = row;
        };
        // prologue: indices of tiles 0 .. LA-1 (waited for), then group j = {x rows of
        // tile j, indices of tile j + LA} for j < LA
        for (int j = 0; j < LA; ++j) issue_idx(j);
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
        for (int j = 0; j < LA; ++j) {
            issue_raw(j);
            issue_idx(j + LA);
            cp_async_commit();
        }
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % STAGES;
            const int slot = t % LA;
            cp_async_wait_group<LA - 1>();   // group t: x rows of tile t, indices of tile t + LA
            __syncwarp();
            const int tag = S.rowtag[pw][slot];
            if (tag >= 0 && tag != xrow) load_xv(tag);
            mbar_wait_backoff(&S.empty[s], ((t / STAGES) & 1) ^ 1, BACKOFF_NS);
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int e = pt + i * NPROD * 32;
                const float4* ru = reinterpret_cast<const float4*>(S.raw_u[slot][e]);
                const float4* rv = reinterpret_cast<const float4*>(S.raw_v[slot][e]);
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const float4 a0 = ru[2 * ks], a1 = ru[2 * ks + 1];
                    const float4 b0 = tag >= 0 ? xv[ks][0] : rv[2 * ks];
                    const float4 b1 = tag >= 0 ? xv[ks][1] : rv[2 * ks + 1];
                    store_split<BF>(smem_u32(S.b_hi[s][ks]), smem_u32(S.b_lo[s][ks]), e,
                                    make_float4(a0.x + b0.x, a0.y + b0.y, a0.z + b0.z, a0.w + b0.w),
                                    make_float4(a1.x + b1.x, a1.y + b1.y, a1.z + b1.z, a1.w + b1.w));
                }
            }
            fence_async_smem();        // generic-proxy stores -> tensor-core (async proxy) reads
            mbar_arrive(&S.full[s]);
            __syncwarp();              // every lane has read S.rowtag[pw][slot] before it is rewritten
            issue_raw(t + LA);         // into the slot just consumed
            issue_idx(t + 2 * LA);
            cp_async_commit();
        }
        cp_async_wait_all();
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % STAGES, b = t % NBUF;
                mbar_wait_backoff(&S.full[s], (t / STAGES) & 1, BACKOFF_NS);
                fence_async_smem();
                mbar_wait_backoff(&S.tempty[b], ((t / NBUF) & 1) ^ 1, BACKOFF_NS);
                tc_fence_after();
                const uint32_t d = tmem + uint32_t(b * NT);
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const uint64_t ah = smem_desc(smem_u32(S.a_hi[ks])), al = smem_desc(smem_u32(S.a_lo[ks]));
                    const uint64_t bh = smem_desc(smem_u32(S.b_hi[s][ks])), bl = smem_desc(smem_u32(S.b_lo[s][ks]));
                    if constexpr (!BF) {
                        mma_tf32(d, ah, bh, ks > 0 ? 1u : 0u);
                        mma_tf32(d, ah, bl, 1u);
                        mma_tf32(d, al, bh, 1u);
                    } else {
                        mma_bf16(d, ah, bh, ks > 0 ? 1u : 0u);   // s_hi (w_hi + w_lo)
                        mma_bf16(d, ah, bl, 1u);                 // s_lo (w_hi + w_lo)
                    }
                }
                mma_commit(&S.empty[s]);
                mma_commit(&S.tfull[b]);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue: thread = feature
        Epi<MAX> ep;
        ep.A = &A;
        ep.i = mbase + tid;
        ep.active = ep.i < A.d2;
        ep.r = int(r_lo);
        ep.r_hi = int(r_hi);
        ep.E0 = E0;
        ep.rs = ep.re = 0;
        if (r_lo < r_hi) {
            ep.prefetch(int(r_lo));
            ep.re = ep.nre;   // row_ptr[r_lo] == E0, so row r_lo spans [0, nre)
            ep.start_row();
        }
        // TMEM address of this warp's lane quarter; opaque so that it stays in a
        // register instead of being rematerialised from %tid every chunk
        uint32_t lane_base;
        asm volatile("mov.b32 %0, %1;" : "=r"(lane_base) : "r"(tmem + (uint32_t(warp * 32) << 16)));
        // a warp whose 32 features all lie beyond d2 (d2 < 128: the W^T rows are
        // zero padding) only keeps the TMEM buffers cycling: no tcgen05.ld -- the
        // TMEM reads are this kernel's bound
        const bool warp_active = mbase + warp * 32 < A.d2;
        if (!warp_active) {
            for (int t = 0; t < ntiles; ++t) {
                const int b = t % NBUF;
                mbar_wait_backoff(&S.tfull[b], (t / NBUF) & 1, BACKOFF_NS);
                tc_fence_after();
                tc_fence_before();
                mbar_arrive(&S.tempty[b]);
            }
        }
        for (int t = 0; warp_active && t < ntiles; ++t) {
            const int b = t % NBUF;
            mbar_wait(&S.tfull[b], (t / NBUF) & 1);
            tc_fence_after();
            const int tb = t * NT;                       // relative to E0
            const int nv_tile = min(NT, nnz_cta - tb);
            // one 32-column chunk per tcgen05.ld (loading both chunks of the tile at once
            // needs 3 CTAs/SM for the registers and measured slower: 4.29 vs 4.07 ms)
            // max: 16-column chunks, software-pipelined -- chunk ch + 1 is read out of TMEM
            // while chunk ch is consumed (same 32 registers as one 32-column chunk):
            // reddit max + args 4.73 -> 4.35 ms, rand-100K 1.92 -> 1.75 ms; sum: one
            // 32-column chunk at a time (pipelined 3.20 -> 3.28 ms)
            constexpr bool LD16 = FG_MLP_LDW == 16 || (FG_MLP_LDW == 0 && MAX);
            if constexpr (LD16) {
                uint32_t va[16], vb[16];
                const uint32_t ta = lane_base + uint32_t(b * NT);
                tmem_ld16(ta, va);
                tmem_wait_ld2(va, vb);
#pragma unroll
                for (int ch = 0; ch < NT / 16; ch += 2) {
                    if (ch + 1 < NT / 16) tmem_ld16(ta + uint32_t((ch + 1) * 16), vb);
                    ep.consume<16>(va, tb + ch * 16, max(0, min(16, nv_tile - ch * 16)));
                    tmem_wait_ld2(vb, va);
                    if (ch + 2 < NT / 16) tmem_ld16(ta + uint32_t((ch + 2) * 16), va);
                    ep.consume<16>(vb, tb + (ch + 1) * 16, max(0, min(16, nv_tile - (ch + 1) * 16)));
                    tmem_wait_ld2(va, vb);
                }
            } else {
#pragma unroll 1
                for (int ch = 0; ch < NT / 32; ++ch) {
                    uint32_t v0[32];
                    tmem_ld32(lane_base + uint32_t(b * NT + ch * 32), v0);
                    tmem_wait_ld(v0);
                    ep.consume<32>(v0, tb + ch * 32, max(0, min(32, nv_tile - ch * 32)));
                }
            }
            tc_fence_before();
            mbar_arrive(&S.tempty[b]);
        }
        if (warp_active)
            while (ep.r < ep.r_hi) ep.advance();   // trailing rows (empty rows after the last edge)
    }
    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

template <int KS, bool MAX, bool BF>
fg_status launch_ks(const Args& A, cudaStream_t st) {
    const int smem = int(sizeof(Smem<KS>)) + 1024;
    const int smem_min = 56 * 1024;                              // bounds residency (TMEM columns)
    const int smem_req = smem < smem_min ? smem_min : smem;
    auto kfn = mlp_tcgen05_kernel<KS, MAX, BF>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_req);
    // the whole unified L1/smem for shared memory: without it the driver picks a
    // carveout that fits ONE 100 KB CTA per SM and the persistent grid runs as two waves
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return fgk::set_error(FG_ECUDA, "mlp_tcgen05: smem attribute: %s", cudaGetErrorString(e));
    int nb = CTAS_PER_SM * fgk::num_sms();
    const int64_t want = (A.nnz + 4 * NT - 1) / (4 * NT);   // >= 4 tiles per CTA
    if (want < nb) nb = int(want < 1 ? 1 : want);
    const dim3 grid{unsigned(nb), unsigned((A.d2 + MT - 1) / MT), 1u};
    kfn<<<grid, THREADS, smem_req, st>>>(A);
    return fgk::check_launch("mlp_tcgen05_kernel");
}

template <int KS, bool BF>
fg_status launch_red(const Args& A, bool mx, cudaStream_t st) {
    return mx ? launch_ks<KS, true, BF>(A, st) : launch_ks<KS, false, BF>(A, st);
}

}  // namespace

namespace fgk {

fg_status launch_spmm_mlp_tcgen05(const fg_graph* g, fg_reduce_op red, int d2, const float* X, const float* W,
                                  int d_in, const float* X_dst, float* out, int32_t* arg_u, int32_t* arg_e,
                                  bool bf16_split, cudaStream_t st) {
    Args A;
    A.n_src = g->n_src;
    A.row_ptr = g->row_ptr;
    A.col_idx = g->col_idx;
    A.eid = g->eid;
    A.X = X;
    A.Xd = X_dst;
    A.W = W;
    A.out = out;
    A.arg_u = arg_u;
    A.arg_e = arg_e;
    A.n_dst = g->n_dst;
    A.nnz = g->nnz;
    A.d_in = d_in;
    A.d2 = d2;
    const bool mx = red == FG_REDUCE_MAX;
    const int ks = (d_in + 7) / 8;
    if (bf16_split) {
        switch (ks) {
            case 1: return launch_red<1, true>(A, mx, st);
            case 2: return launch_red<2, true>(A, mx, st);
            case 3: return launch_red<3, true>(A, mx, st);
            default: return launch_red<4, true>(A, mx, st);
        }
    }
    switch (ks) {
        case 1: return launch_red<1, false>(A, mx, st);
        case 2: return launch_red<2, false>(A, mx, st);
        case 3: return launch_red<3, false>(A, mx, st);
        default: return launch_red<4, false>(A, mx, st);
    }
}

}  // namespace fgk
