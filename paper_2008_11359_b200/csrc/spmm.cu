// spmm.cu -- gSpMM with gathered messages: copy_u and u_mul_e x {sum, max}
// (SURVEY §8(a) rows a1, a2), plus the min / mean reducers and the u_add_e /
// copy_e messages (row f4).  The kernel template lives in spmm_impl.cuh and is
// instantiated per (reducer, op set) in spmm_inst_*.cu; this file holds the
// host-side launch configuration.
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
//     before the compare, matching the oracle's fp32-rounded key; min is the
//     same with the comparison reversed; mean divides the fp32 sum by the
//     in-degree once in the epilogue.
#include <algorithm>
#include <cstdlib>

#include "spmm_impl.cuh"


namespace fgk {

fg_status launch_spmm_gather(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D, const float* X,
                             const float* E, float* out, int32_t* arg_u, int32_t* arg_e, cudaStream_t st,
                             const uint16_t* Xbf16) {
    using namespace fgspmm;
    Args A;
    A.rows = g->rows_by_deg;
    A.n_rows = g->n_dst;
    A.row_ptr = g->row_ptr;
    A.col_idx = g->col_idx;
    A.eid = g->eid;
    A.X = reinterpret_cast<const float4*>(X);
    A.Xh = reinterpret_cast<const uint2*>(Xbf16);
    const int64_t chunk_bytes = Xbf16 ? 8 : 16;   // bytes of X per 4-feature chunk
    A.E = E;
    A.H = H;
    A.D = D;
    A.F4 = H * D / 4;
    A.out = reinterpret_cast<float4*>(out);
    A.arg_u = reinterpret_cast<int4*>(arg_u);
    A.arg_e = reinterpret_cast<int4*>(arg_e);
    A.hyb_code = nullptr;
    A.hyb_hot = nullptr;
    A.hyb_k = 0;
    A.n_vblocks = 0;
    A.seg_lo = A.seg_hi = nullptr;
    A.seg_acc = 0;
    const int op = (msg == FG_MSG_COPY_U)    ? OP_COPY
                   : (msg == FG_MSG_U_ADD_E) ? OP_UADDE
                   : (msg == FG_MSG_COPY_E)  ? OP_COPYE
                                             : (D % 4 == 0 ? OP_UMULE : OP_UMULE_GEN);
    const int mx = (red == FG_REDUCE_MAX) ? R_MAX : (red == FG_REDUCE_MIN) ? R_MIN : (red == FG_REDUCE_MEAN) ? R_MEAN : R_SUM;
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
        const int64_t budget = fgk::l2_tile_budget(g, red == FG_REDUCE_MAX || red == FG_REDUCE_MIN);
        // copy_u only: u_mul_e re-reads E (m x H floats) on every pass, measured slower
        // at every budget (reddit H=8 D=32: 9.1-10.1 ms untiled vs 12.2-43.6 ms tiled)
        if (msg == FG_MSG_COPY_U && budget > 0 && g->n_src * int64_t(F4) * chunk_bytes > budget) {
            int64_t t4 = 32;
            while (t4 > 1 && g->n_src * t4 * chunk_bytes > budget) t4 /= 2;
            F4 = int(t4);            // tile width drives (G, NV) below; the kernel tiles A.F4 by G*NV
        }
    }
    // one float4 per lane up to 32 lanes, then 2-4 float4 per lane (measured: wider
    // lanes -- G x 4 float4 at every width -- were 1.3-3x slower on reddit at
    // F = 32..512: fewer lanes per row exposes more gather latency per row)
    if (F4 <= 32) {
        NV = 1;
        G = 1;
        while (G < F4) G *= 2;
    } else if (F4 <= 64) {
        NV = 2;
    } else if (F4 <= 96) {
        NV = 3;
    }
    // bf16 storage with an even number of 4-feature chunks per (tile) row and a
    // 16-byte aligned X: lanes read PAIRS of chunks (8 features) with one 16-byte
    // load -- half the load instructions of the 8-byte-per-chunk mapping
    const bool pair = Xbf16 && A.F4 % 2 == 0 && F4 % 2 == 0 && (reinterpret_cast<uintptr_t>(Xbf16) & 15u) == 0;
    // fp32 copy_u with an even number of 4-feature chunks per (tile) row and a
    // 32-byte aligned X: lanes read chunk PAIRS with one 32-byte load (LDG.256) --
    // half the load and address instructions per gathered byte (FG_TUNE_SPMM_LDG256)
    const bool pair32 = !Xbf16 && g->tune.spmm_ldg256 && op == OP_COPY && A.F4 % 2 == 0 && F4 % 2 == 0 &&
                        (reinterpret_cast<uintptr_t>(X) & 31u) == 0;
    if (pair || pair32) {
        const int F8 = F4 / 2;
        NV = 2;
        if (F8 <= 32) {
            G = 1;
            while (G < F8) G *= 2;
        } else {
            G = 32;
            NV = 4;   // 128 float4 columns per tile; wider rows take several tiles (grid.y)
        }
    }
    {   // rows with degree >= the heavy threshold run CTA-per-row.  Threshold = the fair
        // share of edges per group in flight, m / (SMs x 2048 / G), clamped to
        // [1024, 4096] (FG_SPMM_HEAVY_DEG overrides).  Measured on reddit: a constant
        // NG x 32 = 256..1024 cost copy_u-sum F=512 14.1 vs 12.5 ms, u_mul_e H=8 9.4 vs
        // 7.8 ms (a group per long row keeps more gathers in flight than a CTA per
        // row); a constant 4096 cost the short F = 32 kernels their tail (rand-100K
        // 0.37 -> 0.52 ms: a 4,000-edge row on one 8-lane group outlasts the rest).
        // The edge count is FG_TUNE_BALANCE_NNZ when set: the sharding code sets the
        // whole graph's, so every shard splits rows exactly as the unsharded op.
        int64_t thr;
        if (g->tune.spmm_heavy_deg > 0) {
            thr = g->tune.spmm_heavy_deg;
        } else {
            const int64_t groups = int64_t(fgk::num_sms()) * (2048 / G);
            const int64_t m = g->tune.balance_nnz > 0 ? g->tune.balance_nnz : g->nnz;
            thr = std::min<int64_t>(4096, std::max<int64_t>(1024, m / std::max<int64_t>(1, groups)));
        }
        A.n_heavy = rows_with_degree_at_least(g, thr);
    }
    // hybrid partitioning (FG_TUNE_HYBRID, table from fg_graph_prepare_hybrid for
    // this row width): copy_u-sum with one float4 per lane and no column tiling
    if (g->tune.hybrid && g->hyb.code && g->hyb.k > 0 && msg == FG_MSG_COPY_U && red == FG_REDUCE_SUM &&
        !Xbf16 && NV == 1 && F4 == A.F4 && g->hyb.row_bytes == int64_t(A.F4) * 16) {
        A.hyb_code = g->hyb.code;
        A.hyb_hot = g->hyb.hot;
        A.hyb_k = int(g->hyb.k);
        return launch_hybrid(A, G, st);
    }
    // source-segmented u_mul_e-sum (the paper's 1D source partitioning, P:462-465,
    // with L2-sized segments; bounds from fg_graph_prepare for this row width):
    // one pass per segment in segment order, each gathering only from its
    // L2-resident X slice and adding onto out.  Column tiling does not apply to
    // u_mul_e (every tile would re-read E); segmenting reads E and col_idx once
    // and re-reads only out (2 x n x F x 4 bytes per extra pass).
    if (op == OP_UMULE && mx == R_SUM && !Xbf16 && F4 == A.F4) {
        const int64_t seg_rows = fgk::spmm_seg_rows(g, int64_t(A.F4) * 16);
        const fg_graph::SegBounds* sb = seg_rows ? fgk::find_seg_bounds(g, seg_rows) : nullptr;
        if (sb) {
            for (int s = 0; s < sb->nseg; ++s) {
                A.seg_lo = sb->bnd + int64_t(s) * g->n_dst;
                A.seg_hi = sb->bnd + int64_t(s + 1) * g->n_dst;
                A.seg_acc = s > 0;
                const fg_status r = launch_seg_pass(A, G, NV, st);
                if (r != FG_OK) return r;
            }
            return FG_OK;
        }
    }
    const int opset = (op == OP_UADDE || op == OP_COPYE) ? 1 : 0;
    if (pair32) {
        switch (mx) {
            case R_MAX: return dispatch_pair32<R_MAX>(A, G, NV, op, st);
            case R_MIN: return dispatch_pair32<R_MIN>(A, G, NV, op, st);
            case R_MEAN: return dispatch_pair32<R_MEAN>(A, G, NV, op, st);
            default: return dispatch_pair32<R_SUM>(A, G, NV, op, st);
        }
    }
    if (Xbf16) {   // bf16 storage: copy_u / u_mul_e x {sum, max, min, mean} (validated by the caller)
        if (mx == R_MAX) return dispatch_x16<R_MAX>(A, G, NV, op, pair, st);
        if (mx == R_MIN) return dispatch_x16<R_MIN>(A, G, NV, op, pair, st);
        if (mx == R_MEAN) return dispatch_x16<R_MEAN>(A, G, NV, op, pair, st);
        return dispatch_x16<R_SUM>(A, G, NV, op, pair, st);
    }
    switch (mx) {
        case R_MAX: return opset ? dispatch_inst<R_MAX, 1>(A, G, NV, op, st) : dispatch_inst<R_MAX, 0>(A, G, NV, op, st);
        case R_MIN: return opset ? dispatch_inst<R_MIN, 1>(A, G, NV, op, st) : dispatch_inst<R_MIN, 0>(A, G, NV, op, st);
        case R_MEAN: return opset ? dispatch_inst<R_MEAN, 1>(A, G, NV, op, st) : dispatch_inst<R_MEAN, 0>(A, G, NV, op, st);
        default: return opset ? dispatch_inst<R_SUM, 1>(A, G, NV, op, st) : dispatch_inst<R_SUM, 0>(A, G, NV, op, st);
    }
}

}  // namespace fgk
