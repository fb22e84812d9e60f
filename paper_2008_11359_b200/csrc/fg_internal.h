// fg_internal.h -- shared internals of libfg.so (NOT part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <deque>
#include <mutex>
#include <vector>

#include "../../include/fg.h"

// Launch-configuration knobs of one handle (the internal "FDS"):
// defaults are the values measured on reddit / proteins / rand-100K (DESIGN.md
// §6, §9).  Read ONCE, at fg_graph_create, from the FG_* environment variables
// (developer overrides), and settable per handle with fg_graph_tune (include/
// fg.h); the launch paths never read the environment.
struct fg_tuning {
    int64_t l2_tile_mb = -1;        // copy_u column-tile budget; -1: 32 MB (max/min) / 64 MB (sum/mean); 0: off
    int64_t spmm_heavy_deg = 0;     // CTA-per-row threshold of the gathered gSpMM; 0: automatic
    int64_t balance_nnz = 0;        // edge count of the automatic threshold; 0: this handle's nnz
    int64_t sddmm_seg_mb = 48;      // source-segment size of the segmented gSDDMM (0: off)
    int64_t sddmm_seg_min_mb = 96;  // segment only when X is wider than this
    int64_t sddmm_persist = -1;     // CTAs/SM of the persistent segmented launch (-1: occupancy)
    int64_t sddmm_l2_tile = 0;      // 1: column-tiled gSDDMM passes (measured slower; ablation)
    int64_t sddmm_dot = 0;          // 0: lanes over features + shuffle reduction; 1: thread per edge (E6 ablation)
    int64_t gat_heavy_deg = 4096;   // CTA-per-row threshold of the fused GAT
    int64_t mlp_impl = 0;           // 0: tcgen05 3xTF32, 1: CUDA-core FFMA, 2: tcgen05 bf16 2-split (K = 32)
    int64_t hybrid = 0;             // 1: hot sources staged in shared memory (needs fg_graph_prepare_hybrid)
    int64_t sddmm_pipe = -1;        // H == 1 wide-row gSDDMM: 0 plain, 1..3 software-pipelined variants, -1 auto
    int64_t sddmm_order = 0;        // segmented gSDDMM unit order: 0 segment-major, 1 Hilbert over (row block, segment)
    int64_t sddmm_rb_mb = 0;        // Hilbert order: destination-block size in MB of Y rows (0: = sddmm_seg_mb)
    int64_t spmm_ldg256 = 0;        // 1: fp32 copy_u gathers as 32-byte chunk-pair loads (measured slower)
    int64_t spmm_seg_mb = 0;        // source-segment size of the segmented u_mul_e-sum passes (0: off;
                                    // measured slower); only when X > sddmm_seg_min_mb
};

struct fg_graph {
    int64_t n_dst = 0, n_src = 0, nnz = 0;
    fg_tuning tune;
    const int64_t* row_ptr = nullptr;   // borrowed, device
    const int32_t* col_idx = nullptr;   // borrowed, device
    const int32_t* eid = nullptr;       // borrowed, device (nullptr = identity)
    int device = 0;
    // set only for handles made by fg_graph_transpose (the library owns their CSR)
    int64_t* owned_row_ptr = nullptr;
    int32_t* owned_col_idx = nullptr;
    int32_t* owned_eid = nullptr;

    // derived (owned, device)
    int32_t* rows_by_deg = nullptr;     // [n_dst] rows sorted by degree, descending (stable)
    int32_t* unit_row = nullptr;        // [n_units] SDDMM work units: (row, first edge)
    int64_t* unit_p0 = nullptr;
    int64_t n_units = 0;
    int unit_chunk = 0;                 // edges per SDDMM unit

    // source-segmented SDDMM unit tables (1D source partitioning retargeted to the
    // L2): built by fg_graph_prepare (synchronous) per segment width;
    // the launch paths only look them up (no allocation, no synchronisation)
    struct SegUnits {
        int64_t seg_rows = 0, rb_rows = 0, n_units = 0;   // rb_rows > 0: Hilbert-ordered 2D tiles
        int32_t* row = nullptr;
        int64_t* p0 = nullptr;
        int64_t* p1 = nullptr;
    };
    std::deque<SegUnits> seg_units;      // deque: references stay valid as it grows
    // source-segmented gSpMM passes (u_mul_e-sum; same 1D source partitioning):
    // bnd[s * n_dst + v] = first CSR position of row v whose source is >= s * seg_rows,
    // s = 0..nseg (bnd[0] = row_ptr[v], bnd[nseg] = row_ptr[v + 1]); fg_graph_prepare
    struct SegBounds {
        int64_t seg_rows = 0;
        int nseg = 0;
        int64_t* bnd = nullptr;   // [(nseg + 1) * n_dst]
    };
    std::deque<SegBounds> seg_bounds;
    std::mutex seg_mu;                   // guards seg_units against concurrent fg_graph_prepare calls

    // hybrid partitioning table (fg_graph_prepare_hybrid): per-edge
    // source codes (u, or -(slot+1) when source u is staged in shared memory)
    // and the staged sources -- the hyb_k of highest out-degree
    struct Hybrid {
        int64_t row_bytes = 0, k = 0;
        int32_t* code = nullptr;   // [nnz]
        int32_t* hot = nullptr;    // [k]
        double hot_edge_share = 0; // fraction of edges whose source is staged
    } hyb;

    // derived (owned, host)
    std::vector<int64_t> deg_sorted;    // degrees in rows_by_deg order (descending)
    int64_t n_nonempty = 0;
    int64_t max_deg = 0;
    int64_t device_bytes = 0;
};

namespace fgk {

// FG_* environment overrides of fg_tuning (fg_graph_create / fg_graph_transpose only)
void tuning_from_env(fg_tuning* t);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// host-side argument checks of fg_spmm / fg_sddmm (api.cu)
fg_status check_spmm(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D, const float* X,
                     const float* E, const float* W, int d_in, const float* X_dst, const float* out,
                     const int32_t* arg_u, const int32_t* arg_e);
fg_status check_sddmm(const fg_graph* g, fg_edge_op op, int H, int D, const float* X, const float* Y,
                      const float* out);

// thread-local error detail
fg_status set_error(fg_status s, const char* fmt, ...);

// number of rows in the degree-sorted list with degree >= t
int64_t rows_with_degree_at_least(const fg_graph* g, int64_t t);

// kernels launchers (return FG_OK or FG_ECUDA); arguments already validated
fg_status launch_spmm_gather(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D,
                             const float* X, const float* E, float* out, int32_t* arg_u,
                             int32_t* arg_e, cudaStream_t st, const uint16_t* Xbf16 = nullptr);
fg_status launch_spmm_mlp(const fg_graph* g, fg_reduce_op red, int d2, const float* X,
                          const float* W, int d_in, const float* X_dst, float* out,
                          int32_t* arg_u, int32_t* arg_e, cudaStream_t st);
fg_status launch_spmm_mlp_tcgen05(const fg_graph* g, fg_reduce_op red, int d2, const float* X, const float* W,
                                  int d_in, const float* X_dst, float* out, int32_t* arg_u, int32_t* arg_e,
                                  bool bf16_split, cudaStream_t st);
fg_status launch_spmm_mlp_simt(const fg_graph* g, fg_reduce_op red, int d2, const float* X, const float* W,
                               int d_in, const float* X_dst, float* out, int32_t* arg_u, int32_t* arg_e,
                               cudaStream_t st);
fg_status launch_sddmm(const fg_graph* g, int H, int D, const float* X, const float* Y, float* out,
                       cudaStream_t st, const uint16_t* Xbf16 = nullptr, const uint16_t* Ybf16 = nullptr,
                       const float* E = nullptr);
fg_status launch_sddmm_binary(const fg_graph* g, int op, int F, const float* X, const float* Y, float* out,
                              cudaStream_t st);
fg_status launch_edge_softmax(const fg_graph* g, int H, const float* S, float* out, cudaStream_t st);

fg_status check_launch(const char* what);

// source-segmented unit table for segments of seg_rows source vertices:
// build_seg_units (fg_graph_prepare: allocates, synchronises) and find_seg_units
// (launch paths: lookup only, NULL when not prepared)
fg_status build_seg_units(fg_graph* g, int64_t seg_rows, int64_t rb_rows, int chunk, cudaStream_t st);
const fg_graph::SegUnits* find_seg_units(const fg_graph* g, int64_t seg_rows, int64_t rb_rows);
// destination-block rows of the Hilbert-ordered unit table (0: segment-major order)
int64_t sddmm_rb_rows(const fg_graph* g, int64_t row_bytes);
// segment rows of the segmented gSDDMM for gathered rows of row_bytes, or 0 when
// the rule does not segment (X = n_src x row_bytes within the budget)
int64_t sddmm_seg_rows(const fg_graph* g, int64_t row_bytes);
// the same for the segmented u_mul_e-sum passes of gSpMM, and its bound tables
int64_t spmm_seg_rows(const fg_graph* g, int64_t row_bytes);
fg_status build_seg_bounds(fg_graph* g, int64_t seg_rows, cudaStream_t st);
const fg_graph::SegBounds* find_seg_bounds(const fg_graph* g, int64_t seg_rows);

// column-tile budget (bytes of the gathered operand per pass) of the copy_u
// gather, the paper's feature-dimension tiling retargeted to the L2.
// Defaults measured on reddit (one B200): select reducers (max / min + argmax)
// 32 MB (F=128 max + args 4.79 ms vs 5.46 at 64 MB), sum / mean 64 MB (F=512
// 13.4-13.6 ms vs 14.0-14.1 at 32 MB); 24 MB and below fall to 4-lane groups and lose.
inline int64_t l2_tile_budget(const fg_graph* g, bool select_reducer = false) {
    const int64_t mb = g->tune.l2_tile_mb >= 0 ? g->tune.l2_tile_mb : (select_reducer ? 32 : 64);
    return mb << 20;
}

inline int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

}  // namespace fgk
