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

struct fg_graph {
    int64_t n_dst = 0, n_src = 0, nnz = 0;
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
    // L2): built lazily per segment width, cached for the handle's life
    struct SegUnits {
        int64_t seg_rows = 0, n_units = 0;
        int32_t* row = nullptr;
        int64_t* p0 = nullptr;
        int64_t* p1 = nullptr;
    };
    std::deque<SegUnits> seg_units;      // deque: references stay valid as it grows
    std::mutex seg_mu;                   // lazily built under this lock (handle shared across streams)

    // derived (owned, host)
    std::vector<int64_t> deg_sorted;    // degrees in rows_by_deg order (descending)
    int64_t n_nonempty = 0;
    int64_t max_deg = 0;
    int64_t device_bytes = 0;
};

namespace fgk {

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
                          int32_t* arg_u, int32_t* arg_e, void* workspace, cudaStream_t st);
fg_status launch_spmm_mlp_tcgen05(const fg_graph* g, fg_reduce_op red, int d2, const float* X, const float* W,
                                  int d_in, const float* X_dst, float* out, int32_t* arg_u, int32_t* arg_e,
                                  void* workspace, cudaStream_t st);
size_t mlp_workspace_bytes(int64_t n_src, int64_t n_dst, int d_in, int d2);
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

// source-segmented unit table for segments of seg_rows source vertices (built on
// first use; the handle owns it)
fg_status get_seg_units(fg_graph* g, int64_t seg_rows, int chunk, cudaStream_t st, const fg_graph::SegUnits** out);

// column-tile budget (bytes of the gathered operand per pass) of the copy_u
// gather, the paper's feature-dimension tiling retargeted to the L2.
// FG_L2_TILE_MB overrides; 0 disables.  Defaults measured on reddit (one B200):
// select reducers (max / min + argmax) 32 MB (F=128 max + args 4.79 ms vs 5.46 at
// 64 MB), sum / mean 64 MB (F=512 13.4-13.6 ms vs 14.0-14.1 at 32 MB); 24 MB and
// below fall to 4-lane groups and lose.
inline int64_t l2_tile_budget(bool select_reducer = false) {
    const char* e = getenv("FG_L2_TILE_MB");
    return int64_t(e ? atoi(e) : (select_reducer ? 32 : 64)) << 20;
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
