// graph.cu -- fg_graph_create: per-topology preprocessing.
//
// The paper generates code per graph topology and amortises it over epochs
// (tuning < 1 % of 200 epochs) and balances load by
// degree (Gunrock-style thread/warp/block assignment P:178; hybrid degree-
// threshold split P:534-539).  The B200 analogue built here, once per graph:
//   * rows sorted by in-degree, descending (longest-processing-time-first
//     order for every row-parallel kernel; the degree bins of fg_spmm are
//     prefixes of this list, chosen per launch from the host copy of the
//     sorted degrees);
//   * the gSDDMM work-unit table: each row cut into chunks of <= unit_chunk
//     edges (SDDMM has no cross-edge reduction, so heavy rows split freely);
//   * optional validation of the CSR invariants on the device.
#include <algorithm>
#include <cstdio>
#include <numeric>
#include <utility>

#include "fg_internal.h"

namespace fgk {
// FG_* environment overrides of the launch knobs, read once per handle here (the
// launch paths read only g->tune); fg_graph_tune sets them explicitly.
void tuning_from_env(fg_tuning* t) {
    auto rd = [](const char* name, int64_t& v) {
        const char* e = getenv(name);
        if (e && *e) v = atoll(e);
    };
    rd("FG_L2_TILE_MB", t->l2_tile_mb);
    rd("FG_SPMM_HEAVY_DEG", t->spmm_heavy_deg);
    rd("FG_SDDMM_SEG_MB", t->sddmm_seg_mb);
    rd("FG_SDDMM_SEG_MIN_MB", t->sddmm_seg_min_mb);
    rd("FG_SDDMM_PERSIST", t->sddmm_persist);
    rd("FG_SDDMM_L2_TILE", t->sddmm_l2_tile);
    rd("FG_SDDMM_DOT", t->sddmm_dot);
    rd("FG_GAT_HEAVY_DEG", t->gat_heavy_deg);
    rd("FG_MLP_IMPL", t->mlp_impl);
    rd("FG_HYBRID", t->hybrid);
    rd("FG_SPMM_SEG_MB", t->spmm_seg_mb);
    rd("FG_SDDMM_PIPE", t->sddmm_pipe);
    rd("FG_SDDMM_ORDER", t->sddmm_order);
    rd("FG_SPMM_LDG256", t->spmm_ldg256);
    rd("FG_SDDMM_RB_MB", t->sddmm_rb_mb);
}
}  // namespace fgk

namespace {

// flags
constexpr unsigned BAD_ROWPTR = 1u, BAD_COL_RANGE = 2u, BAD_COL_ORDER = 4u, BAD_EID_RANGE = 8u,
                   BAD_EID_DUP = 16u;

// one warp per row: row_ptr monotone, col_idx in range and strictly ascending
__global__ void validate_rows(int64_t n_dst, int64_t n_src, int64_t nnz, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ ci, unsigned* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    unsigned f = 0;
    for (int64_t v = warp; v < n_dst; v += nwarps) {
        int64_t s = rp[v], e = rp[v + 1];
        if (s > e || s < 0 || e > nnz) { f |= BAD_ROWPTR; continue; }
        for (int64_t p = s + lane; p < e; p += 32) {
            int32_t c = ci[p];
            if (c < 0 || c >= n_src) f |= BAD_COL_RANGE;
            if (p + 1 < e && ci[p + 1] <= c) f |= BAD_COL_ORDER;
        }
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0 && f) atomicOr(flags, f);
}

__global__ void validate_eid(int64_t nnz, const int32_t* __restrict__ eid, unsigned* seen, unsigned* flags) {
    unsigned f = 0;
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
         p += int64_t(gridDim.x) * blockDim.x) {
        int32_t e = eid[p];
        if (e < 0 || e >= nnz) { f |= BAD_EID_RANGE; continue; }
        unsigned bit = 1u << (e & 31);
        unsigned old = atomicOr(&seen[e >> 5], bit);
        if (old & bit) f |= BAD_EID_DUP;
    }
    if (f) atomicOr(flags, f);
}

}  // namespace

__device__ __forceinline__ int64_t lb_row(const int32_t* __restrict__ ci, int64_t lo, int64_t hi, int64_t key) {
    while (lo < hi) {   // first position in [lo, hi) with ci >= key
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(ci + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// units per (segment, row): segment-major layout cnt[s * n + v]
__global__ void seg_count_kernel(int64_t n, int nseg, int64_t seg_rows, int chunk, const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci, int64_t* __restrict__ cnt) {
    const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int64_t s0 = rp[v], s1 = rp[v + 1];
    int64_t lo = s0;
    for (int s = 0; s < nseg; ++s) {
        const int64_t hi = (s == nseg - 1) ? s1 : lb_row(ci, lo, s1, (s + 1) * seg_rows);
        cnt[int64_t(s) * n + v] = (hi - lo + chunk - 1) / chunk;
        lo = hi;
    }
}

__global__ void seg_write_kernel(int64_t n, int nseg, int64_t seg_rows, int chunk, const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci, const int64_t* __restrict__ off,
                                 int32_t* __restrict__ urow, int64_t* __restrict__ up0, int64_t* __restrict__ up1) {
    const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int64_t s0 = rp[v], s1 = rp[v + 1];
    int64_t lo = s0;
    for (int s = 0; s < nseg; ++s) {
        const int64_t hi = (s == nseg - 1) ? s1 : lb_row(ci, lo, s1, (s + 1) * seg_rows);
        int64_t o = off[int64_t(s) * n + v];
        for (int64_t p = lo; p < hi; p += chunk, ++o) {
            urow[o] = int32_t(v);
            up0[o] = p;
            up1[o] = min(p + chunk, hi);
        }
        lo = hi;
    }
}

// bounds of the source-segmented gSpMM passes: bnd[s * n + v] for s = 0..nseg
__global__ void seg_bound_kernel(int64_t n, int nseg, int64_t seg_rows, const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci, int64_t* __restrict__ bnd) {
    const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int64_t s0 = rp[v], s1 = rp[v + 1];
    int64_t lo = s0;
    bnd[v] = s0;
    for (int s = 1; s < nseg; ++s) {
        lo = lb_row(ci, lo, s1, s * seg_rows);
        bnd[int64_t(s) * n + v] = lo;
    }
    bnd[int64_t(nseg) * n + v] = s1;
}

namespace fgk {
fg_status build_seg_bounds(fg_graph* g, int64_t seg_rows, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g->seg_mu);
    for (auto& sb : g->seg_bounds)
        if (sb.seg_rows == seg_rows) return FG_OK;
    const int64_t n = g->n_dst;
    fg_graph::SegBounds sb;
    sb.seg_rows = seg_rows;
    sb.nseg = int((g->n_src + seg_rows - 1) / seg_rows);
    cudaError_t e = cudaMalloc(&sb.bnd, sizeof(int64_t) * size_t(std::max<int64_t>(1, (sb.nseg + 1) * n)));
    if (e == cudaSuccess && n > 0) {
        seg_bound_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(n, sb.nseg, seg_rows, g->row_ptr, g->col_idx,
                                                                    sb.bnd);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFree(sb.bnd);
        return set_error(e == cudaErrorMemoryAllocation ? FG_ENOMEM : FG_ECUDA, "fg_graph_prepare: segment bounds: %s",
                         cudaGetErrorString(e));
    }
    g->device_bytes += 8 * (sb.nseg + 1) * n;
    g->seg_bounds.push_back(sb);
    return FG_OK;
}

const fg_graph::SegBounds* find_seg_bounds(const fg_graph* g, int64_t seg_rows) {
    std::lock_guard<std::mutex> lock(const_cast<fg_graph*>(g)->seg_mu);
    for (auto& sb : g->seg_bounds)
        if (sb.seg_rows == seg_rows) return &sb;
    return nullptr;
}

int64_t spmm_seg_rows(const fg_graph* g, int64_t row_bytes) {
    const int64_t budget = g->tune.spmm_seg_mb << 20;
    const int64_t min_x = g->tune.sddmm_seg_min_mb << 20;
    if (budget <= 0 || row_bytes <= 0 || g->n_src * row_bytes <= std::max(budget, min_x)) return 0;
    return std::max<int64_t>(32, budget / row_bytes);
}

// Hilbert index of cell (x, y) on an n x n grid (n a power of two)
static int64_t hilbert_d(int64_t n, int64_t x, int64_t y) {
    int64_t d = 0;
    for (int64_t s = n / 2; s > 0; s /= 2) {
        const int64_t rx = (x & s) > 0, ry = (y & s) > 0;
        d += s * s * ((3 * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) {
                x = n - 1 - x;
                y = n - 1 - y;
            }
            std::swap(x, y);
        }
    }
    return d;
}

fg_status build_seg_units(fg_graph* g, int64_t seg_rows, int64_t rb_rows, int chunk, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g->seg_mu);
    for (auto& su : g->seg_units)
        if (su.seg_rows == seg_rows && su.rb_rows == rb_rows) return FG_OK;
    const int64_t n = g->n_dst;
    const int nseg = int((g->n_src + seg_rows - 1) / seg_rows);
    fg_graph::SegUnits su;
    su.seg_rows = seg_rows;
    su.rb_rows = rb_rows;
    int64_t* cnt = nullptr;
    std::vector<int64_t> h(size_t(n) * nseg + 1, 0);
    cudaError_t e = cudaMalloc(&cnt, sizeof(int64_t) * (size_t(n) * nseg + 1));
    if (e == cudaSuccess && n > 0) {
        seg_count_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(n, nseg, seg_rows, chunk, g->row_ptr, g->col_idx, cnt);
        e = cudaMemcpyAsync(h.data(), cnt, sizeof(int64_t) * size_t(n) * nseg, cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
        // exclusive scan of the per-(segment, row) unit counts in traversal order:
        //   rb_rows == 0: segment-major (all units of segment 0 first, rows ascending);
        //   rb_rows > 0 : 2D tiles (row block of rb_rows destinations x source
        //                 segment) in Hilbert-curve order, rows
        //                 ascending inside a tile -- consecutive tiles share their
        //                 destination block (Y rows stay in L2) or their source
        //                 segment (X rows stay in L2)
        int64_t acc = 0;
        auto take = [&](int s, int64_t v0, int64_t v1) {
            for (int64_t v = v0; v < v1; ++v) {
                const size_t i = size_t(s) * size_t(n) + size_t(v);
                const int64_t c = h[i];
                h[i] = acc;
                acc += c;
            }
        };
        if (rb_rows <= 0) {
            for (int s = 0; s < nseg; ++s) take(s, 0, n);
        } else {
            const int64_t nrb = (n + rb_rows - 1) / rb_rows;
            int64_t side = 1;
            while (side < std::max<int64_t>(nrb, nseg)) side *= 2;
            std::vector<std::pair<int64_t, int64_t>> tiles;   // (hilbert index, b * nseg + s)
            for (int64_t b = 0; b < nrb; ++b)
                for (int64_t sg = 0; sg < nseg; ++sg) tiles.emplace_back(hilbert_d(side, b, sg), b * nseg + sg);
            std::sort(tiles.begin(), tiles.end());
            for (auto& t : tiles) {
                const int64_t b = t.second / nseg;
                const int sg = int(t.second % nseg);
                take(sg, b * rb_rows, std::min(n, (b + 1) * rb_rows));
            }
        }
        su.n_units = acc;
        e = cudaMemcpyAsync(cnt, h.data(), sizeof(int64_t) * size_t(n) * nseg, cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess) e = cudaMalloc(&su.row, sizeof(int32_t) * size_t(std::max<int64_t>(su.n_units, 1)));
    if (e == cudaSuccess) e = cudaMalloc(&su.p0, sizeof(int64_t) * size_t(std::max<int64_t>(su.n_units, 1)));
    if (e == cudaSuccess) e = cudaMalloc(&su.p1, sizeof(int64_t) * size_t(std::max<int64_t>(su.n_units, 1)));
    if (e == cudaSuccess && n > 0) {
        seg_write_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(n, nseg, seg_rows, chunk, g->row_ptr, g->col_idx,
                                                                    cnt, su.row, su.p0, su.p1);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(cnt);
    if (e != cudaSuccess) {
        cudaFree(su.row); cudaFree(su.p0); cudaFree(su.p1);
        return set_error(e == cudaErrorMemoryAllocation ? FG_ENOMEM : FG_ECUDA, "fg_graph_prepare: segment units: %s",
                         cudaGetErrorString(e));
    }
    g->device_bytes += 20 * su.n_units;
    g->seg_units.push_back(su);
    return FG_OK;
}

const fg_graph::SegUnits* find_seg_units(const fg_graph* g, int64_t seg_rows, int64_t rb_rows) {
    std::lock_guard<std::mutex> lock(const_cast<fg_graph*>(g)->seg_mu);
    for (auto& su : g->seg_units)
        if (su.seg_rows == seg_rows && su.rb_rows == rb_rows) return &su;
    return nullptr;
}

int64_t sddmm_rb_rows(const fg_graph* g, int64_t row_bytes) {
    if (g->tune.sddmm_order != 1 || row_bytes <= 0) return 0;
    const int64_t mb = g->tune.sddmm_rb_mb > 0 ? g->tune.sddmm_rb_mb : g->tune.sddmm_seg_mb;
    return std::max<int64_t>(32, (mb << 20) / row_bytes);
}

int64_t sddmm_seg_rows(const fg_graph* g, int64_t row_bytes) {
    const int64_t budget = g->tune.sddmm_seg_mb << 20;
    const int64_t min_x = g->tune.sddmm_seg_min_mb << 20;
    if (budget <= 0 || row_bytes <= 0 || g->n_src * row_bytes <= std::max(budget, min_x)) return 0;
    return std::max<int64_t>(32, budget / row_bytes);
}

int64_t rows_with_degree_at_least(const fg_graph* g, int64_t t) {
    // deg_sorted is descending: first index with deg < t
    auto it = std::lower_bound(g->deg_sorted.begin(), g->deg_sorted.end(), t,
                               [](int64_t a, int64_t b) { return a >= b; });
    return int64_t(it - g->deg_sorted.begin());
}
}  // namespace fgk

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            st = fgk::set_error(e_ == cudaErrorMemoryAllocation ? FG_ENOMEM : FG_ECUDA,         \
                                "%s: %s", #x, cudaGetErrorString(e_));                          \
            goto fail;                                                                          \
        }                                                                                       \
    } while (0)

extern "C" fg_status fg_graph_create(int64_t n_dst, int64_t n_src, int64_t nnz, const int64_t* row_ptr,
                                     const int32_t* col_idx, const int32_t* eid, int validate,
                                     fg_stream stream, fg_graph** out) {
    if (!out) return fgk::set_error(FG_EINVAL, "fg_graph_create: out is NULL");
    if (!row_ptr) return fgk::set_error(FG_EINVAL, "fg_graph_create: row_ptr is NULL");
    if (nnz > 0 && !col_idx) return fgk::set_error(FG_EINVAL, "fg_graph_create: col_idx is NULL with nnz > 0");
    if (n_dst < 0 || n_src < 0 || nnz < 0 || nnz >= (int64_t(1) << 31) || n_dst >= (int64_t(1) << 31) ||
        n_src >= (int64_t(1) << 31))
        return fgk::set_error(FG_ESHAPE, "fg_graph_create: bad sizes n_dst=%lld n_src=%lld nnz=%lld",
                              (long long)n_dst, (long long)n_src, (long long)nnz);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    fg_status st = FG_OK;
    fg_graph* g = new fg_graph();
    g->n_dst = n_dst; g->n_src = n_src; g->nnz = nnz;
    g->row_ptr = row_ptr; g->col_idx = col_idx; g->eid = eid;
    cudaGetDevice(&g->device);
    fgk::tuning_from_env(&g->tune);
    unsigned* dflags = nullptr;
    unsigned* seen = nullptr;
    std::vector<int64_t> rp(size_t(n_dst + 1));
    std::vector<int32_t> order;
    std::vector<int32_t> urow;
    std::vector<int64_t> up0;

    CK(cudaMemcpyAsync(rp.data(), row_ptr, sizeof(int64_t) * size_t(n_dst + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (validate) {
        unsigned hflags = 0;
        if (rp[0] != 0 || rp[size_t(n_dst)] != nnz) hflags |= BAD_ROWPTR;
        CK(cudaMalloc(&dflags, sizeof(unsigned)));
        CK(cudaMemsetAsync(dflags, 0, sizeof(unsigned), s));
        if (n_dst > 0) {
            int blocks = int(std::min<int64_t>((n_dst + 7) / 8, 148 * 16));
            validate_rows<<<blocks, 256, 0, s>>>(n_dst, n_src, nnz, row_ptr, col_idx, dflags);
            CK(cudaGetLastError());
        }
        if (eid && nnz > 0) {
            CK(cudaMalloc(&seen, sizeof(unsigned) * size_t((nnz + 31) / 32)));
            CK(cudaMemsetAsync(seen, 0, sizeof(unsigned) * size_t((nnz + 31) / 32), s));
            int blocks = int(std::min<int64_t>((nnz + 255) / 256, 148 * 16));
            validate_eid<<<blocks, 256, 0, s>>>(nnz, eid, seen, dflags);
            CK(cudaGetLastError());
        }
        unsigned f = 0;
        CK(cudaMemcpyAsync(&f, dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        hflags |= f;
        if (hflags) {
            st = fgk::set_error(FG_EGRAPH, "fg_graph_create: CSR invariant violated:%s%s%s%s%s",
                                (hflags & BAD_ROWPTR) ? " row_ptr" : "",
                                (hflags & BAD_COL_RANGE) ? " col_idx-range" : "",
                                (hflags & BAD_COL_ORDER) ? " col_idx-not-strictly-ascending" : "",
                                (hflags & BAD_EID_RANGE) ? " eid-range" : "",
                                (hflags & BAD_EID_DUP) ? " eid-not-a-permutation" : "");
            goto fail;
        }
    } else {
        // cheap host-side sanity even without validation (row_ptr is on the host anyway)
        if (rp[0] != 0 || rp[size_t(n_dst)] != nnz) {
            st = fgk::set_error(FG_EGRAPH, "fg_graph_create: row_ptr[0] != 0 or row_ptr[n_dst] != nnz");
            goto fail;
        }
    }
    for (int64_t v = 0; v < n_dst; ++v)
        if (rp[size_t(v + 1)] < rp[size_t(v)]) {
            st = fgk::set_error(FG_EGRAPH, "fg_graph_create: row_ptr decreases at row %lld", (long long)v);
            goto fail;
        }

    // degree-descending row order (stable): LPT scheduling + degree bins
    order.resize(size_t(n_dst));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        return (rp[size_t(a) + 1] - rp[size_t(a)]) > (rp[size_t(b) + 1] - rp[size_t(b)]);
    });
    g->deg_sorted.resize(size_t(n_dst));
    for (int64_t i = 0; i < n_dst; ++i) {
        int64_t v = order[size_t(i)];
        g->deg_sorted[size_t(i)] = rp[size_t(v + 1)] - rp[size_t(v)];
    }
    g->max_deg = n_dst ? g->deg_sorted[0] : 0;
    g->n_nonempty = fgk::rows_with_degree_at_least(g, 1);

    // SDDMM units in degree-descending row order (heavy rows first)
    {   // edges per SDDMM work unit (FG_SDDMM_CHUNK, default 64: reddit u_dot_v H=1 F=512
        // 15.2-15.3 ms vs 16.5-16.8 at 256 and 18.1 at 512, H=8 8.9 vs 9.6 ms; 32 is 1-3 % slower)
        const char* uc = getenv("FG_SDDMM_CHUNK");
        g->unit_chunk = uc ? std::max(32, atoi(uc)) : 64;
    }
    for (int64_t i = 0; i < g->n_nonempty; ++i) {
        int64_t v = order[size_t(i)];
        for (int64_t p = rp[size_t(v)]; p < rp[size_t(v + 1)]; p += g->unit_chunk) {
            urow.push_back(int32_t(v));
            up0.push_back(p);
        }
    }
    g->n_units = int64_t(urow.size());

    if (n_dst > 0) {
        CK(cudaMalloc(&g->rows_by_deg, sizeof(int32_t) * size_t(n_dst)));
        CK(cudaMemcpyAsync(g->rows_by_deg, order.data(), sizeof(int32_t) * size_t(n_dst), cudaMemcpyHostToDevice, s));
        g->device_bytes += sizeof(int32_t) * n_dst;
    }
    if (g->n_units > 0) {
        CK(cudaMalloc(&g->unit_row, sizeof(int32_t) * size_t(g->n_units)));
        CK(cudaMalloc(&g->unit_p0, sizeof(int64_t) * size_t(g->n_units)));
        CK(cudaMemcpyAsync(g->unit_row, urow.data(), sizeof(int32_t) * size_t(g->n_units), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(g->unit_p0, up0.data(), sizeof(int64_t) * size_t(g->n_units), cudaMemcpyHostToDevice, s));
        g->device_bytes += 12 * g->n_units;
    }
    CK(cudaStreamSynchronize(s));   // host vectors die at return
    if (dflags) cudaFree(dflags);
    if (seen) cudaFree(seen);
    *out = g;
    return FG_OK;
fail:
    if (dflags) cudaFree(dflags);
    if (seen) cudaFree(seen);
    fg_graph_destroy(g);
    return st;
}

extern "C" fg_status fg_graph_destroy(fg_graph* g) {
    if (!g) return fgk::set_error(FG_EINVAL, "fg_graph_destroy: NULL handle");
    if (g->rows_by_deg) cudaFree(g->rows_by_deg);
    if (g->unit_row) cudaFree(g->unit_row);
    if (g->unit_p0) cudaFree(g->unit_p0);
    for (auto& su : g->seg_units) {
        cudaFree(su.row);
        cudaFree(su.p0);
        cudaFree(su.p1);
    }
    for (auto& sb : g->seg_bounds) cudaFree(sb.bnd);
    if (g->hyb.code) cudaFree(g->hyb.code);
    if (g->hyb.hot) cudaFree(g->hyb.hot);
    if (g->owned_row_ptr) cudaFree(g->owned_row_ptr);
    if (g->owned_col_idx) cudaFree(g->owned_col_idx);
    if (g->owned_eid) cudaFree(g->owned_eid);
    delete g;
    return FG_OK;
}

extern "C" fg_status fg_graph_info(const fg_graph* g, fg_graph_info_t* info) {
    if (!g || !info) return fgk::set_error(FG_EINVAL, "fg_graph_info: NULL argument");
    info->n_dst = g->n_dst;
    info->n_src = g->n_src;
    info->nnz = g->nnz;
    info->max_degree = g->max_deg;
    info->n_empty_rows = g->n_dst - g->n_nonempty;
    info->n_sddmm_units = g->n_units;
    info->device_bytes = g->device_bytes;
    return FG_OK;
}

// ---------------------------------------------------------------- knobs and prepare
extern "C" fg_status fg_graph_tune(fg_graph* g, fg_tune_key key, int64_t value) {
    if (!g) return fgk::set_error(FG_EINVAL, "fg_graph_tune: NULL handle");
    fg_tuning& t = g->tune;
    switch (key) {
        case FG_TUNE_L2_TILE_MB: t.l2_tile_mb = value < 0 ? -1 : value; break;
        case FG_TUNE_SPMM_HEAVY_DEG: t.spmm_heavy_deg = std::max<int64_t>(0, value); break;
        case FG_TUNE_BALANCE_NNZ: t.balance_nnz = std::max<int64_t>(0, value); break;
        case FG_TUNE_SDDMM_SEG_MB: t.sddmm_seg_mb = std::max<int64_t>(0, value); break;
        case FG_TUNE_SDDMM_SEG_MIN_MB: t.sddmm_seg_min_mb = std::max<int64_t>(0, value); break;
        case FG_TUNE_SDDMM_PERSIST: t.sddmm_persist = value; break;
        case FG_TUNE_SDDMM_L2_TILE: t.sddmm_l2_tile = value != 0; break;
        case FG_TUNE_SDDMM_DOT: t.sddmm_dot = value != 0; break;
        case FG_TUNE_GAT_HEAVY_DEG: t.gat_heavy_deg = std::max<int64_t>(1, value); break;
        case FG_TUNE_MLP_IMPL:
            if (value < 0 || value > 2) return fgk::set_error(FG_EINVAL, "fg_graph_tune: mlp impl %lld", (long long)value);
            t.mlp_impl = value;
            break;
        case FG_TUNE_HYBRID: t.hybrid = value != 0; break;
        case FG_TUNE_SPMM_SEG_MB: t.spmm_seg_mb = std::max<int64_t>(0, value); break;
        case FG_TUNE_SDDMM_PIPE:
            if (value < -1 || value > 7) return fgk::set_error(FG_EINVAL, "fg_graph_tune: sddmm pipe %lld", (long long)value);
            t.sddmm_pipe = value;
            break;
        case FG_TUNE_SDDMM_ORDER:
            if (value < 0 || value > 1) return fgk::set_error(FG_EINVAL, "fg_graph_tune: sddmm order %lld", (long long)value);
            t.sddmm_order = value;
            break;
        case FG_TUNE_SDDMM_RB_MB: t.sddmm_rb_mb = std::max<int64_t>(0, value); break;
        case FG_TUNE_SPMM_LDG256: t.spmm_ldg256 = value != 0; break;
        default: return fgk::set_error(FG_EINVAL, "fg_graph_tune: bad key %d", int(key));
    }
    return FG_OK;
}

extern "C" fg_status fg_graph_get_tune(const fg_graph* g, fg_tune_key key, int64_t* value) {
    if (!g || !value) return fgk::set_error(FG_EINVAL, "fg_graph_get_tune: NULL argument");
    const fg_tuning& t = g->tune;
    switch (key) {
        case FG_TUNE_L2_TILE_MB: *value = t.l2_tile_mb; break;
        case FG_TUNE_SPMM_HEAVY_DEG: *value = t.spmm_heavy_deg; break;
        case FG_TUNE_BALANCE_NNZ: *value = t.balance_nnz; break;
        case FG_TUNE_SDDMM_SEG_MB: *value = t.sddmm_seg_mb; break;
        case FG_TUNE_SDDMM_SEG_MIN_MB: *value = t.sddmm_seg_min_mb; break;
        case FG_TUNE_SDDMM_PERSIST: *value = t.sddmm_persist; break;
        case FG_TUNE_SDDMM_L2_TILE: *value = t.sddmm_l2_tile; break;
        case FG_TUNE_SDDMM_DOT: *value = t.sddmm_dot; break;
        case FG_TUNE_GAT_HEAVY_DEG: *value = t.gat_heavy_deg; break;
        case FG_TUNE_MLP_IMPL: *value = t.mlp_impl; break;
        case FG_TUNE_HYBRID: *value = t.hybrid; break;
        case FG_TUNE_SPMM_SEG_MB: *value = t.spmm_seg_mb; break;
        case FG_TUNE_SDDMM_PIPE: *value = t.sddmm_pipe; break;
        case FG_TUNE_SDDMM_ORDER: *value = t.sddmm_order; break;
        case FG_TUNE_SDDMM_RB_MB: *value = t.sddmm_rb_mb; break;
        case FG_TUNE_SPMM_LDG256: *value = t.spmm_ldg256; break;
        default: return fgk::set_error(FG_EINVAL, "fg_graph_get_tune: bad key %d", int(key));
    }
    return FG_OK;
}

extern "C" fg_status fg_graph_prepare(fg_graph* g, int64_t row_bytes, fg_stream stream) {
    if (!g) return fgk::set_error(FG_EINVAL, "fg_graph_prepare: NULL handle");
    if (row_bytes <= 0) return fgk::set_error(FG_ESHAPE, "fg_graph_prepare: row_bytes must be > 0");
    if (g->nnz == 0) return FG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t seg_rows = fgk::sddmm_seg_rows(g, row_bytes);   // 0: this width is not segmented
    if (seg_rows) {
        const fg_status s = fgk::build_seg_units(g, seg_rows, fgk::sddmm_rb_rows(g, row_bytes), g->unit_chunk, st);
        if (s != FG_OK) return s;
    }
    const int64_t spmm_rows = fgk::spmm_seg_rows(g, row_bytes);
    return spmm_rows ? fgk::build_seg_bounds(g, spmm_rows, st) : FG_OK;
}

// ---------------------------------------------------------------- hybrid partitioning
namespace {
__global__ void out_degree_kernel(int64_t nnz, const int32_t* __restrict__ ci, int32_t* __restrict__ cnt) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz; p += int64_t(gridDim.x) * blockDim.x)
        atomicAdd(cnt + __ldg(ci + p), 1);   // integer counts: order-independent
}
__global__ void hybrid_code_kernel(int64_t nnz, const int32_t* __restrict__ ci, const int32_t* __restrict__ slot,
                                   int32_t* __restrict__ code) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz; p += int64_t(gridDim.x) * blockDim.x) {
        const int32_t u = __ldg(ci + p);
        const int32_t k = __ldg(slot + u);
        code[p] = k >= 0 ? -(k + 1) : u;
    }
}
}  // namespace

extern "C" fg_status fg_graph_prepare_hybrid(fg_graph* g, int64_t row_bytes, int64_t smem_bytes, fg_stream stream) {
    if (!g) return fgk::set_error(FG_EINVAL, "fg_graph_prepare_hybrid: NULL handle");
    if (row_bytes <= 0 || row_bytes % 16 != 0 || smem_bytes < row_bytes || smem_bytes > 200 * 1024)
        return fgk::set_error(FG_ESHAPE, "fg_graph_prepare_hybrid: row_bytes %lld (multiple of 16) and smem_bytes "
                              "%lld (row_bytes .. 200 KiB)", (long long)row_bytes, (long long)smem_bytes);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (g->hyb.code) cudaFree(g->hyb.code);
    if (g->hyb.hot) cudaFree(g->hyb.hot);
    g->hyb = fg_graph::Hybrid();
    if (g->nnz == 0 || g->n_src == 0) return FG_OK;
    const int64_t n = g->n_src, m = g->nnz;
    const int64_t k = std::min<int64_t>(n, smem_bytes / row_bytes);
    int32_t *cnt = nullptr, *slot = nullptr;
    std::vector<int32_t> hc(static_cast<size_t>(n)), hs(static_cast<size_t>(n), -1);
    std::vector<int32_t> order(static_cast<size_t>(n));
    std::vector<int32_t> hot;
    int64_t hot_edges = 0;
    fg_status st = FG_OK;
    cudaError_t e = cudaMalloc(&cnt, sizeof(int32_t) * size_t(n));
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, sizeof(int32_t) * size_t(n), s);
    if (e == cudaSuccess) {
        out_degree_kernel<<<int(std::min<int64_t>((m + 255) / 256, 148 * 16)), 256, 0, s>>>(m, g->col_idx, cnt);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), cnt, sizeof(int32_t) * size_t(n), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) {
        // the k sources of highest out-degree (ties: lower id), degree > 0
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return hc[size_t(a)] > hc[size_t(b)]; });
        for (int64_t i = 0; i < k && hc[size_t(order[size_t(i)])] > 0; ++i) {
            hs[size_t(order[size_t(i)])] = int32_t(i);
            hot.push_back(order[size_t(i)]);
            hot_edges += hc[size_t(order[size_t(i)])];
        }
    }
    if (e == cudaSuccess) e = cudaMalloc(&slot, sizeof(int32_t) * size_t(n));
    if (e == cudaSuccess) e = cudaMalloc(&g->hyb.code, sizeof(int32_t) * size_t(m));
    if (e == cudaSuccess) e = cudaMalloc(&g->hyb.hot, sizeof(int32_t) * std::max<size_t>(hot.size(), 1));
    if (e == cudaSuccess) e = cudaMemcpyAsync(slot, hs.data(), sizeof(int32_t) * size_t(n), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !hot.empty())
        e = cudaMemcpyAsync(g->hyb.hot, hot.data(), sizeof(int32_t) * hot.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        hybrid_code_kernel<<<int(std::min<int64_t>((m + 255) / 256, 148 * 16)), 256, 0, s>>>(m, g->col_idx, slot,
                                                                                           g->hyb.code);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(cnt);
    cudaFree(slot);
    if (e != cudaSuccess) {
        st = fgk::set_error(e == cudaErrorMemoryAllocation ? FG_ENOMEM : FG_ECUDA, "fg_graph_prepare_hybrid: %s",
                            cudaGetErrorString(e));
        if (g->hyb.code) cudaFree(g->hyb.code);
        if (g->hyb.hot) cudaFree(g->hyb.hot);
        g->hyb = fg_graph::Hybrid();
        return st;
    }
    g->hyb.row_bytes = row_bytes;
    g->hyb.k = int64_t(hot.size());
    g->hyb.hot_edge_share = double(hot_edges) / double(m);
    g->device_bytes += 4 * m + 4 * g->hyb.k;
    return FG_OK;
}

extern "C" fg_status fg_graph_hybrid_info(const fg_graph* g, int64_t* k, double* hot_edge_share) {
    if (!g || !k || !hot_edge_share) return fgk::set_error(FG_EINVAL, "fg_graph_hybrid_info: NULL argument");
    *k = g->hyb.k;
    *hot_edge_share = g->hyb.hot_edge_share;
    return FG_OK;
}
