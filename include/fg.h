/*
 * fg.h -- C ABI of libfg.so, the B200-native (sm_100a) hot path of FeatGraph
 * (Hu et al., "FeatGraph: A Flexible and Efficient Backend for Graph Neural
 * Network Systems", SC20, arXiv 2008.11359).
 *
 * The paper's interface (§3.2):
 *   featgraph.spmat(shape=(n,n), nnz=m)
 *   featgraph.spmm(A, msgfunc, aggregation, target, fds)
 *   featgraph.sddmm(A, edgefunc, target, fds)
 * maps to fg_graph_create / fg_spmm / fg_sddmm below.  `target` is always
 * sm_100a and the feature-dimension schedule (FDS) is internal to the library
 * (launch configuration chosen per (F, degree bin)); the UDFs are the fixed
 * enums fg_msg_op / fg_edge_op, which cover every UDF the paper evaluates
 * (Fig. 3a copy-src, Fig. 3b MLP, Fig. 5 (multi-head) dot product, and the DGL
 * vertex-x-edge builtin of P:375).  Edge softmax (fg_edge_softmax) is not in
 * the paper; it is the standard GAT normalisation the paper's GAT layer needs
 * (P:983).
 *
 * CONVENTIONS (all functions)
 *  - No C++ or CUDA types cross this boundary: tensors are plain pointers, sizes
 *    are int64_t, a stream is an opaque `fg_stream` (a cudaStream_t / CUstream;
 *    NULL = the legacy default stream).
 *  - Graph: destination-major CSR (Eq. (3) P:158 H_V = A X_V
 *    "rows in the adjacency matrix"): row v = [row_ptr[v], row_ptr[v+1]) lists
 *    the sources u = col_idx[p] of the in-edges u -> v, strictly ascending
 *    (no duplicate edges; self-loops allowed).  Edge id of CSR position p is
 *    eid[p] (eid == NULL: identity).  Edge tensors (E, SDDMM output, scores)
 *    are indexed by edge id.
 *  - Every tensor pointer passed to fg_spmm / fg_sddmm / fg_edge_softmax /
 *    fg_graph_create is a DEVICE pointer owned by the caller; the library never
 *    frees caller memory.  Float tensors are fp32, row-major, and must be
 *    16-byte aligned (128-bit lane accesses); F % 4 == 0 (F = H*D, or d2).
 *  - fg_graph borrows row_ptr / col_idx / eid: they must stay alive and
 *    unmodified until fg_graph_destroy.  The handle owns only derived tables.
 *  - Calls are asynchronous on `stream` except the per-topology ones,
 *    fg_graph_create / fg_graph_prepare / fg_graph_transpose (synchronous: they
 *    read the CSR back and allocate the handle's tables).  The op calls never
 *    allocate, synchronise or read the environment, so they can be captured in
 *    a CUDA graph.
 *    Argument errors are detected on the host BEFORE any launch: a non-OK
 *    status means nothing was launched and outputs are untouched.  Device
 *    faults surface at the caller's next synchronisation.
 *  - Outputs are fully overwritten, never accumulated into.
 *  - Results are deterministic: no floating-point atomics; reruns are bitwise
 *    identical.
 *  - A handle is only modified by fg_graph_prepare / fg_graph_tune: between
 *    those, op calls on the same handle from different streams or threads are
 *    safe (no per-call state lives in the handle).  fg_last_error() is
 *    thread-local.
 */
#ifndef FG_H_
#define FG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FG_ABI_VERSION 1

typedef enum {
    FG_OK = 0,
    FG_EINVAL = 1,        /* null pointer, bad enum, misaligned pointer */
    FG_ESHAPE = 2,        /* inconsistent or unsupported dimensions */
    FG_EUNSUPPORTED = 3,  /* valid request, combination not implemented */
    FG_EGRAPH = 4,        /* CSR invariant violated (validate = 1) */
    FG_ECUDA = 5,         /* CUDA runtime / launch error */
    FG_ENOMEM = 6,        /* device or host allocation failed */
    FG_ENCCL = 7          /* NCCL error (multi-GPU calls) */
} fg_status;

/* Message functions phi of Eq. (1). */
typedef enum {
    FG_MSG_COPY_U = 0,   /* phi = x_u                       Fig. 3a */
    FG_MSG_U_MUL_E = 1,  /* phi[h,d] = x_u[h,d] * x_uv[h]   DGL builtin P:375; GAT P:983 */
    FG_MSG_MLP = 2,      /* phi = ReLU((x_u + x_v) W)       Fig. 3b */
    FG_MSG_U_ADD_E = 3,  /* phi[h,d] = x_u[h,d] + x_uv[h]   DGL builtin family P:372-375 (row f4) */
    FG_MSG_COPY_E = 4    /* phi = x_uv (edge feature row)   same family (row f4) */
} fg_msg_op;

/* Aggregations (+) of Eq. (1): sum (Fig. 3a), max (Fig. 1).
 * min and mean are the other two reducers of the DGL builtin family the paper
 * plugs into: min is max with the comparison
 * flipped, mean is sum divided by the in-degree |N(v)| (IEEE fp32 division). */
typedef enum { FG_REDUCE_SUM = 0, FG_REDUCE_MAX = 1, FG_REDUCE_MIN = 2, FG_REDUCE_MEAN = 3 } fg_reduce_op;

/* Edge functions psi of Eq. (2). */
typedef enum {
    FG_EDGE_U_DOT_V = 0, /* psi[h] = sum_d x_u[h,d] y_v[h,d]   Eq. (4); Fig. 5 */
    FG_EDGE_U_ADD_V = 1, /* psi[j] = x_u[j] + y_v[j]           DGL builtin family P:372-375 (row f4) */
    FG_EDGE_U_SUB_V = 2, /* psi[j] = x_u[j] - y_v[j]           same */
    FG_EDGE_U_MUL_V = 3  /* psi[j] = x_u[j] * y_v[j]           same */
} fg_edge_op;

typedef struct fg_graph fg_graph;          /* opaque; changed only by fg_graph_prepare / fg_graph_tune */
typedef struct CUstream_st* fg_stream;      /* == cudaStream_t */

/* ---------------------------------------------------------------- graph */
/*
 * fg_graph_create -- featgraph.spmat.  Builds the per-topology tables
 * (degree-sorted row order, degree bins, SDDMM edge-chunk table), amortised
 * over calls as the paper amortises per-topology code generation.
 *   n_dst, n_src : rows / columns of A (n_dst >= 0, n_src >= 0)
 *   nnz          : number of edges, 0 <= nnz < 2^31
 *   row_ptr      : device int64[n_dst+1]
 *   col_idx      : device int32[nnz]   (may be NULL iff nnz == 0)
 *   eid          : device int32[nnz] or NULL (identity)
 *   validate     : nonzero -> check row_ptr[0] == 0, row_ptr non-decreasing,
 *                  row_ptr[n_dst] == nnz, 0 <= col_idx < n_src strictly
 *                  ascending per row, eid a permutation of [0,nnz); violations
 *                  return FG_EGRAPH (detail in fg_last_error()).
 *   stream       : stream used for the (synchronous) preprocessing.
 *   out          : receives the handle (set only on FG_OK).
 */
fg_status fg_graph_create(int64_t n_dst, int64_t n_src, int64_t nnz, const int64_t* row_ptr,
                          const int32_t* col_idx, const int32_t* eid, int validate,
                          fg_stream stream, fg_graph** out);
fg_status fg_graph_destroy(fg_graph* g);

/* Host-side description of a handle (tests / tooling). */
typedef struct {
    int64_t n_dst, n_src, nnz;
    int64_t max_degree;
    int64_t n_empty_rows;     /* rows of degree 0 */
    int64_t n_sddmm_units;    /* (row, edge chunk) work units of fg_sddmm */
    int64_t device_bytes;     /* bytes of derived tables owned by the handle */
} fg_graph_info_t;
fg_status fg_graph_info(const fg_graph* g, fg_graph_info_t* info);

/*
 * fg_graph_prepare -- the per-topology tables of the source-segmented gSDDMM
 * traversal and of the source-segmented u_mul_e-sum passes of gSpMM for
 * gathered rows of `row_bytes` bytes (H*D*4 for fp32 features, H*D*2 for bf16
 * storage): the paper's 1D source partitioning with segments sized
 * to the B200 L2.  It applies only when the source features
 * are wider than the segmentation threshold (48 MB segments for X > 96 MB by
 * default); otherwise it builds nothing and returns FG_OK.  With
 * FG_TUNE_SPMM_SEG_MB set (off by default), fg_spmm u_mul_e-sum
 * (fp32, D % 4 == 0) on a prepared width runs one pass per segment in segment
 * order, each adding its sources' messages onto out: a group-per-row row keeps
 * the CSR summation order (bit-identical to the unprepared call); a row split
 * CTA-per-row (degree >= the heavy threshold) sums in another fixed order
 * (deterministic, equal to rounding).
 * SYNCHRONOUS on `stream` (allocates device memory, reads counts back), like
 * fg_graph_create; idempotent per width.  fg_sddmm / fg_sddmm_emul /
 * fg_sddmm_x16 / fg_dist_sddmm never allocate or synchronise (so they can be
 * captured in a CUDA graph): for a width that was not prepared they run the
 * unsegmented traversal, which gives bit-identical results (each edge's dot
 * product is evaluated by the same lane partition and reduction tree; only
 * the order of the work units differs) and is slower only when X exceeds the
 * L2.  Not safe concurrently with calls on the same handle.
 *   Errors: FG_EINVAL (NULL), FG_ESHAPE (row_bytes <= 0), FG_ENOMEM, FG_ECUDA.
 */
fg_status fg_graph_prepare(fg_graph* g, int64_t row_bytes, fg_stream stream);

/*
 * fg_graph_tune / fg_graph_get_tune -- the launch-configuration knobs of one
 * handle (the paper's FDS, kept internal: every default is the
 * value measured best on B200, DESIGN.md §6 / §9).  The FG_* environment
 * variables of the same names are read once, by fg_graph_create; the launch
 * paths read only the handle.  Values are read on the host at each launch, so
 * a change applies to later calls; not safe concurrently with other calls on
 * the same handle.  None of them changes a result beyond the fp32 summation
 * order of a sum (max / min / argmax / integer results are invariant), except
 * FG_TUNE_MLP_IMPL = 2 (bf16 2-split, within the same 1e-4 tolerance).
 *   FG_TUNE_L2_TILE_MB     copy_u column-tile budget in MB (-1 default, 0 off)
 *   FG_TUNE_SPMM_HEAVY_DEG CTA-per-row degree threshold of gSpMM (0 automatic)
 *   FG_TUNE_BALANCE_NNZ    edge count the automatic threshold is computed from
 *                          (0: this graph's nnz).  The sharding code sets the
 *                          whole graph's nnz on every shard, so shards split
 *                          rows exactly as the unsharded op: bit-identical sums.
 *   FG_TUNE_SDDMM_SEG_MB, FG_TUNE_SDDMM_SEG_MIN_MB   segmentation (above)
 *   FG_TUNE_SDDMM_PERSIST  CTAs per SM of the segmented launch (-1 occupancy)
 *   FG_TUNE_SDDMM_L2_TILE  1: column-tiled gSDDMM passes (ablation)
 *   FG_TUNE_SDDMM_DOT      1: thread-per-edge dot products (ablation E6)
 *   FG_TUNE_GAT_HEAVY_DEG  CTA-per-row threshold of fg_gat_attention
 *   FG_TUNE_MLP_IMPL       0 tcgen05 3xTF32 (default), 1 CUDA-core FFMA,
 *                          2 tcgen05 bf16 2-split with K = 32 (ablations)
 *   FG_TUNE_HYBRID         1: hot sources staged in shared memory by gSpMM
 *                          copy_u-sum (the paper's hybrid partitioning,
 *                          P:534-539) when fg_graph_prepare_hybrid built the
 *                          table for that width (ablation E7)
 *   FG_TUNE_SPMM_SEG_MB    source-segment size in MB of the segmented
 *                          u_mul_e-sum passes of fg_spmm (0 = off, the default:
 *                          on reddit H=8 D=32 48 MB segments cut DRAM traffic
 *                          19.7 -> 9.4 GB but ran 8.07 vs 7.47 ms; only for X
 *                          wider than FG_TUNE_SDDMM_SEG_MIN_MB, and only once
 *                          fg_graph_prepare built the bounds with it set)
 *   FG_TUNE_SDDMM_PIPE     fp32 gSDDMM with 33..128 float4 per row: -1 auto
 *                          (H == 1: software-pipelined kernel for 65..96,
 *                          unit-prefetching kernel for 33..64 (4) and 97..128
 *                          (7); heads of D = 32 / 64: unit-prefetching up to 64
 *                          float4 (4), 65..96 (7), and at 128 for D = 64 (7)),
 *                          0 plain, 1..3 pipelined variants (H == 1; U = 1 / 2
 *                          edges per stage, 2 / 3 CTAs per SM), 4 unit-
 *                          prefetching (the next unit's indices and Y row
 *                          staged by cp.async; Y in registers, 3 CTAs per SM),
 *                          5 / 6 the same with Y read from shared memory
 *                          (H == 1; 4 / 3 CTAs per SM), 7 unit-prefetching
 *                          with twice the edges in flight at 2 CTAs per SM;
 *                          bit-identical in every setting
 *   FG_TUNE_SDDMM_ORDER    0 segment-major work units (default), 1 2D tiles
 *                          (destination block x source segment) in Hilbert-
 *                          curve order (ablation, measured slower);
 *                          applies to tables built by fg_graph_prepare with it
 *                          set; bit-identical either way
 *   FG_TUNE_SDDMM_RB_MB    Hilbert order: destination-block size in MB of Y
 *                          rows (0: the segment size)
 *   FG_TUNE_SPMM_LDG256    1: fp32 copy_u gathers read 32-byte chunk pairs
 *                          (LDG.256) when X is 32-byte aligned and the row /
 *                          tile width is an even number of 4-feature chunks
 *                          (ablation: 4-17 % slower on every shaped graph);
 *                          0 (default): 16-byte loads.  Changes the lanes per
 *                          row, hence the automatic heavy-row split of sums.
 *   Errors: FG_EINVAL (NULL, unknown key, out-of-range value).
 */
/*
 * fg_graph_prepare_hybrid -- the table of the GPU hybrid partitioning (PAPER.md
 * "reorders the vertices into a low-degree part and a high-degree
 * part according to a threshold; it only partitions high-degree vertices and
 * loads them to shared memory"): the k = smem_bytes / row_bytes sources of
 * highest out-degree (ties: lower id) form the shared-memory partition, and
 * every edge gets a source code (u, or the staged slot) in a copy of col_idx
 * owned by the handle (4 * nnz bytes).  Used by fg_spmm copy_u-sum for rows of
 * exactly row_bytes (fp32 F = row_bytes / 4 <= 128, untiled) when
 * FG_TUNE_HYBRID is 1; results are bit-identical to the plain kernel (same
 * values, same order).  SYNCHRONOUS; replaces any previous hybrid table.
 *   row_bytes  : bytes per source row (multiple of 16)
 *   smem_bytes : shared memory per CTA for the staged rows (row_bytes .. 200 KiB)
 *   Errors: FG_EINVAL, FG_ESHAPE, FG_ENOMEM, FG_ECUDA.
 * fg_graph_hybrid_info -- k and the fraction of edges whose source is staged.
 */
fg_status fg_graph_prepare_hybrid(fg_graph* g, int64_t row_bytes, int64_t smem_bytes, fg_stream stream);
fg_status fg_graph_hybrid_info(const fg_graph* g, int64_t* k, double* hot_edge_share);

typedef enum {
    FG_TUNE_L2_TILE_MB = 0,
    FG_TUNE_SPMM_HEAVY_DEG = 1,
    FG_TUNE_BALANCE_NNZ = 2,
    FG_TUNE_SDDMM_SEG_MB = 3,
    FG_TUNE_SDDMM_SEG_MIN_MB = 4,
    FG_TUNE_SDDMM_PERSIST = 5,
    FG_TUNE_SDDMM_L2_TILE = 6,
    FG_TUNE_SDDMM_DOT = 7,
    FG_TUNE_GAT_HEAVY_DEG = 8,
    FG_TUNE_MLP_IMPL = 9,
    FG_TUNE_HYBRID = 10,
    FG_TUNE_SPMM_SEG_MB = 11,
    FG_TUNE_SDDMM_PIPE = 12,
    FG_TUNE_SDDMM_ORDER = 13,
    FG_TUNE_SDDMM_RB_MB = 14,
    FG_TUNE_SPMM_LDG256 = 15
} fg_tune_key;
fg_status fg_graph_tune(fg_graph* g, fg_tune_key key, int64_t value);
fg_status fg_graph_get_tune(const fg_graph* g, fg_tune_key key, int64_t* value);

/* ---------------------------------------------------------------- gSpMM */
/*
 * fg_spmm -- featgraph.spmm(A, msgfunc, aggregation), Eq. (1):
 *     out[v] = (+)_{u -> v} phi(x_u, x_v, x_uv)
 *
 *   msg = FG_MSG_COPY_U   : X [n_src][H*D]; E, W, X_dst NULL; d_in = 0.
 *   msg = FG_MSG_U_MUL_E  : X [n_src][H*D]; E [nnz][H] indexed by edge id.
 *   msg = FG_MSG_U_ADD_E  : as u_mul_e with phi = x_u + e (fp32 add, rounded
 *                           once before a max/min compare).
 *   msg = FG_MSG_COPY_E   : X NULL; E [nnz][H*D] indexed by edge id, 16-byte
 *                           aligned (the message is the edge's own row).
 *   msg = FG_MSG_MLP      : H == 1, D == d2 (output width); X [n_src][d_in],
 *                           W [d_in][d2], X_dst [n_dst][d_in] (NULL -> X, which
 *                           requires n_src == n_dst); 1 <= d_in <= 32 (d_in = 8
 *                           in the paper).  ReLU after the full
 *                           contraction (Fig. 3b), s = x_u + x_v
 *                           formed in fp32 before the contraction (the paper's
 *                           order).  Runs on the tcgen05 tensor cores
 *                           (3xTF32); X / X_dst 16-byte aligned.
 *   out   : [n_dst][H*D] fp32, fully overwritten.
 *   red   : FG_REDUCE_SUM / _MAX / _MIN / _MEAN (elementwise per feature
 *           column).  mlp supports sum and max only (else FG_EUNSUPPORTED).
 *   arg_u, arg_e : max/min only, each optional (NULL); int32 [n_dst][H*D]:
 *           source id / edge id of the winning edge.  Ties -> lowest CSR
 *           position.  Must be NULL for sum and mean.
 *   Empty rows: out = +0.0 and arg = -1.
 *   workspace / workspace_bytes: device scratch of fg_spmm_workspace_size
 *           bytes; that size is 0 for every op of this version (heavy rows
 *           combine on chip; the mlp producer forms and splits x_u + x_v on
 *           the fly), so NULL / 0 may be passed.  Kept for ABI stability.
 *   Errors: FG_EINVAL (null/misaligned pointer, bad enum, arg_* with sum),
 *           FG_ESHAPE (H < 1, D < 1, (H*D) % 4 != 0, mlp with H != 1 or d_in
 *           out of range, u_mul_e/copy_u with d_in != 0), FG_ECUDA.
 */
fg_status fg_spmm_workspace_size(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D,
                                 int d_in, size_t* bytes);
fg_status fg_spmm(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D,
                  const float* X, const float* E, const float* W, int d_in, const float* X_dst,
                  float* out, int32_t* arg_u, int32_t* arg_e, void* workspace,
                  size_t workspace_bytes, fg_stream stream);

/* ---------------------------------------------------------------- gSDDMM */
/*
 * fg_sddmm -- featgraph.sddmm(A, edgefunc), Eq. (2)/(4):
 *     out[eid(p)][h] = sum_{d<D} X[u][h][d] * Y[v][h][d]   for every edge p = (u -> v)
 *   X : [n_src][H][D];  Y : [n_dst][H][D] (may equal X: Eq. (4) uses X_V on
 *       both sides);  out : [nnz][H], fully overwritten.
 *   Heads are independent reductions (Fig. 5b).  Requires (H*D) % 4 == 0 (else
 *   FG_ESHAPE).  Any D: D = 4 * 2^k with H*D <= 512 (and every H == 1 width)
 *   runs the lane-partitioned kernels; other head shapes a thread-per-edge
 *   kernel (each head's dot one sequential fp32 FMA chain; 2.5-4x slower).
 * Elementwise ops (FG_EDGE_U_ADD_V / _SUB_V / _MUL_V, row f4):
 *     out[eid(p)][j] = X[u][j] OP Y[v][j],  j < H*D;  out : [nnz][H*D] (H is
 *   only a shape factor here); one IEEE fp32 operation per element, so the
 *   result is exact to the rounding of that operation.
 */
fg_status fg_sddmm(const fg_graph* g, fg_edge_op op, int H, int D, const float* X, const float* Y,
                   float* out, fg_stream stream);

/* ---------------------------------------------------------------- edge softmax */
/*
 * fg_edge_softmax -- per destination v and head h, over the in-edges of v:
 *     alpha[e][h] = exp(s[e][h] - max_row) / sum_row exp(s[.][h] - max_row)
 *   scores, out : [nnz][H] indexed by edge id; out may alias scores (in place).
 *   Not in the paper (GAT normalisation).
 */
fg_status fg_edge_softmax(const fg_graph* g, int H, const float* scores, float* out,
                          fg_stream stream);

/* ---------------------------------------------------------------- fused GAT attention */
/*
 * fg_gat_attention -- gSDDMM u_dot_v -> edge softmax -> gSpMM u_mul_e-sum in ONE
 * pass (the paper's kernel fusion, P:378-379 / P:554, applied across the three
 * templates of the GAT layer):
 *     out[v][h,:] = sum_{e=u->v} softmax_e(<X[u][h,:], Y[v][h,:]>) * X[u][h,:]
 *   X [n_src][H][D], Y [n_dst][H][D] (may equal X), out [n_dst][H][D] (empty
 *   rows -> 0); scores: optional [nnz][H] (edge id) receives the pre-softmax
 *   scores s.  Equal in real arithmetic to fg_sddmm + fg_edge_softmax + fg_spmm
 *   (u_mul_e, sum); here s and alpha never leave the SM and X[u] is read once.
 *   Fused for D = 4*2^k <= 128 with H*D <= 512; any other shape with (H*D) % 4
 *   == 0 runs that unfused chain through `scores` (then required: alpha is
 *   formed in place and the pre-softmax scores are written again at the end;
 *   FG_EUNSUPPORTED when scores is NULL).
 */
fg_status fg_gat_attention(const fg_graph* g, int H, int D, const float* X, const float* Y, float* out,
                           float* scores, fg_stream stream);

/*
 * fg_sddmm_emul -- u_dot_v followed by e_mul (row f4: the DGL builtin pair the
 *   SDDMM template covers), the edge function inlined into the
 *   template:
 *     out[eid(p)][h] = ( sum_{d<D} X[u][h][d] * Y[v][h][d] ) * E[eid(p)][h]
 *   X, Y, out as fg_sddmm (u_dot_v); E : fp32 [nnz][H] indexed by edge id;
 *   out must not overlap E (FG_EINVAL).  The scale is applied at the kernel's
 *   result write-back; shape rules and errors as fg_sddmm.
 */
fg_status fg_sddmm_emul(const fg_graph* g, int H, int D, const float* X, const float* Y, const float* E,
                        float* out, fg_stream stream);

/* ---------------------------------------------------------- bf16 features */
/*
 * Row f4: bf16 STORAGE of the vertex features, fp32 arithmetic.
 * The messages and reductions are those of fg_spmm / fg_sddmm (Eq. (1), (4));
 * only the gathered operand is narrower (8 bytes per 4 features instead of
 * 16: the gathers -- the bound of these kernels, DESIGN.md §6 -- move half
 * the bytes).  bf16 -> fp32 is exact, so the result is the fp32 computation on
 * the bf16-representable inputs, to the same tolerance (1e-4 * sum|terms|
 * against the fp64 oracle on the decoded inputs).
 *
 * fg_spmm_x16 -- msg in {FG_MSG_COPY_U, FG_MSG_U_MUL_E} (else
 *   FG_EUNSUPPORTED), red any of sum / max / min / mean.  X : bf16 bits
 *   [n_src][H*D] (uint16, 8-byte aligned); E : fp32 [nnz][H] for u_mul_e,
 *   else NULL; out fp32 [n_dst][H*D]; arg_u / arg_e as fg_spmm (max / min
 *   only).  Same
 *   semantics, tie rules, empty-row conventions and errors as fg_spmm.
 * fg_sddmm_x16 -- op FG_EDGE_U_DOT_V only.  X [n_src][H][D], Y [n_dst][H][D]
 *   bf16 bits (8-byte aligned); out fp32 [nnz][H].  Shape rules as fg_sddmm.
 */
fg_status fg_spmm_x16(const fg_graph* g, fg_msg_op msg, fg_reduce_op red, int H, int D,
                      const uint16_t* X, const float* E, float* out, int32_t* arg_u, int32_t* arg_e,
                      fg_stream stream);
fg_status fg_sddmm_x16(const fg_graph* g, fg_edge_op op, int H, int D, const uint16_t* X,
                       const uint16_t* Y, float* out, fg_stream stream);

/* ---------------------------------------------------------------- backward */
/*
 * Gradients by the paper's gradient duality (the gradient
 * of SpMM follows the SDDMM pattern and vice versa).  Deterministic pulls, no
 * atomics.
 *
 * fg_graph_transpose -- the transposed handle gT (rows = sources, CSC of g),
 *   each row ascending, with eid mapping every transposed position to g's edge
 *   id, so edge tensors are shared between g and gT.  gT OWNS its arrays (built
 *   on the host from a copy of g's CSR; synchronous, per topology, like
 *   fg_graph_create).  Destroy with fg_graph_destroy.
 *
 * fg_spmm_backward -- for out = fg_spmm(g, msg, red, H, D, X, E, ...):
 *   msg in {FG_MSG_COPY_U, FG_MSG_U_MUL_E} (mlp: FG_EUNSUPPORTED -- SPEC.md
 *   S:380 non-goal);
 *   dOut [n_dst][H*D];  dX [n_src][H*D] (optional, needs gT);  dE [nnz][H]
 *   (optional, u_mul_e only, needs X);  max/min need arg_u from the forward
 *   (only the winning edge of each (v, j) receives dOut[v][j]); mean passes
 *   dOut[v] / |N(v)| to every in-edge of v.  Outputs overwritten.
 *
 * fg_sddmm_backward -- for s = fg_sddmm(g, u_dot_v, H, D, X, Y):
 *   dX [n_src][H*D] = sum_{e=u->v} dS[e] Y[v] (needs gT, Y);
 *   dY [n_dst][H*D] = sum_{e=u->v} dS[e] X[u] (needs X).  Either may be NULL.
 *   When Y is X (square graph) the caller adds dX + dY.
 *
 * fg_edge_softmax_backward -- for alpha = fg_edge_softmax(g, H, s):
 *   dscores[e][h] = alpha[e][h] (dalpha[e][h] - sum_{e' in row(e)} alpha[e'][h] dalpha[e'][h]).
 *   dscores must not alias alpha or dalpha.
 */
fg_status fg_graph_transpose(const fg_graph* g, fg_stream stream, fg_graph** out);
fg_status fg_spmm_backward(const fg_graph* g, const fg_graph* gT, fg_msg_op msg, fg_reduce_op red, int H, int D,
                           const float* X, const float* E, const float* dOut, const int32_t* arg_u, float* dX,
                           float* dE, fg_stream stream);
fg_status fg_sddmm_backward(const fg_graph* g, const fg_graph* gT, fg_edge_op op, int H, int D, const float* X,
                            const float* Y, const float* dS, float* dX, float* dY, fg_stream stream);
fg_status fg_edge_softmax_backward(const fg_graph* g, int H, const float* alpha, const float* dalpha,
                                   float* dscores, fg_stream stream);

/* ---------------------------------------------------------------- multi-GPU */
/*
 * Destination-row sharding (one process per GPU).  Each rank
 * owns rows [lo, hi) of A and of X (shard_offsets[r] .. shard_offsets[r+1]);
 * its local graph keeps GLOBAL source ids.  Before a local fg_spmm / fg_sddmm
 * the source features are all-gathered over NVLink with NCCL.
 *
 * fg_comm_init: communicator from an ncclUniqueId (128 bytes) the caller
 *   exchanged out of band (torch.distributed broadcast).  NCCL is loaded at
 *   run time (libnccl.so.2); FG_ENCCL if it is unavailable.
 * fg_comm_unique_id: fills 128 bytes with a fresh ncclUniqueId (rank 0).
 * fg_allgather_rows: X_full[shard_offsets[r] + i][:] = rank r's X_local[i][:]
 *   for every rank r (an all-gather-v of row blocks of `row_elems` fp32 each),
 *   enqueued on `stream`.  X_local may point inside X_full at this rank's block
 *   (in-place).  shard_offsets is a HOST int64[nranks+1].
 */
typedef struct fg_comm fg_comm;
fg_status fg_comm_unique_id(void* unique_id_128);
fg_status fg_comm_init(const void* unique_id_128, int nranks, int rank, fg_comm** out);
fg_status fg_comm_destroy(fg_comm* c);
/* fg_comm_info: the communicator's size and this rank as NCCL reports them
 * (ncclCommCount / ncclCommUserRank) -- the check that every rank joined. */
fg_status fg_comm_info(const fg_comm* c, int* nranks, int* rank);
fg_status fg_allgather_rows(fg_comm* c, const int64_t* shard_offsets, int64_t row_elems,
                            const float* X_local, float* X_full, fg_stream stream);
/*
 * fg_dist_spmm / fg_dist_sddmm -- the sharded ops: fg_allgather_rows of this
 *   rank's source-feature block X_local into X_full (device, [n_src][row]; the
 *   row is H*D floats, d_in for mlp), then fg_spmm / fg_sddmm on `local` (this
 *   rank's destination rows, GLOBAL source ids) reading X_full, both enqueued on
 *   `stream`.  Y_local / X_dst / out_local / arg_* / E are this rank's rows /
 *   edges; every other argument, shape rule and error as fg_spmm / fg_sddmm
 *   (copy_e: FG_EUNSUPPORTED, it gathers no source rows).  All argument checks
 *   of the local op run before the all-gather is enqueued (a non-OK status
 *   means nothing was launched and X_full is untouched).  Per-row results are
 *   bit-identical to the unsharded op when the local handle's automatic
 *   CTA-per-row threshold is computed from the whole graph's edge count
 *   (fg_graph_tune FG_TUNE_BALANCE_NNZ, which the sharding code sets), and
 *   for max / min / argmax always.
 */
fg_status fg_dist_spmm(const fg_graph* local, fg_comm* c, const int64_t* shard_offsets, fg_msg_op msg,
                       fg_reduce_op red, int H, int D, const float* X_local, float* X_full, const float* E,
                       const float* W, int d_in, const float* X_dst, float* out_local, int32_t* arg_u,
                       int32_t* arg_e, void* workspace, size_t workspace_bytes, fg_stream stream);
fg_status fg_dist_sddmm(const fg_graph* local, fg_comm* c, const int64_t* shard_offsets, fg_edge_op op, int H,
                        int D, const float* X_local, float* X_full, const float* Y_local, float* out_local,
                        fg_stream stream);

/* ---------------------------------------------------------------- errors */
const char* fg_status_string(fg_status s);
const char* fg_last_error(void);   /* thread-local detail of the last non-OK status */
int fg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FG_H_ */
