/*
 * oracle/oracle.c -- plain, slow, obviously-correct fp64 CPU reference for the
 * FeatGraph hot path (arXiv 2008.11359).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  It shares no code, header, table or constant with the CUDA path
 * (paper_2008_11359_b200/csrc); the two meet only at the seeded inputs of gen/.
 *
 * Every routine is a direct per-edge loop in the order the paper writes the
 * computation, accumulating in fp64 ("direct per-edge
 * interpretation", "accumulate in f64"); OpenMP parallelises over
 * destination rows only (each row is an independent reduction).  No blocking,
 * no fusion, no reordering of a row's edges.
 *
 * Besides the value `ref`, each routine returns `abssum` = sum of |terms| for
 * every output element; it normalises the tolerance |gpu - ref| <= 1e-4 *
 * abssum (BASELINE.json north_star: "relative error of 1e-4 ... normalised by
 * the sum of absolute terms").
 *
 * Graph: destination-major CSR.  row v = [row_ptr[v], row_ptr[v+1]) lists the
 * sources u = col_idx[p] of the in-edges u->v (Eq. (1) reduces over N(v),
 * PAPER.md P:141-143; Eq. (3) H_V = A X_V).  The edge id of CSR position
 * p is eid[p] (eid == NULL: eid(p) = p); edge tensors are indexed by edge id
 * (SPEC.md S:23).
 *
 * Parity pins: tests/test_oracle_pins.py (dense A.X, masked max, complete-graph
 * X.Y^T, closed-form MLP max, adjoint identity, softmax invariants, SPEC
 * worked examples under tests/golden/).
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>

/* message ops (oracle's own numbering; the binding maps names to these) */
#define OR_COPY_U  0   /* phi = x_u                              P:252-254 (Fig. 3a) */
#define OR_U_MUL_E 1   /* phi = x_u[h,:] * x_uv[h]               P:375 (DGL builtin) */
#define OR_MLP     2   /* phi = ReLU((x_u + x_v) W)              P:289-296 (Fig. 3b) */
#define OR_U_ADD_E 3   /* phi = x_u[h,:] + x_uv[h]               DGL builtin family P:372-375 */
#define OR_COPY_E  4   /* phi = x_uv (edge feature row [F])      same family */
#define OR_SUM 0       /* aggregation: sum */
#define OR_MAX 1       /* aggregation: max                       P:56 (Fig. 1) */
#define OR_MIN 2       /* aggregation: min  (DGL builtin family) */
#define OR_MEAN 3      /* aggregation: mean = sum / |N(v)|  (same family)  */

static inline int64_t edge_id(const int32_t* eid, int64_t p) { return eid ? (int64_t)eid[p] : p; }

/*
 * Generalized SpMM, Eq. (1):  h_v = (+)_{u in N(v)} phi(x_u, x_v, x_uv)
 * evaluated for the listed destination rows (rows == NULL: all rows 0..n_rows-1).
 *
 * Output element (r, j), r = index into the row list, j < F:
 *   copy_u : t = X[u][j]                                   (F = H*D)
 *   u_mul_e: t = X[u][j] * E[eid][j / D]                   (F = H*D, E is [nnz][H])
 *   mlp    : t = max(0, sum_{k<d_in} (X[u][k] + X_dst[v][k]) * W[k][j])   (F = d2; Fig. 3b: ReLU
 *            applied after the full d1 contraction)
 *   u_add_e: t = X[u][j] + E[eid][j / D]                   (F = H*D, E is [nnz][H]); |t| := |x| + |e|
 *   copy_e : t = E[eid][j]                                 (F = H*D, E is [nnz][F]; X unused)
 *   sum: ref = sum over the row's edges in CSR order; abssum = sum |t| (mlp: sum_e sum_k |a_k W_kj|)
 *   max: ref = max_t with the FIRST edge (lowest CSR position) winning ties;
 *        u_mul_e compares the fp32-rounded product (the kernel's precision);
 *        abssum = |terms| of the winning message; arg_u/arg_e = col_idx / eid of the winner.
 *   min: as max with the comparison reversed (strict <: first wins).
 *   mean: ref = (sum over the row) / |N(v)|, abssum = (sum |t|) / |N(v)|.
 *   empty row: ref = +0.0, abssum = 0, arg = -1.
 */
void or_spmm(int64_t n_rows, const int64_t* rows, const int64_t* row_ptr, const int32_t* col_idx,
             const int32_t* eid, int op, int red, int H, int D,
             const float* X, const float* E, const float* W, int d_in, const float* X_dst,
             double* ref, double* abssum, int32_t* arg_u, int32_t* arg_e) {
    const int64_t F = (op == OR_MLP) ? (int64_t)D : (int64_t)H * D;
    #pragma omp parallel
    {
        int64_t* best = (int64_t*)malloc(sizeof(int64_t) * (size_t)(F > 0 ? F : 1));
        #pragma omp for schedule(dynamic, 16)
        for (int64_t r = 0; r < n_rows; ++r) {
            const int64_t v = rows ? rows[r] : r;
            double* acc = ref + r * F;          /* h_v, accumulated in place */
            double* ab = abssum + r * F;
            for (int64_t j = 0; j < F; ++j) {
                acc[j] = (red == OR_SUM || red == OR_MEAN) ? 0.0 : (red == OR_MIN ? INFINITY : -INFINITY);
                ab[j] = 0.0;
                best[j] = -1;
            }
            /* for each in-edge u -> v (ascending CSR position p): message phi, then (+) */
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                const int64_t u = col_idx[p];
                const int64_t e = edge_id(eid, p);
                for (int64_t j = 0; j < F; ++j) {
                    double t, t_abs;
                    if (op == OR_COPY_U) {
                        t = (double)X[u * F + j];
                        t_abs = fabs(t);
                    } else if (op == OR_U_MUL_E) {
                        t = (double)X[u * F + j] * (double)E[e * H + j / D];   /* exact in fp64 */
                        t_abs = fabs(t);
                    } else if (op == OR_U_ADD_E) {
                        t = (double)X[u * F + j] + (double)E[e * H + j / D];   /* exact in fp64 */
                        t_abs = fabs((double)X[u * F + j]) + fabs((double)E[e * H + j / D]);
                    } else if (op == OR_COPY_E) {
                        t = (double)E[e * F + j];
                        t_abs = fabs(t);
                    } else {
                        double z = 0.0; t_abs = 0.0;
                        for (int k = 0; k < d_in; ++k) {
                            double a = (double)X[u * d_in + k] + (double)X_dst[v * d_in + k];
                            double term = a * (double)W[(int64_t)k * F + j];
                            z += term; t_abs += fabs(term);
                        }
                        t = z > 0.0 ? z : 0.0;   /* ReLU = tvm.max(., 0), canonical +0.0 */
                    }
                    if (red == OR_SUM || red == OR_MEAN) {
                        acc[j] += t; ab[j] += t_abs;
                    } else {
                        /* u_mul_e / u_add_e compare the fp32-rounded message (the kernel's precision) */
                        double key = (op == OR_U_MUL_E || op == OR_U_ADD_E) ? (double)(float)t : t;
                        int better = (red == OR_MIN) ? (key < acc[j]) : (key > acc[j]);
                        if (better) { acc[j] = key; best[j] = p; ab[j] = t_abs; }  /* strict: first wins */
                    }
                }
            }
            const int64_t deg = row_ptr[v + 1] - row_ptr[v];
            for (int64_t j = 0; j < F; ++j) {
                if (deg == 0) { acc[j] = 0.0; ab[j] = 0.0; }
                else if (red == OR_MEAN) { acc[j] /= (double)deg; ab[j] /= (double)deg; }
                if (red == OR_MAX || red == OR_MIN) {
                    if (arg_u) arg_u[r * F + j] = best[j] < 0 ? -1 : col_idx[best[j]];
                    if (arg_e) arg_e[r * F + j] = best[j] < 0 ? -1 : (int32_t)edge_id(eid, best[j]);
                }
            }
        }
        free(best);
    }
}

/*
 * Generalized SDDMM, Eq. (2)/(4) with the dot-product edge function of Fig. 5a
 * and its multi-head form Fig. 5b:
 *   h_uv[h] = sum_{d<D} X[u][h][d] * Y[v][h][d]
 * for every edge of the listed rows, written at position o = (offset of row r in
 * the list) + (p - row_ptr[v]) of ref/abssum ([edges of listed rows][H]).
 * Heads are independent reductions.
 */
void or_sddmm(int64_t n_rows, const int64_t* rows, const int64_t* row_ptr, const int32_t* col_idx,
              int H, int D, const float* X, const float* Y, double* ref, double* abssum) {
    const int64_t F = (int64_t)H * D;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
    off[0] = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t v = rows ? rows[r] : r;
        off[r + 1] = off[r] + (row_ptr[v + 1] - row_ptr[v]);
    }
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < n_rows; ++r) {
        const int64_t v = rows ? rows[r] : r;
        for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
            const int64_t u = col_idx[p];
            const int64_t o = off[r] + (p - row_ptr[v]);
            for (int h = 0; h < H; ++h) {
                double s = 0.0, a = 0.0;
                for (int d = 0; d < D; ++d) {
                    double t = (double)X[u * F + (int64_t)h * D + d] * (double)Y[v * F + (int64_t)h * D + d];
                    s += t; a += fabs(t);
                }
                ref[o * H + h] = s;
                abssum[o * H + h] = a;
            }
        }
    }
    free(off);
}

/*
 * u_dot_v followed by e_mul (row f4: the DGL builtin pair the paper's SDDMM
 * template covers): the per-edge, per-head score of Eq. (4) scaled by
 * an edge tensor, as written:
 *     out[e][h] = ( sum_{d<D} X[u][h][d] * Y[v][h][d] ) * E[e][h],  e = eid(p)
 * fp64; abssum = (sum_d |X*Y|) * |E[e][h]|.  Emitted at the listed-row CSR
 * position like or_sddmm (E is indexed by edge id: eid[p], or p when eid is NULL).
 */
void or_sddmm_emul(int64_t n_rows, const int64_t* rows, const int64_t* row_ptr, const int32_t* col_idx,
                   const int32_t* eid, int H, int D, const float* X, const float* Y, const float* E,
                   double* ref, double* abssum) {
    const int64_t F = (int64_t)H * D;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
    off[0] = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t v = rows ? rows[r] : r;
        off[r + 1] = off[r] + (row_ptr[v + 1] - row_ptr[v]);
    }
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < n_rows; ++r) {
        const int64_t v = rows ? rows[r] : r;
        for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
            const int64_t u = col_idx[p];
            const int64_t e = eid ? (int64_t)eid[p] : p;
            const int64_t o = off[r] + (p - row_ptr[v]);
            for (int h = 0; h < H; ++h) {
                double s = 0.0, a = 0.0;
                for (int d = 0; d < D; ++d) {
                    double t = (double)X[u * F + (int64_t)h * D + d] * (double)Y[v * F + (int64_t)h * D + d];
                    s += t; a += fabs(t);
                }
                const double w = (double)E[e * H + h];
                ref[o * H + h] = s * w;
                abssum[o * H + h] = a * fabs(w);
            }
        }
    }
    free(off);
}

/*
 * Elementwise SDDMM edge functions (the u_OP_v members of the DGL builtin
 * family the paper plugs into): Eq. (2) with
 *   psi(x_u, x_v)[j] = X[u][j] OP Y[v][j],  OP in {add (0), sub (1), mul (2)}
 * for every edge of the listed rows, written at the listed-row position o
 * like or_sddmm: ref/abssum [edges of listed rows][F]; abssum = |x| OP' |y|
 * (add/sub: |x| + |y|, mul: |x y|).
 */
void or_sddmm_binary(int64_t n_rows, const int64_t* rows, const int64_t* row_ptr, const int32_t* col_idx,
                     int bop, int64_t F, const float* X, const float* Y, double* ref, double* abssum) {
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
    off[0] = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t v = rows ? rows[r] : r;
        off[r + 1] = off[r] + (row_ptr[v + 1] - row_ptr[v]);
    }
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < n_rows; ++r) {
        const int64_t v = rows ? rows[r] : r;
        for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
            const int64_t u = col_idx[p];
            const int64_t o = off[r] + (p - row_ptr[v]);
            for (int64_t j = 0; j < F; ++j) {
                const double x = (double)X[u * F + j], y = (double)Y[v * F + j];
                double t;
                if (bop == 0) t = x + y;
                else if (bop == 1) t = x - y;
                else t = x * y;
                ref[o * F + j] = t;
                abssum[o * F + j] = (bop == 2) ? fabs(t) : fabs(x) + fabs(y);
            }
        }
    }
    free(off);
}

/*
 * Edge softmax over the in-edges of each destination, per head (not in the
 * paper; the standard GAT / DGL definition needed by the GAT layer, P:983;
 * SURVEY L6):  alpha[p][h] = exp(s[p][h] - mx) / sum_q exp(s[q][h] - mx),
 * mx = max_q s[q][h], q over the row of p.  Scores are read at edge id eid(p)
 * (S[eid][h]); alpha is written at the listed-row position like or_sddmm.
 */
void or_edge_softmax(int64_t n_rows, const int64_t* rows, const int64_t* row_ptr, const int32_t* eid,
                     int H, const float* S, double* alpha) {
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
    off[0] = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t v = rows ? rows[r] : r;
        off[r + 1] = off[r] + (row_ptr[v + 1] - row_ptr[v]);
    }
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < n_rows; ++r) {
        const int64_t v = rows ? rows[r] : r;
        for (int h = 0; h < H; ++h) {
            double mx = -INFINITY, sum = 0.0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                double s = (double)S[edge_id(eid, p) * H + h];
                if (s > mx) mx = s;
            }
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p)
                sum += exp((double)S[edge_id(eid, p) * H + h] - mx);
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                const int64_t o = off[r] + (p - row_ptr[v]);
                alpha[o * H + h] = exp((double)S[edge_id(eid, p) * H + h] - mx) / sum;
            }
        }
    }
    free(off);
}

/* ======================================================================
 * Backward (gradients) -- the gradient duality of PAPER.md P:171-173 ("the
 * gradient computation of SpMM with respect to A requires a dot product ...
 * thus following the SDDMM pattern; likewise the gradient computation of
 * SDDMM follows the SpMM pattern"), written as the chain rule per edge.
 * All over the ORIGINAL graph (edge p = u -> v of row v); accumulations in
 * fp64; dX / dY / dE are zeroed here.  Pinned by torch autograd on dense
 * formulations (tests/test_oracle_backward.py).
 * ====================================================================== */

/* d/dX and d/dE of Eq. (1) for copy_u / u_mul_e with sum or max.
 * sum : dX[u][j] += dOut[v][j] * (u_mul_e ? E[e][j/D] : 1)
 *       dE[e][h] += sum_{d<D} dOut[v][h*D+d] * X[u][h*D+d]           (u_mul_e)
 * max : only the winning edge of (v, j) (arg_u[v][j] = its source, the
 *       forward's first-wins argmax; -1 for empty rows) gets the gradient.
 * min : as max (arg_u = the first-wins argmin).
 * mean: as sum with dOut[v][j] / |N(v)| in place of dOut[v][j]. */
void or_spmm_backward(int64_t n_dst, int64_t n_src, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                      const int32_t* eid, int op, int red, int H, int D, const float* X, const float* E,
                      const float* dOut, const int32_t* arg_u, double* dX, double* dE) {
    const int64_t F = (int64_t)H * D;
    if (dX) for (int64_t i = 0; i < n_src * F; ++i) dX[i] = 0.0;
    if (dE) for (int64_t i = 0; i < nnz * H; ++i) dE[i] = 0.0;
    for (int64_t v = 0; v < n_dst; ++v) {
        for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
            const int64_t u = col_idx[p];
            const int64_t e = edge_id(eid, p);
            for (int64_t j = 0; j < F; ++j) {
                if ((red == OR_MAX || red == OR_MIN) && arg_u[v * F + j] != u) continue;   /* not the winner */
                double g = (double)dOut[v * F + j];
                if (red == OR_MEAN) g /= (double)(row_ptr[v + 1] - row_ptr[v]);
                const double w = (op == OR_U_MUL_E) ? (double)E[e * H + j / D] : 1.0;
                if (dX) dX[u * F + j] += g * w;
                if (dE && op == OR_U_MUL_E) dE[e * H + j / D] += g * (double)X[u * F + j];
            }
        }
    }
}

/* d/dX and d/dY of Eq. (4) u_dot_v: s[e][h] = sum_d X[u][h,d] Y[v][h,d]. */
void or_sddmm_backward(int64_t n_dst, int64_t n_src, const int64_t* row_ptr, const int32_t* col_idx,
                       const int32_t* eid, int H, int D, const float* X, const float* Y, const float* dS,
                       double* dX, double* dY) {
    const int64_t F = (int64_t)H * D;
    if (dX) for (int64_t i = 0; i < n_src * F; ++i) dX[i] = 0.0;
    if (dY) for (int64_t i = 0; i < n_dst * F; ++i) dY[i] = 0.0;
    for (int64_t v = 0; v < n_dst; ++v)
        for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
            const int64_t u = col_idx[p];
            const int64_t e = edge_id(eid, p);
            for (int h = 0; h < H; ++h) {
                const double g = (double)dS[e * H + h];
                for (int d = 0; d < D; ++d) {
                    const int64_t j = (int64_t)h * D + d;
                    if (dX) dX[u * F + j] += g * (double)Y[v * F + j];
                    if (dY) dY[v * F + j] += g * (double)X[u * F + j];
                }
            }
        }
}

/* d/ds of the edge softmax: ds[e][h] = alpha[e][h] * (dalpha[e][h] - sum_{e' in row} alpha[e'][h] dalpha[e'][h]). */
void or_edge_softmax_backward(int64_t n_dst, const int64_t* row_ptr, const int32_t* eid, int H, const float* alpha,
                              const float* dalpha, double* ds) {
    for (int64_t v = 0; v < n_dst; ++v)
        for (int h = 0; h < H; ++h) {
            double dot = 0.0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                const int64_t e = edge_id(eid, p);
                dot += (double)alpha[e * H + h] * (double)dalpha[e * H + h];
            }
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                const int64_t e = edge_id(eid, p);
                ds[e * H + h] = (double)alpha[e * H + h] * ((double)dalpha[e * H + h] - dot);
            }
        }
}

/* ======================================================================
 * GAT attention layer as one definition (fused path f2): for each
 * destination v and head h, the composition of Eq. (4) (u_dot_v score),
 * the edge softmax over v's in-edges and Eq. (1) with the u_mul_e message
 * (P:983), all in fp64:
 *   s_e = sum_d X[u][h,d] Y[v][h,d];  a_e = exp(s_e - max s) / sum exp(. - max s);
 *   ref[v][h,d] = sum_e a_e X[u][h,d];  abssum = sum_e a_e |X[u][h,d]|.
 * ====================================================================== */
void or_gat(int64_t n_dst, const int64_t* row_ptr, const int32_t* col_idx, int H, int D, const float* X,
            const float* Y, double* ref, double* abssum) {
    const int64_t F = (int64_t)H * D;
    #pragma omp parallel
    {
        double* s = NULL;
        int64_t cap = 0;
        #pragma omp for schedule(dynamic, 16)
        for (int64_t v = 0; v < n_dst; ++v) {
            const int64_t deg = row_ptr[v + 1] - row_ptr[v];
            if (deg > cap) { cap = deg; s = (double*)realloc(s, sizeof(double) * (size_t)cap); }
            for (int64_t j = 0; j < F; ++j) { ref[v * F + j] = 0.0; abssum[v * F + j] = 0.0; }
            if (deg == 0) continue;
            for (int h = 0; h < H; ++h) {
                double mx = -INFINITY, sum = 0.0;
                for (int64_t k = 0; k < deg; ++k) {
                    const int64_t u = col_idx[row_ptr[v] + k];
                    double t = 0.0;
                    for (int d = 0; d < D; ++d)
                        t += (double)X[u * F + (int64_t)h * D + d] * (double)Y[v * F + (int64_t)h * D + d];
                    s[k] = t;
                    if (t > mx) mx = t;
                }
                for (int64_t k = 0; k < deg; ++k) sum += exp(s[k] - mx);
                for (int64_t k = 0; k < deg; ++k) {
                    const int64_t u = col_idx[row_ptr[v] + k];
                    const double a = exp(s[k] - mx) / sum;
                    for (int d = 0; d < D; ++d) {
                        const int64_t j = (int64_t)h * D + d;
                        ref[v * F + j] += a * (double)X[u * F + j];
                        abssum[v * F + j] += a * fabs((double)X[u * F + j]);
                    }
                }
            }
        }
        free(s);
    }
}
