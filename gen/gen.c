/*
 * gen/gen.c -- seeded synthetic inputs shared by the oracle tests and the CUDA
 * path.  This file holds NONE of the method's arithmetic (no aggregation, no
 * dot products, no softmax): only counter-based random numbers, degree
 * sequences and neighbour sampling.  Recipe: DESIGN.md "Input recipe";
 * SURVEY.md §8(d) "Inputs".
 *
 * Determinism: every random number is splitmix64 of a (seed, stream, counter)
 * key, so each destination row draws from its own stream and the CSR is
 * byte-identical for any OpenMP thread count (SPEC.md S:71 determinism).
 *
 * Graph orientation: destination-major CSR, row v lists the in-neighbours u of
 * v sorted strictly ascending (Eq. (3) H = A X; "rows in
 * the adjacency matrix").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static inline uint64_t sm64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
/* key for (seed, stream); value i of that stream = sm64(key ^ sm64(i)) */
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return sm64(sm64(seed) ^ (stream * 0xD1B54A32D192ED03ULL));
}
static inline uint64_t draw(uint64_t key, uint64_t i) { return sm64(key ^ sm64(i + 0x632BE59BD9B4E019ULL)); }
static inline double u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); } /* [0,1) */

uint64_t fggen_rand_u64(uint64_t seed, uint64_t stream, uint64_t i) { return draw(stream_key(seed, stream), i); }

/* ---------------------------------------------------------------- features */
/* regime 0: real, U[-1,1) as multiples of 2^-23 (exact fp32);
 * regime 1: real, U[0,1) as multiples of 2^-24;
 * regime 2: integer uniform in [lo, hi] (stored as fp32, exact);
 * regime 3: real, U[-scale, scale) rounded to fp32 (used for W ~ U[-1/sqrt(d1), 1/sqrt(d1))). */
void fggen_features(int64_t count, uint64_t seed, uint64_t stream, int regime,
                    int64_t lo, int64_t hi, double scale, float* out) {
    uint64_t key = stream_key(seed, stream);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        uint64_t r = draw(key, (uint64_t)i);
        float v;
        if (regime == 0) {
            int64_t q = (int64_t)(r >> 40) - (1LL << 23);           /* [-2^23, 2^23) */
            v = (float)ldexp((double)q, -23);
        } else if (regime == 1) {
            v = (float)ldexp((double)(r >> 40), -24);
        } else if (regime == 2) {
            uint64_t span = (uint64_t)(hi - lo + 1);
            v = (float)(lo + (int64_t)(r % span));
        } else {
            int64_t q = (int64_t)(r >> 40) - (1LL << 23);
            v = (float)(ldexp((double)q, -23) * scale);
        }
        out[i] = v;
    }
}

/* ------------------------------------------------------------ degree sequences */
typedef struct { double frac; int64_t idx; } frac_t;
static int cmp_frac(const void* pa, const void* pb) {
    const frac_t* a = (const frac_t*)pa; const frac_t* b = (const frac_t*)pb;
    if (a->frac > b->frac) return -1;
    if (a->frac < b->frac) return 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* Lognormal in-degrees, rescaled and clipped to [dmin, dmax] so they sum to m
 * EXACTLY (largest-remainder rounding).  SURVEY §8(c) L11 (a proposal, not the
 * paper's: the paper gives only |V|, |E| and the average degree, Table
 * tab:dataset P:614-618).  Returns 0 on success, -1 if m is unreachable. */
int fggen_degrees_lognormal(int64_t n, int64_t m, double sigma, int64_t dmin, int64_t dmax,
                            uint64_t seed, int64_t* deg) {
    if (n <= 0) return m == 0 ? 0 : -1;
    if (m < n * dmin || m > n * dmax) return -1;
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    uint64_t key = stream_key(seed, 1);
    for (int64_t i = 0; i < n; ++i) {
        double u1 = u01(draw(key, 2 * (uint64_t)i)), u2 = u01(draw(key, 2 * (uint64_t)i + 1));
        if (u1 < 1e-300) u1 = 1e-300;
        double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        w[i] = exp(sigma * z);
    }
    /* bisection on the scale s: S(s) = sum clip(s*w_i) is monotone in s */
    double lo = 0.0, hi = 1.0;
    for (;;) {
        double S = 0; for (int64_t i = 0; i < n; ++i) S += clampd(hi * w[i], (double)dmin, (double)dmax);
        if (S >= (double)m) break;
        hi *= 2.0;
        if (hi > 1e300) { free(w); return -1; }
    }
    for (int it = 0; it < 200; ++it) {
        double mid = 0.5 * (lo + hi);
        double S = 0; for (int64_t i = 0; i < n; ++i) S += clampd(mid * w[i], (double)dmin, (double)dmax);
        if (S < (double)m) lo = mid; else hi = mid;
    }
    frac_t* fr = (frac_t*)malloc(sizeof(frac_t) * (size_t)n);
    int64_t tot = 0;
    for (int64_t i = 0; i < n; ++i) {
        double x = clampd(hi * w[i], (double)dmin, (double)dmax);
        int64_t f = (int64_t)floor(x);
        deg[i] = f; tot += f;
        fr[i].frac = (f < dmax) ? x - (double)f : -1.0; fr[i].idx = i;
    }
    int64_t rem = m - tot;
    if (rem > 0) {
        qsort(fr, (size_t)n, sizeof(frac_t), cmp_frac);
        for (int64_t k = 0; k < n && rem > 0; ++k) if (deg[fr[k].idx] < dmax) { deg[fr[k].idx]++; rem--; }
        /* (rem > 0 after one sweep cannot happen: m <= n*dmax and S(hi) >= m) */
        for (int64_t i = 0; i < n && rem > 0; ++i) while (deg[i] < dmax && rem > 0) { deg[i]++; rem--; }
    } else if (rem < 0) {
        /* S(hi) may exceed m by rounding; take back from the smallest fractions */
        qsort(fr, (size_t)n, sizeof(frac_t), cmp_frac);
        for (int64_t k = n - 1; k >= 0 && rem < 0; --k) if (deg[fr[k].idx] > dmin) { deg[fr[k].idx]--; rem++; }
    }
    free(fr); free(w);
    return rem == 0 ? 0 : -1;
}

/* Random permutation of [0, n) (sort by random 64-bit key, ties by index). */
typedef struct { uint64_t key; int64_t idx; } pkey_t;
static int cmp_pkey(const void* pa, const void* pb) {
    const pkey_t* a = (const pkey_t*)pa; const pkey_t* b = (const pkey_t*)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}
void fggen_permutation(int64_t n, uint64_t seed, uint64_t stream, int64_t* perm) {
    pkey_t* k = (pkey_t*)malloc(sizeof(pkey_t) * (size_t)(n > 0 ? n : 1));
    uint64_t key = stream_key(seed, stream);
    for (int64_t i = 0; i < n; ++i) { k[i].key = draw(key, (uint64_t)i); k[i].idx = i; }
    qsort(k, (size_t)n, sizeof(pkey_t), cmp_pkey);
    for (int64_t i = 0; i < n; ++i) perm[i] = k[i].idx;
    free(k);
}

/* rand-100K two-block degrees: n_high vertices of degree deg_high and n_low of
 * degree deg_low, block membership by a seeded permutation (PAPER.md P:601:
 * "20K vertices have an average degree of 2000 and the remaining 80K vertices
 * have an average degree of 100"; SURVEY L9 reads "average" as exact). */
void fggen_degrees_two_block(int64_t n_high, int64_t deg_high, int64_t n_low, int64_t deg_low,
                             uint64_t seed, int64_t* deg) {
    int64_t n = n_high + n_low;
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    fggen_permutation(n, seed, 2, perm);
    for (int64_t i = 0; i < n; ++i) deg[perm[i]] = (i < n_high) ? deg_high : deg_low;
    free(perm);
}

/* ------------------------------------------------------------- neighbour sampling */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b; return (x > y) - (x < y);
}
typedef struct { double key; int32_t idx; } es_t;
static int cmp_es(const void* pa, const void* pb) {
    const es_t* a = (const es_t*)pa; const es_t* b = (const es_t*)pb;
    if (a->key != b->key) return a->key > b->key ? -1 : 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

/* Fill a destination-major CSR: row v gets deg[v] DISTINCT sources in
 * [0, n_src), sorted ascending.  weights == NULL -> uniform sources; else
 * sources are drawn without replacement with probability proportional to
 * weights[u] (Chung-Lu).  Sparse rows: alias-table draws with
 * duplicate rejection; dense rows (4*deg >= n_src): Efraimidis-Spirakis keys.
 * row_ptr must be filled by the caller (prefix sum of deg).  Returns 0, or -1
 * if some deg[v] > n_src. */
int fggen_fill_csr(int64_t n_dst, int64_t n_src, const int64_t* deg, const double* weights,
                   uint64_t seed, const int64_t* row_ptr, int32_t* col_idx) {
    for (int64_t v = 0; v < n_dst; ++v) if (deg[v] > n_src || deg[v] < 0) return -1;
    /* Vose alias table */
    double* prob = NULL; int32_t* alias = NULL;
    if (weights) {
        prob = (double*)malloc(sizeof(double) * (size_t)n_src);
        alias = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_src);
        int32_t* small = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_src);
        int32_t* large = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_src);
        double tot = 0; for (int64_t u = 0; u < n_src; ++u) tot += weights[u];
        int64_t ns = 0, nl = 0;
        for (int64_t u = 0; u < n_src; ++u) {
            prob[u] = weights[u] * (double)n_src / tot; alias[u] = (int32_t)u;
            if (prob[u] < 1.0) small[ns++] = (int32_t)u; else large[nl++] = (int32_t)u;
        }
        while (ns > 0 && nl > 0) {
            int32_t s = small[--ns], l = large[nl - 1];
            alias[s] = l;
            prob[l] = (prob[l] + prob[s]) - 1.0;
            if (prob[l] < 1.0) { nl--; small[ns++] = l; }
        }
        while (nl > 0) prob[large[--nl]] = 1.0;
        while (ns > 0) prob[small[--ns]] = 1.0;
        free(small); free(large);
    }
    int err = 0;
    #pragma omp parallel
    {
        int32_t* buf = NULL; size_t cap = 0;
        es_t* es = NULL;
        #pragma omp for schedule(dynamic, 64)
        for (int64_t v = 0; v < n_dst; ++v) {
            int64_t d = deg[v];
            int32_t* out = col_idx + row_ptr[v];
            if (d == 0) continue;
            uint64_t key = stream_key(seed, 1000 + (uint64_t)v);
            uint64_t ctr = 0;
            if (4 * d >= n_src) {
                if (!es) es = (es_t*)malloc(sizeof(es_t) * (size_t)n_src);
                for (int64_t u = 0; u < n_src; ++u) {
                    double r = u01(draw(key, ctr++));
                    if (r < 1e-300) r = 1e-300;
                    double w = weights ? weights[u] : 1.0;
                    es[u].key = (w > 0) ? log(r) / w : -1e300 + (double)0;  /* larger key wins */
                    es[u].idx = (int32_t)u;
                }
                qsort(es, (size_t)n_src, sizeof(es_t), cmp_es);
                for (int64_t k = 0; k < d; ++k) out[k] = es[k].idx;
                qsort(out, (size_t)d, sizeof(int32_t), cmp_i32);
                continue;
            }
            if ((size_t)(2 * d) > cap) { cap = (size_t)(2 * d); buf = (int32_t*)realloc(buf, cap * sizeof(int32_t)); }
            int64_t have = 0;
            while (have < d) {
                int64_t need = d - have;
                for (int64_t k = 0; k < need; ++k) {
                    uint64_t r = draw(key, ctr++);
                    uint64_t col = ((r >> 32) * (uint64_t)n_src) >> 32;
                    int32_t u = (int32_t)col;
                    if (weights) {
                        double coin = (double)(r & 0xFFFFFFFFULL) * (1.0 / 4294967296.0);
                        if (coin >= prob[u]) u = alias[u];
                    }
                    buf[have + k] = u;
                }
                int64_t tot = have + need;
                qsort(buf, (size_t)tot, sizeof(int32_t), cmp_i32);
                int64_t w = 0;
                for (int64_t k = 0; k < tot; ++k) if (w == 0 || buf[k] != buf[w - 1]) buf[w++] = buf[k];
                have = w;
            }
            memcpy(out, buf, sizeof(int32_t) * (size_t)d);
        }
        free(buf); free(es);
    }
    free(prob); free(alias);
    return err;
}
