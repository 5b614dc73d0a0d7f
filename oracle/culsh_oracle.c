/*
 * culsh_oracle.c -- CPU restatement of the reference CULSH-MF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2111_11682_b200/) never links, imports or calls it.
 *
 * Every function restates one numba kernel of the reference package
 * (/root/reference/pkg/src/lshmf/<module>.py) in plain C with the same operation
 * order.  All floating point is IEEE binary64 with contraction disabled
 * (-ffp-contract=off), matching numba's fastmath-off code (no FMA).
 *
 * Pinned against the reference: the tests/golden fixtures were produced by the
 * reference itself (tests/golden/make_golden.py) and tests/test_oracle.py
 * checks this file bit-for-bit against them.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

/* Minimal pthread parallel-for (the reference uses numba prange / a thread pool). */
typedef void (*pf_body_t)(int64_t lo, int64_t hi, void *ctx);
typedef struct { pf_body_t body; void *ctx; int64_t n, chunk; volatile int64_t *next; } pf_arg_t;

static void *pf_worker(void *p) {
    pf_arg_t *a = (pf_arg_t *)p;
    for (;;) {
        int64_t lo = __atomic_fetch_add(a->next, a->chunk, __ATOMIC_RELAXED);
        if (lo >= a->n) break;
        int64_t hi = lo + a->chunk < a->n ? lo + a->chunk : a->n;
        a->body(lo, hi, a->ctx);
    }
    return NULL;
}

static void parallel_for(int64_t n, int64_t chunk, int nthreads, pf_body_t body, void *ctx) {
    if (nthreads <= 1 || n <= chunk) { if (n > 0) body(0, n, ctx); return; }
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    volatile int64_t next = 0;
    pf_arg_t arg = {body, ctx, n, chunk, &next};
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, pf_worker, &arg);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

#define GOLDEN64 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL

/* lsh.py:53-58 _splitmix64 */
uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + GOLDEN64;
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

/* lsh.py:61-65 _map_key */
uint64_t orc_map_key(uint64_t seed, int64_t g, int64_t m) {
    uint64_t h = orc_splitmix64(seed);
    h = orc_splitmix64(h ^ ((uint64_t)(g + 1) * GOLDEN64));
    return orc_splitmix64(h ^ ((uint64_t)(m + 1) * MIX1));
}

/* lsh.py:68-78 _assign_bits: bits[i,g,m,t] = (sm(key(g,m) ^ i) >> t) & 1 */
void orc_assign_bits(uint64_t seed, int q, int p, int64_t M, int G, uint8_t *bits) {
    for (int g = 0; g < q; ++g)
        for (int m = 0; m < p; ++m) {
            uint64_t key = orc_map_key(seed, g, m);
            for (int64_t i = 0; i < M; ++i) {
                uint64_t h = orc_splitmix64(key ^ (uint64_t)i);
                uint8_t *dst = bits + (((i * q + g) * p + m) * (int64_t)G);
                for (int t = 0; t < G; ++t) dst[t] = (uint8_t)((h >> t) & 1ULL);
            }
        }
}

/* lsh.py:117-123 _psi */
static inline double psi_of(double v, int e) {
    if (e == 1) return v;
    if (e == 2) return v * v;
    return (v * v) * (v * v);
}

/* lsh.py:161-179 _accumulate_all (prange over columns -> parallel_for over columns) */
typedef struct {
    const int64_t *col_ptr; const int32_t *col_rows; const double *col_vals;
    const uint8_t *bits; int64_t W; int e; double *acc;
} acc_ctx_t;

/* a - ps == a + (-ps) in IEEE arithmetic, so the select form below is the reference's
 * if/else bit for bit; written branch-free it vectorises (numba's LLVM build of the
 * reference does the same), and target_clones picks AVX-512 / AVX2 on the host that
 * runs it (the .so is built in one container and run on another box). */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void acc_body(int64_t jlo, int64_t jhi, void *p) {
    const acc_ctx_t *c = (const acc_ctx_t *)p;
    const int64_t W = c->W;
    for (int64_t j = jlo; j < jhi; ++j) {
        double *restrict a = c->acc + j * W;
        for (int64_t w = 0; w < W; ++w) a[w] = 0.0;
        for (int64_t idx = c->col_ptr[j]; idx < c->col_ptr[j + 1]; ++idx) {
            const int64_t i = c->col_rows[idx];
            const double ps = psi_of(c->col_vals[idx], c->e), ng = -ps;
            const uint8_t *restrict b = c->bits + i * W;
            for (int64_t w = 0; w < W; ++w) a[w] += b[w] != 0 ? ps : ng;
        }
    }
}

void orc_accumulate_all(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                        int64_t N, const uint8_t *bits, int q, int p, int G, int e,
                        double *acc, int nthreads) {
    acc_ctx_t c = {col_ptr, col_rows, col_vals, bits, (int64_t)q * p * G, e, acc};
    parallel_for(N, 8, nthreads, acc_body, &c);
}

/* online.py:96-117 _accumulate_into (serial, ascending row within column) */
void orc_accumulate_into(double *acc, const int64_t *col_ptr, const int32_t *col_rows,
                         const double *col_vals, int64_t N, const uint8_t *bits,
                         int q, int p, int G, int e) {
    const int64_t W = (int64_t)q * p * G;
    for (int64_t j = 0; j < N; ++j) {
        double *a = acc + j * W;
        for (int64_t idx = col_ptr[j]; idx < col_ptr[j + 1]; ++idx) {
            const int64_t i = col_rows[idx];
            const double ps = psi_of(col_vals[idx], e);
            const uint8_t *b = bits + i * W;
            for (int64_t w = 0; w < W; ++w) {
                if (b[w] != 0) a[w] += ps; else a[w] -= ps;
            }
        }
    }
}

/* lsh.py:182-183 _threshold: sig = acc >= 0 */
/* Host threads for the stages below (set from Python; every stage's output is
 * independent of the thread count). */
static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n > 0 ? n : 1; }

typedef struct { const double *acc; uint8_t *sig; } thr_ctx_t;
static void thr_body(int64_t lo, int64_t hi, void *p) {
    const thr_ctx_t *c = (const thr_ctx_t *)p;
    for (int64_t k = lo; k < hi; ++k) c->sig[k] = c->acc[k] >= 0.0 ? 1 : 0;
}

void orc_threshold(const double *acc, int64_t n, uint8_t *sig) {
    thr_ctx_t c = {acc, sig};
    parallel_for(n, 1 << 20, g_threads, thr_body, &c);
}

/* lsh.py:246-260 _pack_group_keys over all groups (lsh.py:417-423): bit m*G+t of
 * group g's key is sig[j,g,m,t] */
typedef struct { const uint8_t *sig; int64_t N; int q, p, G; uint64_t *keys; } pack_ctx_t;
static void pack_body(int64_t jlo, int64_t jhi, void *pp) {
    const pack_ctx_t *c = (const pack_ctx_t *)pp;
    for (int64_t j = jlo; j < jhi; ++j)
        for (int g = 0; g < c->q; ++g) {
            uint64_t k = 0;
            unsigned shift = 0;
            const uint8_t *s = c->sig + ((j * c->q + g) * (int64_t)c->p) * c->G;
            for (int m = 0; m < c->p; ++m)
                for (int t = 0; t < c->G; ++t) {
                    if (s[m * c->G + t] != 0) k |= 1ULL << shift;
                    shift += 1;
                }
            c->keys[(int64_t)g * c->N + j] = k;
        }
}

void orc_pack_group_keys(const uint8_t *sig, int64_t N, int q, int p, int G, uint64_t *keys) {
    pack_ctx_t c = {sig, N, q, p, G, keys};
    parallel_for(N, 256, g_threads, pack_body, &c);
}

/* ---- bucketing: lsh.py:263-287 _group_runs (stable argsort) ---- */
typedef struct { uint64_t key; int64_t j; } kj_t;

static int cmp_kj(const void *a, const void *b) {
    const kj_t *x = (const kj_t *)a, *y = (const kj_t *)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->j < y->j) ? -1 : (x->j > y->j);   /* (key, index) order == stable argsort */
}

static void group_runs(const uint64_t *keys, int64_t N, int64_t *order,
                       int64_t *run_start, int64_t *run_end, kj_t *tmp) {
    for (int64_t j = 0; j < N; ++j) { tmp[j].key = keys[j]; tmp[j].j = j; }
    qsort(tmp, (size_t)N, sizeof(kj_t), cmp_kj);
    for (int64_t a = 0; a < N; ++a) order[a] = tmp[a].j;
    int64_t a = 0;
    while (a < N) {
        int64_t b = a + 1;
        while (b < N && tmp[b].key == tmp[a].key) ++b;
        for (int64_t x = a; x < b; ++x) { run_start[tmp[x].j] = a; run_end[tmp[x].j] = b; }
        a = b;
    }
}

/* similarity.py:137-161 _topk_insert: descending buffer, strict compares (ties keep
 * the earlier, i.e. lower, index ahead).  Returns the new count. */
static int topk_insert(double *best_sim, int32_t *best_idx, int count, int K, double s, int32_t j2) {
    int pos;
    if (count < K) {
        pos = count;
        while (pos > 0 && best_sim[pos - 1] < s) {
            best_sim[pos] = best_sim[pos - 1]; best_idx[pos] = best_idx[pos - 1]; --pos;
        }
        best_sim[pos] = s; best_idx[pos] = j2;
        return count + 1;
    }
    if (s > best_sim[K - 1]) {
        pos = K - 1;
        while (pos > 0 && best_sim[pos - 1] < s) {
            best_sim[pos] = best_sim[pos - 1]; best_idx[pos] = best_idx[pos - 1]; --pos;
        }
        best_sim[pos] = s; best_idx[pos] = j2;
    }
    return count;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* lsh.py:331-374 _fine_topk_core for one target column with its candidate list */
static void fine_topk_one(int32_t *cand, int64_t ncand, int64_t j, int K, uint64_t seed,
                          int64_t N_total, double *best_cnt, int32_t *best_idx, int32_t *out) {
    qsort(cand, (size_t)ncand, sizeof(int32_t), cmp_i32);
    int count = 0;
    int64_t a = 0;
    while (a < ncand) {
        int64_t b = a;
        while (b < ncand && cand[b] == cand[a]) ++b;
        count = topk_insert(best_cnt, best_idx, count, K, (double)(b - a), cand[a]);
        a = b;
    }
    if (count < K) {
        uint64_t key = orc_splitmix64(orc_splitmix64(seed ^ 0xC0FFEEULL) ^ (uint64_t)j);
        uint64_t t = 0;
        while (count < K) {
            uint64_t h = orc_splitmix64(key ^ t);
            t += 1;
            int32_t c = (int32_t)(h % (uint64_t)N_total);
            if (c == j) continue;
            int dup = 0;
            for (int x = 0; x < count; ++x) if (best_idx[x] == c) { dup = 1; break; }
            if (!dup) { best_idx[count] = c; best_cnt[count] = 0.0; ++count; }
        }
    }
    memcpy(out, best_idx, sizeof(int32_t) * (size_t)K);
}

/* lsh.py:401-414 _topk_from_group_keys, generalised with online.py:152-184
 * (j_base/n_cols target subset).  keys is (q, N_total).  entries is (n_cols, K).
 * Returns the total candidate count (sum over targets of bucket-1 over groups). */
typedef struct { const uint64_t *keys; int64_t N; int64_t *order, *rs, *re; } runs_ctx_t;
static void runs_body(int64_t glo, int64_t ghi, void *pp) {
    const runs_ctx_t *c = (const runs_ctx_t *)pp;
    kj_t *tmp = (kj_t *)malloc(sizeof(kj_t) * (size_t)(c->N > 0 ? c->N : 1));
    for (int64_t g = glo; g < ghi; ++g)
        group_runs(c->keys + g * c->N, c->N, c->order + g * c->N, c->rs + g * c->N, c->re + g * c->N, tmp);
    free(tmp);
}

typedef struct {
    const int64_t *order, *rs, *re, *offsets; int q; int64_t N_total, j_base; int K; uint64_t seed;
    int32_t *cand, *entries;
} fine_ctx_t;
static void fine_body(int64_t lo, int64_t hi, void *pp) {
    const fine_ctx_t *c = (const fine_ctx_t *)pp;
    double *best_cnt = (double *)malloc(sizeof(double) * (size_t)(c->K > 0 ? c->K : 1));
    int32_t *best_idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(c->K > 0 ? c->K : 1));
    for (int64_t jj = lo; jj < hi; ++jj) {
        const int64_t j = c->j_base + jj;
        int64_t f = c->offsets[jj];
        /* lsh.py:308-328 _fill_candidates: groups in order, bucket mates in sorted order */
        for (int g = 0; g < c->q; ++g) {
            const int64_t *og = c->order + (int64_t)g * c->N_total;
            for (int64_t pos = c->rs[(int64_t)g * c->N_total + j]; pos < c->re[(int64_t)g * c->N_total + j]; ++pos)
                if (og[pos] != j) c->cand[f++] = (int32_t)og[pos];
        }
        fine_topk_one(c->cand + c->offsets[jj], c->offsets[jj + 1] - c->offsets[jj], j, c->K, c->seed,
                      c->N_total, best_cnt, best_idx, c->entries + jj * (int64_t)c->K);
    }
    free(best_cnt); free(best_idx);
}

int64_t orc_topk_from_group_keys(const uint64_t *keys, int q, int64_t N_total, int64_t j_base,
                                 int64_t n_cols, int K, uint64_t seed, int32_t *entries) {
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)q * (size_t)N_total);
    int64_t *rs = (int64_t *)malloc(sizeof(int64_t) * (size_t)q * (size_t)N_total);
    int64_t *re = (int64_t *)malloc(sizeof(int64_t) * (size_t)q * (size_t)N_total);
    runs_ctx_t rc = {keys, N_total, order, rs, re};
    parallel_for(q, 1, g_threads, runs_body, &rc);
    /* lsh.py:308-328 _fill_candidates: offsets = prefix sum of sum_g (bucket - 1) */
    int64_t *offsets = (int64_t *)calloc((size_t)n_cols + 1, sizeof(int64_t));
    for (int64_t jj = 0; jj < n_cols; ++jj) {
        int64_t c = 0;
        for (int g = 0; g < q; ++g) {
            int64_t j = j_base + jj;
            c += re[(int64_t)g * N_total + j] - rs[(int64_t)g * N_total + j] - 1;
        }
        offsets[jj + 1] = offsets[jj] + c;
    }
    int64_t total = offsets[n_cols];
    int32_t *cand = (int32_t *)malloc(sizeof(int32_t) * (size_t)(total > 0 ? total : 1));
    fine_ctx_t fc = {order, rs, re, offsets, q, N_total, j_base, K, seed, cand, entries};
    parallel_for(n_cols, 64, g_threads, fine_body, &fc);
    free(cand); free(offsets);
    free(order); free(rs); free(re);
    return total;
}

/* ---------------------------------------------------------------- SGD ---- */

typedef struct {
    double gb, gbh, gu, gv, gw, gc;   /* rates   (b, b_hat, u, v, w, c) */
    double lb, lbh, lu, lv, lw, lc;   /* regularisers */
} orc_rates_t;

/* factorization.py:218-232 _lookup: binary search of j in row i's sorted CSR */
static inline double lookup(const int64_t *row_ptr, const int32_t *row_cols, const double *row_vals,
                            int64_t i, int64_t j, int *found) {
    int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        int64_t c = row_cols[mid];
        if (c == j) { *found = 1; return row_vals[mid]; }
        if (c < j) lo = mid + 1; else hi = mid;
    }
    *found = 0;
    return NAN;
}

typedef struct {
    const int64_t *row_ptr; const int32_t *row_cols; const double *row_vals;
    double mu; double *b, *bhat, *U, *V, *W, *C;
    const int32_t *nbr; int F, K;
    const double *base_b, *base_bhat;
} model_t;

/* factorization.py:235-263 _predict_one */
static double predict_one(const model_t *md, int64_t i, int64_t j) {
    const int F = md->F, K = md->K;
    double pred = md->mu + md->b[i] + md->bhat[j];
    double dot = 0.0;
    for (int f = 0; f < F; ++f) dot += md->U[i * F + f] * md->V[j * F + f];
    pred += dot;
    if (K > 0) {
        int64_t nr = 0, nn = 0;
        double sw = 0.0, sc = 0.0;
        for (int k = 0; k < K; ++k) {
            int64_t j1 = md->nbr[j * K + k];
            int found;
            double rv = lookup(md->row_ptr, md->row_cols, md->row_vals, i, j1, &found);
            if (!isnan(rv)) {
                nr += 1;
                sw += (rv - (md->mu + md->base_b[i] + md->base_bhat[j1])) * md->W[j * K + k];
            } else {
                nn += 1;
                sc += md->C[j * K + k];
            }
        }
        if (nr > 0) pred += sw / sqrt((double)nr);
        if (nn > 0) pred += sc / sqrt((double)nn);
    }
    return pred;
}

/* factorization.py:266-329 _update_one */
static double update_one(const model_t *md, int64_t i, int64_t j, double r, const orc_rates_t *rt,
                         int update_row, int update_col, uint8_t *expl, double *resid) {
    const int F = md->F, K = md->K;
    double *U = md->U, *V = md->V, *W = md->W, *C = md->C;
    double pred = md->mu + md->b[i] + md->bhat[j];
    double dot = 0.0;
    for (int f = 0; f < F; ++f) dot += U[i * F + f] * V[j * F + f];
    pred += dot;
    int64_t nr = 0, nn = 0;
    double sw = 0.0, sc = 0.0;
    for (int k = 0; k < K; ++k) {
        int64_t j1 = md->nbr[j * K + k];
        int found;
        double rv = lookup(md->row_ptr, md->row_cols, md->row_vals, i, j1, &found);
        if (!isnan(rv)) {
            expl[k] = 1;
            resid[k] = rv - (md->mu + md->base_b[i] + md->base_bhat[j1]);
            nr += 1;
            sw += resid[k] * W[j * K + k];
        } else {
            expl[k] = 0;
            nn += 1;
            sc += C[j * K + k];
        }
    }
    if (nr > 0) pred += sw / sqrt((double)nr);
    if (nn > 0) pred += sc / sqrt((double)nn);
    const double e = r - pred;
    const double inv_r = nr > 0 ? 1.0 / sqrt((double)nr) : 0.0;
    const double inv_n = nn > 0 ? 1.0 / sqrt((double)nn) : 0.0;
    if (update_row) md->b[i] += rt->gb * (e - rt->lb * md->b[i]);
    if (update_col) md->bhat[j] += rt->gbh * (e - rt->lbh * md->bhat[j]);
    if (update_row && update_col) {
        for (int f = 0; f < F; ++f) {
            double uf = U[i * F + f], vf = V[j * F + f];
            U[i * F + f] = uf + rt->gu * (e * vf - rt->lu * uf);
            V[j * F + f] = vf + rt->gv * (e * uf - rt->lv * vf);
        }
    } else if (update_row) {
        for (int f = 0; f < F; ++f)
            U[i * F + f] += rt->gu * (e * V[j * F + f] - rt->lu * U[i * F + f]);
    } else if (update_col) {
        for (int f = 0; f < F; ++f)
            V[j * F + f] += rt->gv * (e * U[i * F + f] - rt->lv * V[j * F + f]);
    }
    if (update_col) {
        for (int k = 0; k < K; ++k) {
            if (expl[k] != 0) W[j * K + k] += rt->gw * (inv_r * e * resid[k] - rt->lw * W[j * K + k]);
            else C[j * K + k] += rt->gc * (inv_n * e - rt->lc * C[j * K + k]);
        }
    }
    return e;
}

static int64_t lower_bound_i32(const int32_t *a, int64_t lo, int64_t hi, int64_t v) {
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

#define MODEL_ARGS \
    const int64_t *row_ptr, const int32_t *row_cols, const double *row_vals, \
    double mu, double *b, double *bhat, double *U, double *V, double *W, double *C, \
    const int32_t *nbr, int F, int K, const double *base_b, const double *base_bhat

#define MODEL_INIT \
    model_t md = {row_ptr, row_cols, row_vals, mu, b, bhat, U, V, W, C, nbr, F, K, base_b, base_bhat}; \
    uint8_t expl_buf[4096]; double resid_buf[4096]; \
    if (K > 4096) return -1;

/* factorization.py:332-363 _full_pass_block.  Returns 0 or 1 (non-finite error). */
int orc_full_pass_block(int64_t col_lo, int64_t col_hi, int64_t row_lo, int64_t row_hi, int64_t M,
                        const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                        MODEL_ARGS, const orc_rates_t *rt, int update_row, int update_col) {
    MODEL_INIT
    for (int64_t j = col_lo; j < col_hi; ++j) {
        int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        int64_t a = lo, c = hi;
        if (row_lo > 0) a = lower_bound_i32(col_rows, lo, hi, row_lo);
        if (row_hi < M) c = lower_bound_i32(col_rows, lo, hi, row_hi);
        for (int64_t idx = a; idx < c; ++idx) {
            double e = update_one(&md, col_rows[idx], j, col_vals[idx], rt, update_row, update_col,
                                  expl_buf, resid_buf);
            if (!isfinite(e)) return 1;
        }
    }
    return 0;
}

/* parallel.py:55-64 _block_pointers: out (N, nb) */
void orc_block_pointers(const int64_t *col_ptr, const int32_t *col_rows, int64_t N,
                        const int64_t *row_bounds, int nb, int64_t *out) {
    for (int64_t j = 0; j < N; ++j)
        for (int r = 0; r < nb; ++r)
            out[j * nb + r] = lower_bound_i32(col_rows, col_ptr[j], col_ptr[j + 1], row_bounds[r]);
}

/* parallel.py:110-128 _stage_pass (one worker's block) */
int orc_stage_pass(int64_t col_lo, int64_t col_hi, int rb, const int64_t *block_ptr, int nb,
                   const int32_t *col_rows, const double *col_vals, MODEL_ARGS, const orc_rates_t *rt) {
    MODEL_INIT
    for (int64_t j = col_lo; j < col_hi; ++j)
        for (int64_t idx = block_ptr[j * nb + rb]; idx < block_ptr[j * nb + rb + 1]; ++idx) {
            double e = update_one(&md, col_rows[idx], j, col_vals[idx], rt, 1, 1, expl_buf, resid_buf);
            if (!isfinite(e)) return 1;
        }
    return 0;
}

/* parallel.py:166-227 parallel_train, one epoch: D stages, worker d takes row block
 * (d+s)%D of its own column block d; stages separated by a barrier (thread join).
 * Workers run on up to nthreads threads (the reference uses a D-thread pool). */
typedef struct {
    int D, s; const int64_t *col_bounds, *block_ptr; const int32_t *col_rows; const double *col_vals;
    const int64_t *row_ptr; const int32_t *row_cols; const double *row_vals;
    double mu; double *b, *bhat, *U, *V, *W, *C; const int32_t *nbr; int F, K;
    const double *base_b, *base_bhat; const orc_rates_t *rt; volatile int bad;
} stage_ctx_t;

static void stage_body(int64_t dlo, int64_t dhi, void *p) {
    stage_ctx_t *c = (stage_ctx_t *)p;
    for (int64_t d = dlo; d < dhi; ++d) {
        int rb = (int)((d + c->s) % c->D);
        int bad = orc_stage_pass(c->col_bounds[d], c->col_bounds[d + 1], rb, c->block_ptr, c->D + 1,
                                 c->col_rows, c->col_vals, c->row_ptr, c->row_cols, c->row_vals,
                                 c->mu, c->b, c->bhat, c->U, c->V, c->W, c->C, c->nbr, c->F, c->K,
                                 c->base_b, c->base_bhat, c->rt);
        if (bad) c->bad = 1;
    }
}

int orc_parallel_epoch(int D, const int64_t *col_bounds, const int64_t *block_ptr,
                       const int32_t *col_rows, const double *col_vals, MODEL_ARGS,
                       const orc_rates_t *rt, int nthreads) {
    stage_ctx_t c = {D, 0, col_bounds, block_ptr, col_rows, col_vals, row_ptr, row_cols, row_vals,
                     mu, b, bhat, U, V, W, C, nbr, F, K, base_b, base_bhat, rt, 0};
    for (int s = 0; s < D; ++s) {
        c.s = s;
        parallel_for(D, 1, nthreads < D ? nthreads : D, stage_body, &c);
        if (c.bad) return 1;
    }
    return 0;
}

/* online.py:230-250 _online_row_pass */
int orc_online_row_pass(int64_t row_lo, int64_t row_hi, int64_t N_old, MODEL_ARGS,
                        const orc_rates_t *rt) {
    MODEL_INIT
    for (int64_t i = row_lo; i < row_hi; ++i)
        for (int64_t idx = row_ptr[i]; idx < row_ptr[i + 1]; ++idx) {
            int64_t j = row_cols[idx];
            if (j >= N_old) continue;
            double e = update_one(&md, i, j, row_vals[idx], rt, 1, 0, expl_buf, resid_buf);
            if (!isfinite(e)) return 1;
        }
    return 0;
}

/* online.py:253-271 _online_col_pass */
int orc_online_col_pass(int64_t col_lo, int64_t col_hi, int64_t M_old,
                        const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                        MODEL_ARGS, const orc_rates_t *rt) {
    MODEL_INIT
    for (int64_t j = col_lo; j < col_hi; ++j)
        for (int64_t idx = col_ptr[j]; idx < col_ptr[j + 1]; ++idx) {
            int64_t i = col_rows[idx];
            double e = update_one(&md, i, j, col_vals[idx], rt, i >= M_old, 1, expl_buf, resid_buf);
            if (!isfinite(e)) return 1;
        }
    return 0;
}

/* factorization.py:394-409 _rmse_kernel */
double orc_rmse(const int32_t *t_rows, const int32_t *t_cols, const double *t_vals, int64_t n,
                const int64_t *row_ptr, const int32_t *row_cols, const double *row_vals,
                double mu, const double *b, const double *bhat, const double *U, const double *V,
                const double *W, const double *C, const int32_t *nbr, int F, int K,
                const double *base_b, const double *base_bhat,
                int do_clamp, double clamp_lo, double clamp_hi, double unscale) {
    model_t md = {row_ptr, row_cols, row_vals, mu, (double *)b, (double *)bhat, (double *)U,
                  (double *)V, (double *)W, (double *)C, nbr, F, K, base_b, base_bhat};
    double total = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        double pred = predict_one(&md, t_rows[k], t_cols[k]);
        if (do_clamp) {
            if (pred < clamp_lo) pred = clamp_lo;
            else if (pred > clamp_hi) pred = clamp_hi;
        }
        double d = (pred - t_vals[k]) * unscale;
        total += d * d;
    }
    return sqrt(total / (double)n);
}

/* factorization.py:235-263, one prediction (API: predict) */
double orc_predict(int64_t i, int64_t j, const int64_t *row_ptr, const int32_t *row_cols,
                   const double *row_vals, double mu, const double *b, const double *bhat,
                   const double *U, const double *V, const double *W, const double *C,
                   const int32_t *nbr, int F, int K, const double *base_b, const double *base_bhat) {
    model_t md = {row_ptr, row_cols, row_vals, mu, (double *)b, (double *)bhat, (double *)U,
                  (double *)V, (double *)W, (double *)C, nbr, F, K, base_b, base_bhat};
    return predict_one(&md, i, j);
}

/* factorization.py:366-391 _basic_pass: row-major basic MF over rows_subset (in that
 * order); pred = (use_biases ? mu + b_i + b_hat_j : 0) with the products added one by
 * one; returns 1 on the first non-finite error (before its update). */
int orc_basic_pass(const int64_t *rows_subset, int64_t n_rows, const int64_t *row_ptr,
                   const int32_t *row_cols, const double *row_vals, double mu, double *b, double *bhat,
                   double *U, double *V, int F, int use_biases, const orc_rates_t *rt) {
    for (int64_t ii = 0; ii < n_rows; ++ii) {
        const int64_t i = rows_subset[ii];
        for (int64_t idx = row_ptr[i]; idx < row_ptr[i + 1]; ++idx) {
            const int64_t j = row_cols[idx];
            double pred = 0.0;
            if (use_biases) pred = mu + b[i] + bhat[j];
            for (int f = 0; f < F; ++f) pred += U[i * F + f] * V[j * F + f];
            const double e = row_vals[idx] - pred;
            if (!isfinite(e)) return 1;
            if (use_biases) {
                b[i] += rt->gb * (e - rt->lb * b[i]);
                bhat[j] += rt->gbh * (e - rt->lbh * bhat[j]);
            }
            for (int f = 0; f < F; ++f) {
                const double uf = U[i * F + f], vf = V[j * F + f];
                U[i * F + f] = uf + rt->gu * (e * vf - rt->lu * uf);
                V[j * F + f] = vf + rt->gv * (e * uf - rt->lv * vf);
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------ similarity --- */

/* similarity.py:57-90 _pair_stats: co-rated statistics by a sorted merge, sums in
 * ascending row order.  out = {n, s1, s2, s12, q1, q2}. */
void orc_pair_stats(const int32_t *r1, const double *v1, int64_t n1, const int32_t *r2,
                    const double *v2, int64_t n2, double *out) {
    int64_t n = 0, a = 0, b = 0;
    double s1 = 0.0, s2 = 0.0, s12 = 0.0, q1 = 0.0, q2 = 0.0;
    while (a < n1 && b < n2) {
        if (r1[a] == r2[b]) {
            double x = v1[a], y = v2[b];
            n += 1; s1 += x; s2 += y; s12 += x * y; q1 += x * x; q2 += y * y;
            ++a; ++b;
        } else if (r1[a] < r2[b]) {
            ++a;
        } else {
            ++b;
        }
    }
    out[0] = (double)n; out[1] = s1; out[2] = s2; out[3] = s12; out[4] = q1; out[5] = q2;
}

/* similarity.py:93-107 _pearson_from_stats (same expression order, no contraction) */
double orc_pearson_from_stats(const double *st) {
    double n = st[0];
    if (n < 2) return 0.0;
    double cov = st[3] - st[1] * st[2] / n;
    double var1 = st[4] - st[1] * st[1] / n;
    double var2 = st[5] - st[2] * st[2] / n;
    if (var1 <= 0.0 || var2 <= 0.0) return 0.0;
    double rho = cov / sqrt(var1 * var2);
    if (rho > 1.0) rho = 1.0;
    else if (rho < -1.0) rho = -1.0;
    return rho;
}

/* similarity.py:128-135 / :175-178: n/(n+lambda) * rho, 0 without co-support */
static double shrunk_of(const double *st, double lambda_rho) {
    if (st[0] == 0.0) return 0.0;
    return st[0] / (st[0] + lambda_rho) * orc_pearson_from_stats(st);
}

typedef struct {
    const int64_t *col_ptr; const int32_t *col_rows; const double *col_vals;
    int64_t N; int K; double lambda_rho; int32_t *entries; const int64_t *targets;
} gsm_ctx_t;

static void gsm_body(int64_t lo, int64_t hi, void *p) {
    gsm_ctx_t *c = (gsm_ctx_t *)p;
    double *best_sim = (double *)malloc(sizeof(double) * (size_t)c->K);
    int32_t *best_idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)c->K);
    double st[6];
    for (int64_t t = lo; t < hi; ++t) {
        const int64_t j1 = c->targets ? c->targets[t] : t;
        int count = 0;
        const int64_t a0 = c->col_ptr[j1], a1 = c->col_ptr[j1 + 1];
        for (int64_t j2 = 0; j2 < c->N; ++j2) {
            if (j2 == j1) continue;
            const int64_t b0 = c->col_ptr[j2], b1 = c->col_ptr[j2 + 1];
            orc_pair_stats(c->col_rows + a0, c->col_vals + a0, a1 - a0, c->col_rows + b0,
                           c->col_vals + b0, b1 - b0, st);
            count = topk_insert(best_sim, best_idx, count, c->K, shrunk_of(st, c->lambda_rho), (int32_t)j2);
        }
        memcpy(c->entries + t * c->K, best_idx, sizeof(int32_t) * (size_t)c->K);
    }
    free(best_sim);
    free(best_idx);
}

/* similarity.py:164-185 _gsm_topk_kernel: exact all-pairs top-K, prange over j1 */
void orc_gsm_topk(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals, int64_t N,
                  int K, double lambda_rho, int32_t *entries, int nthreads) {
    gsm_ctx_t c = {col_ptr, col_rows, col_vals, N, K, lambda_rho, entries, NULL};
    parallel_for(N, 4, nthreads, gsm_body, &c);
}

/* the same for a subset of target columns (all N candidates): entries (n_targets, K) */
void orc_gsm_topk_targets(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals, int64_t N,
                          const int64_t *targets, int64_t n_targets, int K, double lambda_rho,
                          int32_t *entries, int nthreads) {
    gsm_ctx_t c = {col_ptr, col_rows, col_vals, N, K, lambda_rho, entries, targets};
    parallel_for(n_targets, 1, nthreads, gsm_body, &c);
}
