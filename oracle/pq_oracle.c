/*
 * pq_oracle.c — plain, slow, obviously-correct CPU oracle for PQTopK.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2408_09992_b200/csrc); neither includes the other.
 *
 * Citations: P:n = PAPER.md line n (arXiv 2408.09992 LaTeX), S:n = SPEC.md
 * line n, R<n> = reading n in DESIGN.md ("Readings of the paper").
 *
 * Precision (R5, R6, R7): Eq. 4 dot products accumulate in fp64 (fp32*fp32
 * products are exact in fp64); item scores (Eq. 5) are fp32 sums in split
 * order k = 0..m-1 starting from +0.0f, IEEE round-to-nearest, no FMA (none
 * is possible: only adds), no FTZ/DAZ (checked at run time), compiled with
 * -O2 -fno-fast-math -ffp-contract=off.
 *
 * Ranking (R3): score descending, then item id ascending; -0 and +0 compare
 * equal (they cannot both occur because the +0.0f start canonicalises -0).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <xmmintrin.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* 0 when the x87/SSE environment is IEEE (FTZ and DAZ clear), else the MXCSR. */
int orc_check_fpenv(void) {
    unsigned int csr = _mm_getcsr();
    return (csr & 0x8040u) ? (int)csr : 0;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count for the following calls (plumbing for the 1-thread timing; the
 * results do not depend on it: test_thread_count_invariance). */
void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------------------
 * Eq. 4: s_{k,j} = psi_{k,j} . phi_k, with phi_k the k-th contiguous
 * d/m chunk of phi (R10).  S64[u][k][g] in fp64, t ascending; C holds the
 * condition scale sum_t |psi*phi| used by the mixed tolerance (R5).
 * ------------------------------------------------------------------------- */
void orc_subscores64(const float* phi, const float* psi, int64_t B, int32_t d,
                     int32_t m, int32_t b, double* S64, double* C) {
    const int32_t dm = d / m;
    for (int64_t u = 0; u < B; ++u)
        for (int32_t k = 0; k < m; ++k)
            for (int32_t g = 0; g < b; ++g) {
                double s = 0.0, c = 0.0;
                for (int32_t t = 0; t < dm; ++t) {
                    double p = (double)psi[((int64_t)k * b + g) * dm + t] *
                               (double)phi[u * d + (int64_t)k * dm + t];
                    s += p;
                    c += fabs(p);
                }
                S64[(u * m + k) * b + g] = s;
                if (C) C[(u * m + k) * b + g] = c;
            }
}

/* ---------------------------------------------------------------------------
 * Eq. 5, Algorithm 1: item-major.  For every item:
 *   score = +0.0f; for k in 0..m-1: score = score + S[k][G[i][k]]   (fp32)
 * S is one user's [m][b] table.
 * ------------------------------------------------------------------------- */
void orc_scores_alg1(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                     const float* S, float* r) {
    (void)b;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        float score = 0.0f;
        for (int32_t k = 0; k < m; ++k)
            score = score + S[(int64_t)k * b + codes[i * m + k]];
        r[i] = score;
    }
}

/* Algorithm 2, RecJPQScore: split-major with an N-length
 * accumulator "initialised to 0"; the split loop is sequential. */
void orc_scores_alg2(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                     const float* S, float* r) {
    for (int64_t i = 0; i < N; ++i) r[i] = 0.0f;
    for (int32_t k = 0; k < m; ++k)
        for (int64_t i = 0; i < N; ++i)
            r[i] += S[(int64_t)k * b + codes[i * m + k]];
}

/* ---------------------------------------------------------------------------
 * TopK (Alg. 1): the first min(K, N) items of the
 * order (score desc, id asc).  Plain definition: sort all N, take a prefix.
 * ------------------------------------------------------------------------- */
typedef struct { float s; int64_t id; } orc_pair;
typedef struct { double s; int64_t id; } orc_pair64;

/* 1 when a ranks strictly before b. */
static int before(float as, int64_t aid, float bs, int64_t bid) {
    if (as > bs) return 1;
    if (as < bs) return 0;
    return aid < bid;
}
static int cmp_pair(const void* x, const void* y) {
    const orc_pair* a = (const orc_pair*)x; const orc_pair* c = (const orc_pair*)y;
    if (before(a->s, a->id, c->s, c->id)) return -1;
    if (before(c->s, c->id, a->s, a->id)) return 1;
    return 0;
}
static int cmp_pair64(const void* x, const void* y) {
    const orc_pair64* a = (const orc_pair64*)x; const orc_pair64* c = (const orc_pair64*)y;
    if (a->s > c->s) return -1;
    if (a->s < c->s) return 1;
    return (a->id < c->id) ? -1 : (a->id > c->id);
}

/* Writes min(K,N) entries; slots [min(K,N), K) get id -1, score -inf (R11).
 * Returns the number of valid entries, or -1 on allocation failure. */
int64_t orc_topk_sort(const float* r, int64_t N, int64_t K, int64_t id_base,
                      int32_t* ids, float* scores) {
    orc_pair* a = (orc_pair*)malloc(sizeof(orc_pair) * (size_t)(N > 0 ? N : 1));
    if (!a) return -1;
    for (int64_t i = 0; i < N; ++i) { a[i].s = r[i]; a[i].id = id_base + i; }
    qsort(a, (size_t)N, sizeof(orc_pair), cmp_pair);
    int64_t n = K < N ? K : N;
    for (int64_t j = 0; j < K; ++j) {
        ids[j] = j < n ? (int32_t)a[j].id : -1;
        scores[j] = j < n ? a[j].s : -INFINITY;
    }
    free(a);
    return n;
}

int64_t orc_topk_sort64(const double* r, int64_t N, int64_t K, int64_t id_base,
                        int32_t* ids, double* scores) {
    orc_pair64* a = (orc_pair64*)malloc(sizeof(orc_pair64) * (size_t)(N > 0 ? N : 1));
    if (!a) return -1;
    for (int64_t i = 0; i < N; ++i) { a[i].s = r[i]; a[i].id = id_base + i; }
    qsort(a, (size_t)N, sizeof(orc_pair64), cmp_pair64);
    int64_t n = K < N ? K : N;
    for (int64_t j = 0; j < K; ++j) {
        ids[j] = j < n ? (int32_t)a[j].id : -1;
        scores[j] = j < n ? a[j].s : -INFINITY;
    }
    free(a);
    return n;
}

/* ---------------------------------------------------------------------------
 * PQTopK (Algorithm 1) for a batch of users, without an N-length
 * score array: each thread keeps the best K of its items in a bounded binary
 * heap whose root is the worst kept entry (order: before()); the per-thread
 * heaps are then merged by a full sort.  The result is independent of the
 * thread count because the (score, id) order is total.
 * S is [B][m][b]; ids/scores are [B][K].
 * ------------------------------------------------------------------------- */
static void heap_sift_down(orc_pair* h, int64_t n, int64_t i) {
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, w = i;   /* w = worst of i, l, r */
        if (l < n && before(h[w].s, h[w].id, h[l].s, h[l].id)) w = l;
        if (r < n && before(h[w].s, h[w].id, h[r].s, h[r].id)) w = r;
        if (w == i) return;
        orc_pair t = h[i]; h[i] = h[w]; h[w] = t; i = w;
    }
}
static void heap_sift_up(orc_pair* h, int64_t i) {
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!before(h[p].s, h[p].id, h[i].s, h[i].id)) return;
        orc_pair t = h[i]; h[i] = h[p]; h[p] = t; i = p;
    }
}

int orc_pq_topk(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                const float* S, int64_t B, int64_t K, int64_t id_base,
                int32_t* ids, float* scores) {
    if (K <= 0 || B <= 0) return 0;
    int nt = orc_max_threads();
    orc_pair* heaps = (orc_pair*)malloc(sizeof(orc_pair) * (size_t)(nt * K));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)nt);
    orc_pair* all = (orc_pair*)malloc(sizeof(orc_pair) * (size_t)(nt * K));
    if (!heaps || !fill || !all) { free(heaps); free(fill); free(all); return -1; }
    for (int64_t u = 0; u < B; ++u) {
        const float* Su = S + u * (int64_t)m * b;
        for (int t = 0; t < nt; ++t) fill[t] = 0;
        #pragma omp parallel num_threads(nt)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            orc_pair* h = heaps + (int64_t)t * K;
            int64_t n = 0;
            #pragma omp for schedule(static)
            for (int64_t i = 0; i < N; ++i) {
                float score = 0.0f;                       /* Alg. 1 */
                for (int32_t k = 0; k < m; ++k)           /* Alg. 1 */
                    score = score + Su[(int64_t)k * b + codes[i * m + k]];
                int64_t id = id_base + i;
                if (n < K) { h[n].s = score; h[n].id = id; heap_sift_up(h, n); ++n; }
                else if (before(score, id, h[0].s, h[0].id)) {
                    h[0].s = score; h[0].id = id; heap_sift_down(h, n, 0);
                }
            }
            fill[t] = n;
        }
        int64_t tot = 0;
        for (int t = 0; t < nt; ++t) {
            memcpy(all + tot, heaps + (int64_t)t * K, sizeof(orc_pair) * (size_t)fill[t]);
            tot += fill[t];
        }
        qsort(all, (size_t)tot, sizeof(orc_pair), cmp_pair);     /* TopK */
        for (int64_t j = 0; j < K; ++j) {
            ids[u * K + j] = j < tot ? (int32_t)all[j].id : -1;
            scores[u * K + j] = j < tot ? all[j].s : -INFINITY;
        }
    }
    free(heaps); free(fill); free(all);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Dense baseline (Eq. 2; Eq. 3).
 * Reconstruction: w_i = psi_{1,g_i1} || ... || psi_{m,g_im}.
 * ------------------------------------------------------------------------- */
void orc_reconstruct(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                     const float* psi, int32_t d, float* W) {
    const int32_t dm = d / m;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i)
        for (int32_t k = 0; k < m; ++k)
            for (int32_t t = 0; t < dm; ++t)
                W[i * d + (int64_t)k * dm + t] =
                    psi[((int64_t)k * b + codes[i * m + k]) * dm + t];
}

/* r64[i] = w_i . phi in fp64 (t ascending over the reconstructed row). */
void orc_dense_scores64(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                        const float* psi, int32_t d, const float* phi, double* r64) {
    const int32_t dm = d / m;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        double s = 0.0;
        for (int32_t k = 0; k < m; ++k)
            for (int32_t t = 0; t < dm; ++t)
                s += (double)psi[((int64_t)k * b + codes[i * m + k]) * dm + t] *
                     (double)phi[(int64_t)k * dm + t];
        r64[i] = s;
    }
}

/* ---------------------------------------------------------------------------
 * Tuple-bucket top-K: an independent algorithm for b^m small (SURVEY §8(c)
 * step 5), used to pin the tie handling of the C5 config.
 *   1. score each of the T = b^m code tuples with the fp32 k-ordered sum;
 *   2. bucket the items by tuple (counting sort: ids ascending per bucket);
 *   3. visit tuples by descending score; tuples whose fp32 scores are exactly
 *      equal form one group whose item ids are merged ascending;
 *   4. emit until K items are out.
 * tuple index t = sum_k g_k * b^(m-1-k).
 * ------------------------------------------------------------------------- */
typedef struct { float s; int64_t t; } orc_tup;
static int cmp_tup(const void* x, const void* y) {
    const orc_tup* a = (const orc_tup*)x; const orc_tup* c = (const orc_tup*)y;
    if (a->s > c->s) return -1;
    if (a->s < c->s) return 1;
    return (a->t < c->t) ? -1 : (a->t > c->t);
}
static int cmp_i64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, c = *(const int64_t*)y;
    return (a < c) ? -1 : (a > c);
}

int orc_tuple_topk(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                   const float* S, int64_t B, int64_t K, int64_t id_base,
                   int32_t* ids, float* scores) {
    int64_t T = 1;
    for (int32_t k = 0; k < m; ++k) { T *= b; if (T > (1 << 24)) return -2; }
    int64_t* start = (int64_t*)calloc((size_t)T + 1, sizeof(int64_t));
    int64_t* items = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    orc_tup* tup = (orc_tup*)malloc(sizeof(orc_tup) * (size_t)T);
    int64_t* grp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    if (!start || !items || !tup || !grp) { free(start); free(items); free(tup); free(grp); return -1; }
    for (int64_t i = 0; i < N; ++i) {
        int64_t t = 0;
        for (int32_t k = 0; k < m; ++k) t = t * b + codes[i * m + k];
        start[t + 1]++;
    }
    for (int64_t t = 0; t < T; ++t) start[t + 1] += start[t];
    {
        int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)T);
        if (!pos) { free(start); free(items); free(tup); free(grp); return -1; }
        memcpy(pos, start, sizeof(int64_t) * (size_t)T);
        for (int64_t i = 0; i < N; ++i) {      /* stable: ids ascending per tuple */
            int64_t t = 0;
            for (int32_t k = 0; k < m; ++k) t = t * b + codes[i * m + k];
            items[pos[t]++] = i;
        }
        free(pos);
    }
    for (int64_t u = 0; u < B; ++u) {
        const float* Su = S + u * (int64_t)m * b;
        for (int64_t t = 0; t < T; ++t) {
            float s = 0.0f;
            int64_t rem = t;
            int32_t g[64];
            for (int32_t k = m - 1; k >= 0; --k) { g[k] = (int32_t)(rem % b); rem /= b; }
            for (int32_t k = 0; k < m; ++k) s = s + Su[(int64_t)k * b + g[k]];
            tup[t].s = s; tup[t].t = t;
        }
        qsort(tup, (size_t)T, sizeof(orc_tup), cmp_tup);
        int64_t out = 0, j = 0;
        while (out < K && j < T) {
            int64_t e = j, n = 0;
            while (e < T && tup[e].s == tup[j].s) ++e;        /* equal-score group */
            for (int64_t q = j; q < e; ++q) {
                int64_t t = tup[q].t;
                for (int64_t p = start[t]; p < start[t + 1]; ++p) grp[n++] = items[p];
            }
            qsort(grp, (size_t)n, sizeof(int64_t), cmp_i64);
            for (int64_t q = 0; q < n && out < K; ++q, ++out) {
                ids[u * K + out] = (int32_t)(id_base + grp[q]);
                scores[u * K + out] = tup[j].s;
            }
            j = e;
        }
        for (; out < K; ++out) { ids[u * K + out] = -1; scores[u * K + out] = -INFINITY; }
    }
    free(start); free(items); free(tup); free(grp);
    return 0;
}
