/*
 * datagen.c -- seeded synthetic labelled graphs for the BASELINE.json configs
 * (SURVEY.md §8(d)), plus per-label canonical CSR construction in the layout the
 * reference's LabeledGraph holds (int64 indptr/indices, rows sorted, duplicates
 * collapsed: sparse_bool.py:51-59, graph_store.py:161-176).
 *
 * This is input preparation, the analogue of graph_store.load_graph: it runs
 * before any timed region (cli.py:98-107) and feeds BOTH the CUDA engine and the
 * CPU oracle the same bytes.  Every random draw is a pure function of
 * (seed, stream, counter) -- no sequential RNG state -- so the output is
 * independent of the thread count, and the same integer arithmetic can be run
 * on the device later.
 *
 * Built as a plain host library (gcc -fopenmp) into librpq_datagen.so.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* splitmix64 finaliser */
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* counter-based draw: 64 random bits for (seed, stream, counter) */
static inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
    return mix64(mix64(seed * 0xD1B54A32D192ED03ULL + stream) ^ ctr);
}

/* uniform integer in [0, n) from 32 random bits (multiply-high) */
static inline uint32_t bounded(uint32_t r32, uint32_t n) {
    return (uint32_t)(((uint64_t)r32 * (uint64_t)n) >> 32);
}

EXPORT uint64_t rpqgen_draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
    return draw(seed, stream, ctr);
}

/* Zipf(s) CDF over nl ranks scaled to 2^32: thresholds[k] = floor(2^32 * cdf_k),
 * thresholds[nl-1] = 2^32.  Rank k (0-based) has weight (k+1)^-s. */
EXPORT void rpqgen_zipf_thresholds(int32_t nl, double s, uint64_t* thresholds) {
    double total = 0.0;
    for (int32_t k = 0; k < nl; ++k) total += pow((double)(k + 1), -s);
    double acc = 0.0;
    for (int32_t k = 0; k < nl; ++k) {
        acc += pow((double)(k + 1), -s);
        double t = floor(acc / total * 4294967296.0);
        thresholds[k] = (uint64_t)t;
    }
    thresholds[nl - 1] = 4294967296ULL;
}

static inline int32_t zipf_pick(uint32_t r32, const uint64_t* thr, int32_t nl) {
    int32_t lo = 0, hi = nl - 1; /* first k with r32 < thr[k] */
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if ((uint64_t)r32 < thr[mid]) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* ------------------------------------------------------------------------ */
/* parallel LSD radix sort of uint64 keys on the low `bits` bits             */
/* ------------------------------------------------------------------------ */

static void radix_sort_u64(uint64_t* keys, uint64_t* tmp, int64_t n, int bits) {
    const int DIGIT = 16;
    const int64_t NB = 1 << DIGIT;
    int nthreads = omp_get_max_threads();
    int64_t* hist = (int64_t*)calloc((size_t)nthreads * NB, sizeof(int64_t));
    uint64_t* src = keys;
    uint64_t* dst = tmp;
    int passes = (bits + DIGIT - 1) / DIGIT;
    for (int p = 0; p < passes; ++p) {
        int shift = p * DIGIT;
        memset(hist, 0, (size_t)nthreads * NB * sizeof(int64_t));
#pragma omp parallel num_threads(nthreads)
        {
            int t = omp_get_thread_num();
            int64_t lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
            int64_t* h = hist + (int64_t)t * NB;
            for (int64_t i = lo; i < hi; ++i) h[(src[i] >> shift) & (NB - 1)]++;
        }
        /* exclusive prefix over (digit, thread) so the sort stays stable */
        int64_t run = 0;
        for (int64_t d = 0; d < NB; ++d)
            for (int t = 0; t < nthreads; ++t) {
                int64_t c = hist[(int64_t)t * NB + d];
                hist[(int64_t)t * NB + d] = run;
                run += c;
            }
#pragma omp parallel num_threads(nthreads)
        {
            int t = omp_get_thread_num();
            int64_t lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
            int64_t* h = hist + (int64_t)t * NB;
            for (int64_t i = lo; i < hi; ++i) dst[h[(src[i] >> shift) & (NB - 1)]++] = src[i];
        }
        uint64_t* sw = src; src = dst; dst = sw;
    }
    if (src != keys) memcpy(keys, src, (size_t)n * sizeof(uint64_t));
    free(hist);
}

/* ------------------------------------------------------------------------ */
/* Erdos-Renyi (cfg1): ne directed edges, uniform endpoints, uniform labels.  */
/* Self-loops and duplicates are kept here; the CSR build collapses dups.    */
/* ------------------------------------------------------------------------ */
EXPORT int64_t rpqgen_er(int32_t nv, int64_t ne, int32_t nl, uint64_t seed,
                         int32_t* src, int32_t* dst, int32_t* lab) {
    if (nv <= 0 || ne < 0 || nl <= 0) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ne; ++i) {
        uint64_t r0 = draw(seed, 1, (uint64_t)i);
        uint64_t r1 = draw(seed, 2, (uint64_t)i);
        src[i] = (int32_t)bounded((uint32_t)(r0 >> 32), (uint32_t)nv);
        dst[i] = (int32_t)bounded((uint32_t)r0, (uint32_t)nv);
        lab[i] = (int32_t)bounded((uint32_t)(r1 >> 32), (uint32_t)nl);
    }
    return ne;
}

/* ------------------------------------------------------------------------ */
/* R-MAT (cfg2/3/5): m raw edges over 2^scale vertices with quadrant          */
/* probabilities (a, b, c, 1-a-b-c); no vertex permutation; self-loops are   */
/* dropped and (u, v) duplicates collapsed; each surviving pair gets ONE      */
/* Zipf(zipf_s) label over nl ranks drawn from hash(seed, u, v).              */
/* Output is sorted by (u, v).  Buffers must hold m entries.  Returns count.  */
/* ------------------------------------------------------------------------ */
EXPORT int64_t rpqgen_rmat(int32_t scale, int64_t m, double a, double b, double c,
                           int32_t nl, double zipf_s, uint64_t seed,
                           int32_t* src, int32_t* dst, int32_t* lab) {
    if (scale <= 0 || scale > 30 || m < 0 || nl <= 0) return -1;
    const uint64_t ta = (uint64_t)floor(a * 4294967296.0);
    const uint64_t tab = (uint64_t)floor((a + b) * 4294967296.0);
    const uint64_t tabc = (uint64_t)floor((a + b + c) * 4294967296.0);
    uint64_t* keys = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    uint64_t* tmp = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    if (!keys || !tmp) { free(keys); free(tmp); return -2; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        uint64_t u = 0, v = 0;
        for (int k = 0; k < scale; k += 2) {
            uint64_t r = draw(seed, 10, (uint64_t)i * 64 + (uint64_t)k);
            for (int h = 0; h < 2 && k + h < scale; ++h) {
                uint64_t r32 = h ? (r & 0xFFFFFFFFULL) : (r >> 32);
                uint64_t rowbit = r32 >= tab;
                uint64_t colbit = (r32 >= ta && r32 < tab) || r32 >= tabc;
                u = (u << 1) | rowbit;
                v = (v << 1) | colbit;
            }
        }
        keys[i] = (u == v) ? ~0ULL : ((u << 32) | v);
    }
    radix_sort_u64(keys, tmp, m, 64);
    free(tmp);
    /* unique + drop the self-loop sentinel (sorted to the end) */
    int64_t n = 0;
    for (int64_t i = 0; i < m; ++i) {
        if (keys[i] == ~0ULL) break;
        if (n == 0 || keys[n - 1] != keys[i]) keys[n++] = keys[i];
    }
    uint64_t* thr = (uint64_t*)malloc((size_t)nl * sizeof(uint64_t));
    rpqgen_zipf_thresholds(nl, zipf_s, thr);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)keys[i];
        src[i] = (int32_t)u;
        dst[i] = (int32_t)v;
        uint64_t r = draw(seed, 11, keys[i]);
        lab[i] = zipf_pick((uint32_t)(r >> 32), thr, nl);
    }
    free(thr);
    free(keys);
    return n;
}

/* ------------------------------------------------------------------------ */
/* Chung-Lu (cfg4): nv vertices, m raw edges, weights w_i = (i+1)^(-1/(g-1)). */
/* Sources drawn proportional to w, destinations proportional to w under an */
/* independent permutation (pi(i) = (i * P + off) mod nv, P odd, gcd=1).       */
/* Self-loops dropped, (u,v) dups collapsed, one Zipf label per pair.         */
/* ------------------------------------------------------------------------ */
static uint64_t gcd_u64(uint64_t x, uint64_t y) { while (y) { uint64_t t = x % y; x = y; y = t; } return x; }

EXPORT int64_t rpqgen_chunglu(int32_t nv, int64_t m, double gamma, int32_t nl, double zipf_s,
                              uint64_t seed, int32_t* src, int32_t* dst, int32_t* lab) {
    if (nv <= 1 || m < 0 || nl <= 0 || gamma <= 1.0) return -1;
    const double ex = -1.0 / (gamma - 1.0);
    /* cumulative weights, scaled to 2^62 integers for exact inverse-CDF sampling */
    double* cw = (double*)malloc((size_t)nv * sizeof(double));
    uint64_t* cdf = (uint64_t*)malloc((size_t)nv * sizeof(uint64_t));
    if (!cw || !cdf) { free(cw); free(cdf); return -2; }
    double tot = 0.0;
    for (int32_t i = 0; i < nv; ++i) { tot += pow((double)i + 1.0, ex); cw[i] = tot; }
    for (int32_t i = 0; i < nv; ++i) cdf[i] = (uint64_t)floor(cw[i] / tot * 4611686018427387904.0);
    cdf[nv - 1] = 4611686018427387904ULL;
    free(cw);
    uint64_t P = (draw(seed, 20, 0) | 1ULL) % (uint64_t)nv;
    while (P < 2 || gcd_u64(P, (uint64_t)nv) != 1) P = (P + 1) % (uint64_t)nv;
    uint64_t off = draw(seed, 20, 1) % (uint64_t)nv;
    uint64_t* keys = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    uint64_t* tmp = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    if (!keys || !tmp) { free(keys); free(tmp); free(cdf); return -2; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        uint64_t r0 = draw(seed, 21, (uint64_t)i) >> 2;
        uint64_t r1 = draw(seed, 22, (uint64_t)i) >> 2;
        int64_t lo = 0, hi = nv - 1;
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (r0 < cdf[mid]) hi = mid; else lo = mid + 1; }
        uint64_t u = (uint64_t)lo;
        lo = 0; hi = nv - 1;
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (r1 < cdf[mid]) hi = mid; else lo = mid + 1; }
        uint64_t v = ((uint64_t)lo * P + off) % (uint64_t)nv;
        keys[i] = (u == v) ? ~0ULL : ((u << 32) | v);
    }
    free(cdf);
    radix_sort_u64(keys, tmp, m, 64);
    free(tmp);
    int64_t n = 0;
    for (int64_t i = 0; i < m; ++i) {
        if (keys[i] == ~0ULL) break;
        if (n == 0 || keys[n - 1] != keys[i]) keys[n++] = keys[i];
    }
    uint64_t* thr = (uint64_t*)malloc((size_t)nl * sizeof(uint64_t));
    rpqgen_zipf_thresholds(nl, zipf_s, thr);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        src[i] = (int32_t)(keys[i] >> 32);
        dst[i] = (int32_t)(uint32_t)keys[i];
        uint64_t r = draw(seed, 23, keys[i]);
        lab[i] = zipf_pick((uint32_t)(r >> 32), thr, nl);
    }
    free(thr);
    free(keys);
    return n;
}

/* ------------------------------------------------------------------------ */
/* Per-label canonical CSR (the LabeledGraph layout).                         */
/* rpqgen_label_count: edges carrying `label` (before dedup).                 */
/* rpqgen_label_csr: rows = src (or dst when transpose), sorted unique cols.  */
/*   indptr: nv+1 int64; indices: capacity >= rpqgen_label_count; returns nnz.*/
/* ------------------------------------------------------------------------ */
EXPORT int64_t rpqgen_label_count(int64_t ne, const int32_t* lab, int32_t label) {
    int64_t cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(static)
    for (int64_t i = 0; i < ne; ++i) cnt += (lab[i] == label);
    return cnt;
}

static int cmp_i64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}

EXPORT int64_t rpqgen_label_csr(int32_t nv, int64_t ne, const int32_t* src, const int32_t* dst,
                                const int32_t* lab, int32_t label, int32_t transpose,
                                int64_t* indptr, int64_t* indices) {
    const int32_t* rows = transpose ? dst : src;
    const int32_t* cols = transpose ? src : dst;
    int64_t* cnt = (int64_t*)calloc((size_t)nv + 1, sizeof(int64_t));
    if (!cnt) return -2;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ne; ++i)
        if (lab[i] == label) __atomic_fetch_add(&cnt[rows[i] + 1], 1, __ATOMIC_RELAXED);
    indptr[0] = 0;
    for (int32_t r = 0; r < nv; ++r) indptr[r + 1] = indptr[r] + cnt[r + 1];
    for (int32_t r = 0; r <= nv; ++r) cnt[r] = indptr[r];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ne; ++i)
        if (lab[i] == label) {
            int64_t pos = __atomic_fetch_add(&cnt[rows[i]], 1, __ATOMIC_RELAXED);
            indices[pos] = cols[i];
        }
    /* sort + unique each row; record new lengths in cnt */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int32_t r = 0; r < nv; ++r) {
        int64_t lo = indptr[r], hi = indptr[r + 1];
        int64_t len = hi - lo;
        if (len > 1) {
            int64_t* p = indices + lo;
            if (len < 24) {
                for (int64_t i = 1; i < len; ++i) {
                    int64_t x = p[i], j = i - 1;
                    while (j >= 0 && p[j] > x) { p[j + 1] = p[j]; --j; }
                    p[j + 1] = x;
                }
            } else {
                qsort(p, (size_t)len, sizeof(int64_t), cmp_i64);
            }
            int64_t k = 1;
            for (int64_t i = 1; i < len; ++i) if (p[i] != p[k - 1]) p[k++] = p[i];
            len = k;
        }
        cnt[r] = len;
    }
    /* compact */
    int64_t out = 0;
    for (int32_t r = 0; r < nv; ++r) {
        int64_t lo = indptr[r], len = cnt[r];
        if (out != lo) memmove(indices + out, indices + lo, (size_t)len * sizeof(int64_t));
        indptr[r] = out;
        out += len;
    }
    indptr[nv] = out;
    free(cnt);
    return out;
}

/* total out-degree over all labels of each vertex (int64 out[nv]) */
EXPORT void rpqgen_out_degree(int32_t nv, int64_t ne, const int32_t* src, int64_t* out) {
    memset(out, 0, (size_t)nv * sizeof(int64_t));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ne; ++i) __atomic_fetch_add(&out[src[i]], 1, __ATOMIC_RELAXED);
}
