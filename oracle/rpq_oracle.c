/*
 * rpq_oracle.c -- CPU restatement of the reference's single-source 2-RPQ path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2412_10287_b200/)
 * links, imports or calls this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, as the checker and as
 * the timed CPU baseline ("kind": "port").
 *
 * Parity pin: tests/test_oracle_golden.py checks both entry points below against
 * golden vectors produced by running the reference package itself
 * (/root/reference/pkg/src/rpq, via tests/golden/make_golden.py).
 *
 * Two independent restatements:
 *
 *  oracle_bfs   -- rpq/oracle.py:21-59 (oracle_ssr): breadth-first search over
 *                  (state, vertex) pairs with a visited set, made
 *                  level-synchronous so that it also yields the masked loop's
 *                  iteration count (rpq/engine.py:146-171: one iteration per
 *                  frontier expansion, including the final empty one) and the
 *                  product-edge count TE of SURVEY.md §8(d).
 *
 *  oracle_port  -- rpq/engine.py:146-232 (eval_ssr_masked / _no_mask / _hybrid)
 *                  on the reference's own data representation: position sets as
 *                  sorted, de-duplicated flat keys row*ncols+col
 *                  (rpq/sparse_bool.py:104-110), bool_matmul as a row gather
 *                  followed by sort+unique (sparse_bool.py:231-251), or_sum as a
 *                  sorted union (:198-206), mask_complement as a sorted
 *                  difference (:218-228).  This is the "reference CPU
 *                  implementation" that bench.py times.
 *
 * Semantics shared by both:
 *  - P is seeded with {(q_s, source)} for every start state (engine.py:106-109,
 *    :154-155), so the source is an answer iff a start state is final.
 *  - transitions whose label index >= num_labels are skipped (engine.py:100-101,
 *    oracle.py:27-28).
 *  - (label, inverted) traverses backward[label] = transpose(forward[label])
 *    (graph_store.py:52, :87-91).
 *  - the answer is {v : exists q in finals, (q, v) in P} (engine.py:112-114).
 */
#define _POSIX_C_SOURCE 200809L
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* graph: COO kept by reference (caller owns), per-(label, dir) CSR on demand */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t* indptr; /* nv + 1 */
    int32_t* indices;
    int64_t nnz;
} ocsr;

typedef struct {
    int32_t nv, nl;
    int64_t ne;
    const int32_t* src;
    const int32_t* dst;
    const int32_t* lab;
    ocsr* slots; /* 2 * nl, lazily filled */
    pthread_mutex_t mu;
} ograph;

EXPORT void* oracle_graph_create(int32_t nv, int32_t nl, int64_t ne, const int32_t* src,
                                 const int32_t* dst, const int32_t* lab) {
    ograph* g = (ograph*)calloc(1, sizeof(ograph));
    g->nv = nv; g->nl = nl; g->ne = ne; g->src = src; g->dst = dst; g->lab = lab;
    g->slots = (ocsr*)calloc((size_t)(2 * (nl > 0 ? nl : 1)), sizeof(ocsr));
    pthread_mutex_init(&g->mu, NULL);
    return g;
}

EXPORT void oracle_graph_destroy(void* gp) {
    ograph* g = (ograph*)gp;
    if (!g) return;
    for (int32_t i = 0; i < 2 * g->nl; ++i) { free(g->slots[i].indptr); free(g->slots[i].indices); }
    free(g->slots);
    pthread_mutex_destroy(&g->mu);
    free(g);
}

static int cmp_i32(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

/* canonical CSR of label `l` (transposed when inv): rows sorted, dups collapsed */
static ocsr* slot_csr(ograph* g, int32_t l, int32_t inv) {
    ocsr* s = &g->slots[2 * l + (inv ? 1 : 0)];
    pthread_mutex_lock(&g->mu);
    if (!s->indptr) {
        const int32_t* rows = inv ? g->dst : g->src;
        const int32_t* cols = inv ? g->src : g->dst;
        int64_t* ptr = (int64_t*)calloc((size_t)g->nv + 1, sizeof(int64_t));
        for (int64_t i = 0; i < g->ne; ++i) if (g->lab[i] == l) ptr[rows[i] + 1]++;
        for (int32_t r = 0; r < g->nv; ++r) ptr[r + 1] += ptr[r];
        int64_t n = ptr[g->nv];
        int32_t* idx = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
        int64_t* fill = (int64_t*)malloc((size_t)g->nv * sizeof(int64_t));
        memcpy(fill, ptr, (size_t)g->nv * sizeof(int64_t));
        for (int64_t i = 0; i < g->ne; ++i) if (g->lab[i] == l) idx[fill[rows[i]]++] = cols[i];
        free(fill);
        int64_t out = 0;
        for (int32_t r = 0; r < g->nv; ++r) {
            int64_t lo = ptr[r], hi = ptr[r + 1];
            if (hi - lo > 1) qsort(idx + lo, (size_t)(hi - lo), sizeof(int32_t), cmp_i32);
            int64_t start = out;
            for (int64_t i = lo; i < hi; ++i)
                if (out == start || idx[out - 1] != idx[i]) idx[out++] = idx[i];
            ptr[r] = start;
        }
        ptr[g->nv] = out;
        s->indices = idx;
        s->nnz = out;
        __atomic_store_n(&s->indptr, ptr, __ATOMIC_RELEASE);
    }
    pthread_mutex_unlock(&g->mu);
    return s;
}

EXPORT int64_t oracle_graph_prepare(void* gp, int32_t label, int32_t inv) {
    ograph* g = (ograph*)gp;
    if (label < 0 || label >= g->nl) return -1;
    return slot_csr(g, label, inv)->nnz;
}

/* copy out one slot's CSR (for fixture cross-checks): indptr nv+1, indices nnz */
EXPORT int64_t oracle_graph_slot(void* gp, int32_t label, int32_t inv, int64_t* indptr,
                                 int32_t* indices) {
    ograph* g = (ograph*)gp;
    if (label < 0 || label >= g->nl) return -1;
    ocsr* s = slot_csr(g, label, inv);
    if (indptr) memcpy(indptr, s->indptr, ((size_t)g->nv + 1) * sizeof(int64_t));
    if (indices) memcpy(indices, s->indices, (size_t)s->nnz * sizeof(int32_t));
    return s->nnz;
}

/* ------------------------------------------------------------------------ */
/* stats shared by both entry points                                          */
/* ------------------------------------------------------------------------ */
#define ORACLE_MAX_LEVELS 4096
typedef struct {
    int32_t iterations;  /* masked-loop iterations (engine.py:157-160) */
    int32_t levels;      /* number of non-empty frontiers after the seed */
    int64_t te;          /* product edges traversed */
    int64_t x;           /* (pair, transition) row-pointer lookups */
    int64_t pairs;       /* |P| */
    int64_t reach;       /* |answer| */
    double seconds;      /* wall time of the evaluation proper */
    int64_t level_new[ORACLE_MAX_LEVELS];
} ostats;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* oracle_bfs: level-synchronous product BFS (oracle.py:21-59)                */
/* ------------------------------------------------------------------------ */
EXPORT int oracle_bfs(void* gp, int32_t nstates, int32_t ntrans, const int32_t* t_src,
                      const int32_t* t_label, const int32_t* t_inv, const int32_t* t_dst,
                      int32_t nstarts, const int32_t* starts, int32_t nfinals,
                      const int32_t* finals, int32_t source, uint8_t* reach, ostats* st) {
    ograph* g = (ograph*)gp;
    const int64_t nv = g->nv;
    if (source < 0 || source >= nv) return 2;
    if (nstates <= 0) return 1;
    double t0 = now_s();
    /* per-state transition lists (usable labels only) */
    int32_t* tcount = (int32_t*)calloc((size_t)nstates + 1, sizeof(int32_t));
    int32_t* torder = (int32_t*)malloc((size_t)(ntrans > 0 ? ntrans : 1) * sizeof(int32_t));
    ocsr** tslot = (ocsr**)malloc((size_t)(ntrans > 0 ? ntrans : 1) * sizeof(ocsr*));
    for (int32_t t = 0; t < ntrans; ++t) {
        tslot[t] = NULL;
        if (t_label[t] < 0 || t_label[t] >= g->nl) continue; /* engine.py:100-101 */
        if (t_src[t] < 0 || t_src[t] >= nstates || t_dst[t] < 0 || t_dst[t] >= nstates) continue;
        tslot[t] = slot_csr(g, t_label[t], t_inv[t]);
        tcount[t_src[t] + 1]++;
    }
    for (int32_t q = 0; q < nstates; ++q) tcount[q + 1] += tcount[q];
    {
        int32_t* fill = (int32_t*)malloc((size_t)nstates * sizeof(int32_t));
        memcpy(fill, tcount, (size_t)nstates * sizeof(int32_t));
        for (int32_t t = 0; t < ntrans; ++t) if (tslot[t]) torder[fill[t_src[t]]++] = t;
        free(fill);
    }
    const int64_t words = (nv + 63) / 64;
    uint64_t* vis = (uint64_t*)calloc((size_t)(words * nstates), sizeof(uint64_t));
    int64_t cap = 1024;
    int64_t* cur = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
    int64_t* nxt = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
    int64_t ncur = 0, nnxt = 0;
    memset(st, 0, sizeof(*st));
    for (int32_t i = 0; i < nstarts; ++i) {
        int32_t q = starts[i];
        if (q < 0 || q >= nstates) continue;
        uint64_t* w = &vis[q * words + (source >> 6)];
        if (*w & (1ULL << (source & 63))) continue;
        *w |= 1ULL << (source & 63);
        cur[ncur++] = (int64_t)q * nv + source;
    }
    st->pairs = ncur;
    int32_t iterations = 0;
    while (ncur) {
        nnxt = 0;
        for (int64_t i = 0; i < ncur; ++i) {
            int32_t q = (int32_t)(cur[i] / nv);
            int64_t v = cur[i] % nv;
            for (int32_t k = tcount[q]; k < tcount[q + 1]; ++k) {
                int32_t t = torder[k];
                const ocsr* s = tslot[t];
                int32_t q2 = t_dst[t];
                int64_t lo = s->indptr[v], hi = s->indptr[v + 1];
                st->x++;
                st->te += hi - lo;
                uint64_t* row = vis + (int64_t)q2 * words;
                for (int64_t e = lo; e < hi; ++e) {
                    int32_t w = s->indices[e];
                    uint64_t bit = 1ULL << (w & 63);
                    if (row[w >> 6] & bit) continue;
                    row[w >> 6] |= bit;
                    if (nnxt == cap) {
                        cap *= 2;
                        cur = (int64_t*)realloc(cur, (size_t)cap * sizeof(int64_t));
                        nxt = (int64_t*)realloc(nxt, (size_t)cap * sizeof(int64_t));
                    }
                    nxt[nnxt++] = (int64_t)q2 * nv + w;
                }
            }
        }
        iterations++;
        if (nnxt && st->levels < ORACLE_MAX_LEVELS) st->level_new[st->levels] = nnxt;
        if (nnxt) st->levels++;
        st->pairs += nnxt;
        int64_t* sw = cur; cur = nxt; nxt = sw;
        ncur = nnxt;
    }
    st->iterations = iterations;
    memset(reach, 0, (size_t)nv);
    for (int32_t i = 0; i < nfinals; ++i) {
        int32_t q = finals[i];
        if (q < 0 || q >= nstates) continue;
        const uint64_t* row = vis + (int64_t)q * words;
        for (int64_t v = 0; v < nv; ++v) if (row[v >> 6] >> (v & 63) & 1) reach[v] = 1;
    }
    for (int64_t v = 0; v < nv; ++v) st->reach += reach[v];
    st->seconds = now_s() - t0;
    free(vis); free(cur); free(nxt); free(tcount); free(torder); free(tslot);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* oracle_port: engine.py's masked / no_mask / hybrid loops on sorted keys    */
/* ------------------------------------------------------------------------ */
typedef struct { uint64_t* k; int64_t n; } keyset;

static void ks_free(keyset* s) { free(s->k); s->k = NULL; s->n = 0; }

/* LSD radix sort + unique, single-threaded (the reference's kernels are
 * sequential: sparse_bool.py:18-24) -- np.unique in sparse_bool.py:250 */
static void sort_unique(uint64_t* a, int64_t n, int bits, int64_t* nout) {
    if (n <= 1) { *nout = n; return; }
    if (n < 64) {
        for (int64_t i = 1; i < n; ++i) {
            uint64_t x = a[i]; int64_t j = i - 1;
            while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
            a[j + 1] = x;
        }
    } else {
        uint64_t* tmp = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
        uint64_t* s = a; uint64_t* d = tmp;
        int64_t cnt[2049];
        for (int shift = 0; shift < bits; shift += 11) {
            memset(cnt, 0, sizeof(cnt));
            for (int64_t i = 0; i < n; ++i) cnt[((s[i] >> shift) & 2047) + 1]++;
            for (int b = 0; b < 2048; ++b) cnt[b + 1] += cnt[b];
            for (int64_t i = 0; i < n; ++i) d[cnt[(s[i] >> shift) & 2047]++] = s[i];
            uint64_t* t = s; s = d; d = t;
        }
        if (s != a) memcpy(a, s, (size_t)n * sizeof(uint64_t));
        free(tmp);
    }
    int64_t k = 1;
    for (int64_t i = 1; i < n; ++i) if (a[i] != a[k - 1]) a[k++] = a[i];
    *nout = k;
}

/* or_sum (sparse_bool.py:198-206): sorted union */
static keyset ks_union(const keyset* a, const keyset* b) {
    keyset r;
    r.k = (uint64_t*)malloc((size_t)(a->n + b->n + 1) * sizeof(uint64_t));
    int64_t i = 0, j = 0, n = 0;
    while (i < a->n && j < b->n) {
        if (a->k[i] < b->k[j]) r.k[n++] = a->k[i++];
        else if (a->k[i] > b->k[j]) r.k[n++] = b->k[j++];
        else { r.k[n++] = a->k[i++]; j++; }
    }
    while (i < a->n) r.k[n++] = a->k[i++];
    while (j < b->n) r.k[n++] = b->k[j++];
    r.n = n;
    return r;
}

/* mask_complement (sparse_bool.py:218-228): sorted difference a \ m */
static keyset ks_diff(const keyset* a, const keyset* m) {
    keyset r;
    r.k = (uint64_t*)malloc((size_t)(a->n + 1) * sizeof(uint64_t));
    int64_t i = 0, j = 0, n = 0;
    while (i < a->n) {
        while (j < m->n && m->k[j] < a->k[i]) j++;
        if (j < m->n && m->k[j] == a->k[i]) { i++; continue; }
        r.k[n++] = a->k[i++];
    }
    r.n = n;
    return r;
}

static keyset ks_copy(const keyset* a) {
    keyset r;
    r.k = (uint64_t*)malloc((size_t)(a->n + 1) * sizeof(uint64_t));
    memcpy(r.k, a->k, (size_t)a->n * sizeof(uint64_t));
    r.n = a->n;
    return r;
}

typedef struct {
    int32_t npairs;         /* (N^T, G) per usable symbol, sorted (engine.py:92-103) */
    int32_t* nt_off;        /* npairs + 1 offsets into nt_rows/nt_cols */
    int32_t* nt_rows;       /* N^T entries (q', q), row-major sorted */
    int32_t* nt_cols;
    const ocsr** gslot;     /* adjacency per pair */
} symtab;

static int cmp_trans(const void* x, const void* y) {
    const int32_t* a = (const int32_t*)x; const int32_t* b = (const int32_t*)y;
    for (int i = 0; i < 4; ++i) if (a[i] != b[i]) return (a[i] > b[i]) - (a[i] < b[i]);
    return 0;
}

/* bool_matmul(bool_matmul(N^T, M), G) for one symbol (engine.py:120-121) */
static keyset symbol_product(const symtab* T, int32_t p, const keyset* m, int64_t nv, int bits) {
    /* t1 = N^T x M : rows q', cols v.  Gather rows q of M for each (q', q). */
    int64_t total = 0;
    /* M's row ranges via binary search on keys */
    for (int32_t e = T->nt_off[p]; e < T->nt_off[p + 1]; ++e) {
        uint64_t lo_key = (uint64_t)T->nt_cols[e] * (uint64_t)nv, hi_key = lo_key + (uint64_t)nv;
        int64_t lo = 0, hi = m->n;
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (m->k[mid] < lo_key) lo = mid + 1; else hi = mid; }
        int64_t a = lo; hi = m->n;
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (m->k[mid] < hi_key) lo = mid + 1; else hi = mid; }
        total += lo - a;
    }
    keyset t1;
    t1.k = (uint64_t*)malloc((size_t)(total + 1) * sizeof(uint64_t));
    t1.n = 0;
    for (int32_t e = T->nt_off[p]; e < T->nt_off[p + 1]; ++e) {
        uint64_t q = (uint64_t)T->nt_cols[e], q2 = (uint64_t)T->nt_rows[e];
        uint64_t lo_key = q * (uint64_t)nv, hi_key = lo_key + (uint64_t)nv;
        int64_t lo = 0, hi = m->n;
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (m->k[mid] < lo_key) lo = mid + 1; else hi = mid; }
        for (int64_t i = lo; i < m->n && m->k[i] < hi_key; ++i)
            t1.k[t1.n++] = q2 * (uint64_t)nv + (m->k[i] - lo_key);
    }
    sort_unique(t1.k, t1.n, bits, &t1.n);
    /* t2 = t1 x G */
    const ocsr* g = T->gslot[p];
    total = 0;
    for (int64_t i = 0; i < t1.n; ++i) {
        int64_t v = (int64_t)(t1.k[i] % (uint64_t)nv);
        total += g->indptr[v + 1] - g->indptr[v];
    }
    keyset t2;
    t2.k = (uint64_t*)malloc((size_t)(total + 1) * sizeof(uint64_t));
    t2.n = 0;
    for (int64_t i = 0; i < t1.n; ++i) {
        uint64_t row = t1.k[i] / (uint64_t)nv;
        int64_t v = (int64_t)(t1.k[i] % (uint64_t)nv);
        for (int64_t e = g->indptr[v]; e < g->indptr[v + 1]; ++e)
            t2.k[t2.n++] = row * (uint64_t)nv + (uint64_t)g->indices[e];
    }
    ks_free(&t1);
    sort_unique(t2.k, t2.n, bits, &t2.n);
    return t2;
}

/* _step_sum (engine.py:117-124) */
static keyset step_sum(const symtab* T, const keyset* m, int64_t nv, int bits) {
    keyset acc = {NULL, 0};
    acc.k = (uint64_t*)malloc(sizeof(uint64_t));
    for (int32_t p = 0; p < T->npairs; ++p) {
        keyset part = symbol_product(T, p, m, nv, bits);
        keyset u = ks_union(&acc, &part);
        ks_free(&acc); ks_free(&part);
        acc = u;
    }
    return acc;
}

/* algorithm: 0 masked, 1 no_mask, 2 hybrid.  threshold: hybrid switch_threshold
 * (engine.py:57).  timeout_s < 0: none.  Returns 0, 1 invalid, 2 bad vertex,
 * 3 timeout (iterations reported). */
EXPORT int oracle_port(void* gp, int32_t nstates, int32_t ntrans, const int32_t* t_src,
                       const int32_t* t_label, const int32_t* t_inv, const int32_t* t_dst,
                       int32_t nstarts, const int32_t* starts, int32_t nfinals,
                       const int32_t* finals, int32_t source, int32_t algorithm,
                       double threshold, double timeout_s, uint8_t* reach, ostats* st) {
    ograph* g = (ograph*)gp;
    const int64_t nv = g->nv;
    if (algorithm < 0 || algorithm > 2 || nstates <= 0) return 1;
    if (source < 0 || source >= nv) return 2; /* engine.py:141-143 */
    double t0 = now_s();
    memset(st, 0, sizeof(*st));
    int bits = 1;
    while (bits < 64 && ((uint64_t)1 << bits) < (uint64_t)nstates * (uint64_t)nv) bits++;

    /* symbol table: sorted (label, inv) with label < nl; N^T entries sorted */
    int32_t* rec = (int32_t*)malloc((size_t)(ntrans > 0 ? ntrans : 1) * 4 * sizeof(int32_t));
    int32_t nrec = 0;
    for (int32_t t = 0; t < ntrans; ++t) {
        if (t_label[t] < 0 || t_label[t] >= g->nl) continue;
        rec[4 * nrec + 0] = t_label[t];
        rec[4 * nrec + 1] = t_inv[t] ? 1 : 0;
        rec[4 * nrec + 2] = t_dst[t]; /* N^T row */
        rec[4 * nrec + 3] = t_src[t]; /* N^T col */
        nrec++;
    }
    qsort(rec, (size_t)nrec, 4 * sizeof(int32_t), cmp_trans);
    symtab T;
    T.npairs = 0;
    T.nt_off = (int32_t*)malloc((size_t)(nrec + 1) * sizeof(int32_t));
    T.nt_rows = (int32_t*)malloc((size_t)(nrec + 1) * sizeof(int32_t));
    T.nt_cols = (int32_t*)malloc((size_t)(nrec + 1) * sizeof(int32_t));
    T.gslot = (const ocsr**)malloc((size_t)(nrec + 1) * sizeof(ocsr*));
    int32_t ne = 0;
    for (int32_t i = 0; i < nrec; ++i) {
        if (i > 0 && rec[4 * i + 2] == rec[4 * (i - 1) + 2] && rec[4 * i + 3] == rec[4 * (i - 1) + 3] &&
            rec[4 * i] == rec[4 * (i - 1)] && rec[4 * i + 1] == rec[4 * (i - 1) + 1])
            continue; /* duplicate transition */
        if (i == 0 || rec[4 * i] != rec[4 * (i - 1)] || rec[4 * i + 1] != rec[4 * (i - 1) + 1]) {
            T.nt_off[T.npairs] = ne;
            T.gslot[T.npairs] = slot_csr(g, rec[4 * i], rec[4 * i + 1]);
            T.npairs++;
        }
        T.nt_rows[ne] = rec[4 * i + 2];
        T.nt_cols[ne] = rec[4 * i + 3];
        ne++;
    }
    T.nt_off[T.npairs] = ne;
    free(rec);

    /* _seed (engine.py:106-109) */
    keyset p;
    p.k = (uint64_t*)malloc((size_t)(nstarts + 1) * sizeof(uint64_t));
    p.n = 0;
    for (int32_t i = 0; i < nstarts; ++i)
        if (starts[i] >= 0 && starts[i] < nstates) p.k[p.n++] = (uint64_t)starts[i] * (uint64_t)nv + (uint64_t)source;
    sort_unique(p.k, p.n, bits, &p.n);

    int status = 0;
    int32_t iterations = 0;
    const double deadline = timeout_s < 0 ? 1e300 : t0 + timeout_s;
    if (algorithm == 0) {
        /* eval_ssr_masked (engine.py:146-171) */
        keyset m = ks_copy(&p);
        while (m.n) {
            if (now_s() > deadline) { status = 3; break; }
            keyset s = step_sum(&T, &m, nv, bits);
            keyset nm = ks_diff(&s, &p);
            ks_free(&s); ks_free(&m);
            m = nm;
            iterations++;
            if (m.n && st->levels < ORACLE_MAX_LEVELS) st->level_new[st->levels] = m.n;
            if (m.n) st->levels++;
            keyset np = ks_union(&p, &m);
            ks_free(&p);
            p = np;
        }
        ks_free(&m);
    } else {
        /* eval_ssr_no_mask (engine.py:174-194) and eval_ssr_hybrid (:197-232) */
        keyset prev = {(uint64_t*)malloc(sizeof(uint64_t)), 0};
        keyset m = {NULL, 0};
        int switched = 0;
        for (;;) {
            if (now_s() > deadline) { status = 3; break; }
            if (algorithm == 2 && !switched && (double)p.n > threshold) {
                m = ks_diff(&p, &prev);
                switched = 1;
            }
            if (!switched) {
                keyset s = step_sum(&T, &p, nv, bits);
                keyset nw = ks_union(&p, &s);
                ks_free(&s);
                iterations++;
                if (nw.n == p.n) { ks_free(&nw); break; }
                if (st->levels < ORACLE_MAX_LEVELS) st->level_new[st->levels] = nw.n - p.n;
                st->levels++;
                ks_free(&prev);
                prev = p;
                p = nw;
            } else {
                keyset s = step_sum(&T, &m, nv, bits);
                keyset nm = ks_diff(&s, &p);
                ks_free(&s); ks_free(&m);
                m = nm;
                iterations++;
                if (m.n == 0) break;
                if (st->levels < ORACLE_MAX_LEVELS) st->level_new[st->levels] = m.n;
                st->levels++;
                keyset np = ks_union(&p, &m);
                ks_free(&p);
                p = np;
            }
        }
        ks_free(&prev);
        ks_free(&m);
    }
    st->iterations = iterations;
    st->pairs = p.n;
    /* _project_finals (engine.py:112-114) */
    memset(reach, 0, (size_t)nv);
    uint8_t* isfinal = (uint8_t*)calloc((size_t)nstates, 1);
    for (int32_t i = 0; i < nfinals; ++i) if (finals[i] >= 0 && finals[i] < nstates) isfinal[finals[i]] = 1;
    for (int64_t i = 0; i < p.n; ++i) {
        uint64_t q = p.k[i] / (uint64_t)nv;
        if (isfinal[q]) reach[p.k[i] % (uint64_t)nv] = 1;
    }
    for (int64_t v = 0; v < nv; ++v) st->reach += reach[v];
    free(isfinal);
    ks_free(&p);
    free(T.nt_off); free(T.nt_rows); free(T.nt_cols); free(T.gslot);
    st->seconds = now_s() - t0;
    return status;
}
