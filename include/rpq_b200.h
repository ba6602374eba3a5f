/*
 * rpq_b200.h -- C ABI of the B200-native single-source 2-RPQ engine.
 *
 * Drop-in boundary for the reference package's query entry point
 *   rpq.engine.eval_ssr(g: LabeledGraph, n: TwoNfa, source, opts) -> EvalResult
 *   (/root/reference/pkg/src/rpq/engine.py:242-251)
 * and its single-destination caller eval_sdr (engine.py:254-266).  The reference
 * has no native code and no FFI; its "plugin interface" for this path is that
 * Python function, so the Python package paper_2412_10287_b200 mirrors it
 * (same names, argument meaning, errors) and binds THIS header through ctypes
 * (see INTEGRATION.md).  No torch types cross this boundary: plain pointers,
 * sizes and an opaque cudaStream_t passed as void*.
 *
 * Entry points and the reference interface each one replaces:
 *   rpq_graph_create / rpq_graph_set_label
 *       LabeledGraph.__init__ keeping forward[l] and backward[l] = transpose
 *       (graph_store.py:35-52); the arrays are the reference's own int64 CSR
 *       indptr/indices (sparse_bool.py:51-59), narrowed to 32 bits on device.
 *   rpq_query_create
 *       _label_pairs (engine.py:92-103): the automaton's usable symbols
 *       (label index < num_labels) and their transition matrices, given as
 *       (src state, label, inverted, dst state) triples, plus start_set /
 *       final_set (query_compiler.py:241-247).
 *   rpq_query_run / rpq_query_wait
 *       the evaluator loop (engine.py:146-232): seed (:106-109), frontier step
 *       _step_sum + mask_complement + or_sum (:117-124, :159-165) until the
 *       frontier is empty, the per-iteration deadline check (_Clock.check,
 *       :87-89), and _project_finals (:112-114).
 *   rpq_ssr
 *       one-shot eval_ssr: create query, run, wait, copy the answer, destroy.
 *
 * Status codes (Python mapping, engine.py error behaviour):
 *   RPQ_OK 0, RPQ_EINVAL 1 -> ValueError, RPQ_ERANGE 2 -> IndexError
 *   (engine.py:141-143), RPQ_ETIMEOUT 3 -> QueryTimeout(elapsed, iterations)
 *   (engine.py:45-51), RPQ_ECUDA 4 -> RuntimeError, RPQ_ENOMEM 5 -> MemoryError,
 *   RPQ_ENOLABEL 6 -> a label the automaton uses is not resident on the device.
 * rpq_last_error() returns a thread-local message for the last failure.
 */
#ifndef RPQ_B200_H
#define RPQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RPQ_ABI_VERSION 3

#if defined(__GNUC__)
#define RPQ_API __attribute__((visibility("default")))
#else
#define RPQ_API
#endif

#define RPQ_OK 0
#define RPQ_EINVAL 1
#define RPQ_ERANGE 2
#define RPQ_ETIMEOUT 3
#define RPQ_ECUDA 4
#define RPQ_ENOMEM 5
#define RPQ_ENOLABEL 6

#define RPQ_STATS_LEVELS 64

typedef struct rpq_graph rpq_graph;
typedef struct rpq_query rpq_query;

typedef struct rpq_stats {
    int32_t status;          /* RPQ_* of the run */
    int32_t iterations;      /* masked-loop iterations (engine.py:157-160), incl. the final empty step */
    int32_t levels;          /* non-empty frontiers produced after the seed */
    int32_t grid;            /* CTAs of the persistent step kernel */
    int64_t te;              /* product edges traversed, SURVEY.md §8(d) TE: exact when
                                count_te is set, else the edges push levels expanded */
    int64_t segments;        /* (pair, transition group) row lookups with degree > 0 */
    int64_t visited_pairs;   /* |P| at exit */
    int64_t reach_count;     /* |answer| */
    float device_ms;         /* CUDA-event time, first kernel to answer ready */
    int32_t pull_levels;     /* levels run in the pull direction */
    int64_t level_new[RPQ_STATS_LEVELS];    /* |F_L|: new (state, vertex) pairs per level */
    int64_t level_edges[RPQ_STATS_LEVELS];  /* push-model edges expanded from F_L (-1: pulled) */
    int64_t level_ns[RPQ_STATS_LEVELS];     /* kernel start -> level L's decision taken (CTA 0) */
    int64_t work_ns[RPQ_STATS_LEVELS];      /* kernel start -> last CTA done with level L's work */
    int64_t bar_ns[RPQ_STATS_LEVELS];       /* kernel start -> CTA 0 past the barrier after level L */
    int8_t level_dir[RPQ_STATS_LEVELS];     /* 0 push, 1 pull */
    int32_t answer_list;     /* rpq_query_eval_list only: 1 = the answer buffer holds answer_words
                                (word index, word) uint32 pairs instead of the bitmap */
    int64_t answer_words;    /* nonzero words of the answer bitmap (list runs) */
} rpq_stats;

/* Multi-source batches: up to RPQ_BATCH sources per run (one bit each). */
#define RPQ_BATCH 64

typedef struct rpq_batch_stats {
    int32_t status;          /* RPQ_* of the run */
    int32_t nsrc;            /* sources in the run */
    int32_t levels;          /* levels expanded (max over the batch) */
    int32_t grid;            /* CTAs of the persistent kernel */
    int64_t te;              /* sum over sources of product edges traversed (exact) */
    int64_t rows;            /* edges read: each frontier row once for all sources holding it */
    int64_t visited_pairs;   /* sum over sources of |P_s| */
    float device_ms;         /* CUDA-event time of the run */
    int32_t iterations[RPQ_BATCH];   /* per source: masked-loop iterations (engine.py:157-160),
                                        i.e. non-empty frontiers incl. the seed */
    int64_t reach_count[RPQ_BATCH];  /* per source: |answer_s| */
    int64_t level_items[RPQ_STATS_LEVELS];  /* (state, vertex) items with a non-empty source word */
    int64_t level_new[RPQ_STATS_LEVELS];    /* (pair, source) discoveries forming level L */
    int64_t level_ns[RPQ_STATS_LEVELS];     /* kernel start -> level L starts (CTA 0) */
    int64_t level_rows[RPQ_STATS_LEVELS];   /* edges read before level L starts */
} rpq_batch_stats;

/* level direction policy (rpq_query_set_options) */
#define RPQ_DIR_AUTO 0   /* per level: pull when m_f * alpha > m_u (Beamer) */
#define RPQ_DIR_PUSH 1   /* always expand the frontier's rows (SpMSpV over CSR) */
#define RPQ_DIR_PULL 2   /* always scan unvisited rows of the transpose (CSC) */

RPQ_API int rpq_abi_version(void);
/* 1 in the checked build (librpq_b200_checked.so, -DRPQ_CHECKED: device-side
 * bounds checks on every data-dependent index; a failed check fails the run
 * with RPQ_ECUDA "bounds check failed at file:line"), 0 otherwise. */
RPQ_API int rpq_checked_build(void);
RPQ_API const char* rpq_last_error(void);
/* SM count, L2 bytes and HBM bytes of a device (for launch sizing / reports) */
RPQ_API int rpq_device_info(int32_t device, int32_t* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes);

/* ---- graph residency ---------------------------------------------------- */
RPQ_API int rpq_graph_create(int32_t num_vertices, int32_t num_labels, int32_t device, rpq_graph** out);
/* Upload label `label`: forward CSR (rows = sources) and backward CSR
 * (= transpose, rows = destinations), each with num_vertices+1 int64 row
 * pointers and int64 column indices, as held by LabeledGraph.forward/backward.
 * Narrowed on device to uint32 row pointers / int32 columns.  Idempotent. */
RPQ_API int rpq_graph_set_label(rpq_graph* g, int32_t label,
                        int64_t fwd_nnz, const int64_t* fwd_indptr, const int64_t* fwd_indices,
                        int64_t bwd_nnz, const int64_t* bwd_indptr, const int64_t* bwd_indices);
/* Same from int32 arrays (the generator's native layout). */
RPQ_API int rpq_graph_set_label_i32(rpq_graph* g, int32_t label,
                            int64_t fwd_nnz, const int32_t* fwd_indptr, const int32_t* fwd_indices,
                            int64_t bwd_nnz, const int32_t* bwd_indptr, const int32_t* bwd_indices);
/* Graph from an edge list (src[i] --label[i]--> dst[i], int32 vertex and
 * label indices), ingested on the device: duplicates (src, label, dst)
 * collapse, self-loops stay (graph_store.py:161-176).  A label's forward and
 * backward CSR are built on the device the first time a query uses it (or by
 * rpq_graph_materialize_label), so graphs with thousands of labels only pay
 * for the labels queried. */
RPQ_API int rpq_graph_create_coo(int32_t num_vertices, int32_t num_labels, int64_t nnz, const int32_t* src,
                                 const int32_t* dst, const int32_t* label, int32_t device, rpq_graph** out);
RPQ_API int rpq_graph_materialize_label(rpq_graph* g, int32_t label);
/* Copy a resident label's CSR (transpose: the backward direction) to host:
 * rowptr uint32[num_vertices+1], col int32[nnz]; either may be NULL. */
RPQ_API int rpq_graph_copy_label(const rpq_graph* g, int32_t label, int32_t transpose, uint32_t* rowptr,
                                 int32_t* col, int64_t col_capacity, int64_t* nnz);
RPQ_API int rpq_graph_label_resident(const rpq_graph* g, int32_t label);
RPQ_API int64_t rpq_graph_device_bytes(const rpq_graph* g);
RPQ_API int rpq_graph_destroy(rpq_graph* g);

/* ---- queries ------------------------------------------------------------- */
/* Transitions are (t_src[i] --(t_label[i], t_inv[i])--> t_dst[i]); those with
 * t_label >= num_labels are dropped (engine.py:100-101).  Every usable label
 * must be resident (else RPQ_ENOLABEL). */
RPQ_API int rpq_query_create(rpq_graph* g, int32_t nstates, int32_t ntrans,
                     const int32_t* t_src, const int32_t* t_label, const uint8_t* t_inv,
                     const int32_t* t_dst, int32_t nstarts, const int32_t* starts,
                     int32_t nfinals, const int32_t* finals, rpq_query** out);
/* Direction policy (RPQ_DIR_*), exact-TE accounting on/off, Beamer's alpha
 * (default: auto, off, 4).  Results do not depend on these. */
RPQ_API int rpq_query_set_options(rpq_query* q, int32_t direction, int32_t count_te, double alpha);
/* Tuning knobs (results do not depend on them):
 *   RPQ_TUNE_EMIT_MODE: how a push level's successors get their work queue --
 *     0 (default) at discovery, 1 from the frontier bitmap in vertex order
 *     (an extra epoch per level), 2 by frontier size;
 *   RPQ_TUNE_EMIT_INLINE_MAX: mode 2 emits at discovery while |F_L| < value. */
#define RPQ_TUNE_EMIT_MODE 0
#define RPQ_TUNE_EMIT_INLINE_MAX 1
#define RPQ_TUNE_FLAGS 3  /* push variants: bit 0 (default on) claim without probing P first,
                             bit 1 prefetch candidate targets' row pointers into L2,
                             bit 2 never cut a push level's emission off at m_u / alpha,
                             bit 3 defer prediction with the all-rows mean degree (round 1),
                             bit 4 push without the shared-memory claim cache */
#define RPQ_TUNE_SMALL 4  /* 1 (default): state spaces of <= 12,288 x 32 pairs run on one CTA
                             with shared-memory bitmaps; 0: always the grid kernel */
#define RPQ_TUNE_DEFER 5  /* push level L does not emit F_{L+1}'s queue at discovery when
                             m_f(F_L) x min(growth, densest slot's mean degree over non-empty rows)
                             x value > m_u (0: always emit; default 1.5) */
#define RPQ_TUNE_TRACE 2  /* diagnostics: record per-CTA phase stamps of the first `value` levels */
#define RPQ_TUNE_ZERO_COPY 6  /* 1 (default): the grid kernel's last CTA writes the statistics
                                 block straight into pinned host memory (no copy node after
                                 the kernel); 0: a device-to-host copy after the kernel */
RPQ_API int rpq_query_set_tuning(rpq_query* q, int32_t key, double value);
/* Enqueue one evaluation from `source` on `stream` (a cudaStream_t, or NULL for
 * the query's own stream).  timeout_s < 0 or inf: no deadline.  The deadline is
 * checked on the device at the top of every iteration, like _Clock.check. */
RPQ_API int rpq_query_run(rpq_query* q, int32_t source, double timeout_s, void* stream);
/* Wait for the last run; fills stats (may be NULL) and returns its status. */
RPQ_API int rpq_query_wait(rpq_query* q, rpq_stats* stats);
/* One evaluation, start to answer, in one call (the eval_ssr fast path):
 * rpq_query_set_options + small-kernel switch + run on the query's stream +
 * wait + the answer bitmap (ceil(nv/32) words; NULL/0 to keep it on the
 * device).  Returns the run's status; stats may be NULL.
 * A source none of whose rows in the start states' symbols has an edge is
 * answered on the host (the first step of the masked loop is empty,
 * engine.py:154-160): no launch, stats->grid == 0.  Not when count_te is set
 * or stats is NULL; accessors of device-side results (rpq_query_copy_visited,
 * _copy_reach[_bits], _reach_device) run such a query on the device first. */
RPQ_API int rpq_query_eval(rpq_query* q, int32_t source, double timeout_s, int32_t direction, int32_t count_te,
                           double alpha, int32_t allow_small, rpq_stats* stats, uint32_t* reach_words,
                           int64_t nwords);
/* rpq_query_eval whose answer may come back as a list: when reach_words lies
 * in an rpq_host_alloc block and stats is non-NULL, a sparse answer (fewer
 * than half of the bitmap's words nonzero) is written as stats->answer_words
 * (word index, word) uint32 pairs at reach_words[0 ..) and stats->answer_list
 * is set; otherwise the bitmap, as rpq_query_eval.  An empty answer moves no
 * bytes.  (The reference's answer is a Python set, engine.py:112-114.) */
RPQ_API int rpq_query_eval_list(rpq_query* q, int32_t source, double timeout_s, int32_t direction,
                                int32_t count_te, double alpha, int32_t allow_small, rpq_stats* stats,
                                uint32_t* reach_words, int64_t nwords);
/* Device pointer to the uint8[num_vertices] answer of the last run (expanded
 * from the answer bitmap on the run's stream on first request). */
RPQ_API int rpq_query_reach_device(rpq_query* q, uint8_t** d_reach);
/* Copy the answer of the last run to host (uint8[num_vertices], 1 = reachable). */
RPQ_API int rpq_query_copy_reach(rpq_query* q, uint8_t* host_reach);
/* One traversal step (step_update, engine.py:127-138): given the frontier M
 * and the visited set P as bitmaps (nstates rows of row_words uint32 words,
 * bit v%32 of word v/32), write mask_complement(step_sum(M), P) -- the pairs
 * one symbol away from M that are not in P -- as a bitmap of the same shape.
 * Synchronous. */
RPQ_API int rpq_query_step(rpq_query* q, const uint32_t* m_words, const uint32_t* p_words, int64_t row_words,
                           uint32_t* out_words);
/* Diagnostics (RPQ_TUNE_TRACE): per level L, CTA c, stamp k (0 level start,
 * 1 plan epoch done, 2 last warp done with the expansion, 3 past the barrier,
 * 4 counters flushed, 7 decision taken (stamped at the decision that
 * starts level L); slots 5-6 unused) in ns from kernel
 * start at host[(L * grid + c) * 8 + k]; *grid receives the CTA count. */
RPQ_API int rpq_query_copy_trace(rpq_query* q, uint64_t* host, int64_t n, int32_t* grid);
/* Owned target words [word_lo, word_hi) of a partitioned rank: a pull step
 * scans only these targets (empty range: all).  Default empty. */
RPQ_API int rpq_query_set_owned(rpq_query* q, int64_t word_lo, int64_t word_hi);
/* Words per state row of the query's bitmaps (>= ceil(nv/32), multiple of 4). */
RPQ_API int rpq_query_row_words(const rpq_query* q, int64_t* row_words);
/* Device-resident step for the vertex-partitioned evaluator:
 * on `stream`, out = step_sum(M) masked by the complement of P, and P |= out,
 * by push or (direction auto/pull, M dense) pull over the owned targets.
 * d_m, d_p, d_out are device bitmaps of nstates rows x rpq_query_row_words
 * words, distinct.  Asynchronous; rpq_query_wait returns its status. */
RPQ_API int rpq_query_step_device(rpq_query* q, const uint32_t* d_m, uint32_t* d_p, uint32_t* d_out,
                                  void* stream);
/* A chain of device steps (one partitioned query): rpq_query_step_begin zeroes
 * the chain's accumulator on `stream`; consecutive rpq_query_step_device calls
 * with unchanged options then enqueue without any host round trip (each step
 * whose M is non-empty counts one iteration of the masked loop, and a failed
 * step latches its status); rpq_query_step_end waits and returns the count
 * and the first failure.  engine.py:157-160 (`while m.nnz` iterations). */
RPQ_API int rpq_query_step_begin(rpq_query* q, void* stream);
RPQ_API int rpq_query_step_end(rpq_query* q, int64_t* steps);
/* Output mode: 0 (default) keeps the answer on the device; 1 also copies the
 * answer bitmap (ceil(nv/32) uint32 words, bit v%32 of word v/32) into pinned
 * host memory as part of every run, ready after rpq_query_wait. */
RPQ_API int rpq_query_set_output(rpq_query* q, int32_t mode);
/* Pinned, device-mapped host memory for answers (cudaHostAlloc mapped |
 * portable).  An answer buffer passed to rpq_query_eval that lies inside such
 * a block is written by the kernel epilogue directly over PCIe: no copy node
 * and no host-side memcpy (the eval_ssr fast path's result arrays).  Replaces
 * nothing in the reference (its answers are Python sets built by
 * _project_finals, engine.py:112-114); rpq_host_free releases a block. */
RPQ_API int rpq_host_alloc(int64_t bytes, void** out);
RPQ_API int rpq_host_free(void* p);
/* The answer of the last run as a bitmap (host copy). */
RPQ_API int rpq_query_copy_reach_bits(rpq_query* q, uint32_t* host_words, int64_t nwords);
/* Copy the full visited matrix P (nstates rows x ceil(nv/32) uint32 words). */
RPQ_API int rpq_query_copy_visited(rpq_query* q, uint32_t* host_words, int64_t nwords);
/* Bytes one run moves: host->device (the automaton tables, re-sent with every
 * run) and device->host (the run's status/statistics block, plus the answer
 * bitmap in output mode 1). */
RPQ_API int rpq_query_io_bytes(const rpq_query* q, int64_t* h2d_per_run, int64_t* d2h_per_run);
RPQ_API int rpq_query_destroy(rpq_query* q);

/* ---- multi-source batches (eval_ssr_batch) ---------------
 * One run evaluates the query from nsrc <= RPQ_BATCH sources at once; answer
 * row s equals rpq_query_run(sources[s]).  Frontier rows are shared by the
 * sources that hold them at the same level (bit-sliced source words).
 * Workspaces are allocated on the first batch run of a query. */
RPQ_API int rpq_query_run_batch(rpq_query* q, int32_t nsrc, const int32_t* sources, double timeout_s,
                                void* stream);
RPQ_API int rpq_query_wait_batch(rpq_query* q, rpq_batch_stats* stats);
/* Answer bitmaps of the last batch run: nsrc rows of row_words uint32 words
 * (>= ceil(nv/32)), bit v%32 of word v/32 of row s = v reachable from sources[s]. */
RPQ_API int rpq_query_copy_batch_bits(rpq_query* q, uint32_t* host_words, int64_t row_words);
/* Device pointer to the same bitmaps (RPQ_BATCH rows of *row_words words). */
RPQ_API int rpq_query_batch_bits_device(rpq_query* q, uint32_t** d_bits, int64_t* row_words);

/* eval_ssr for automata beyond the persistent kernel's table limits (more than
 * 256 states or (state, symbol) groups, more than 128 distinct symbols): the
 * reference's masked loop (rpq/engine.py:146-171; it iterates N.alphabet and
 * has no such limit) as one device push step per level over the transition
 * list in global memory.  Same answer (packed: bit v%32 of word v/32, nwords >=
 * ceil(nv/32)) and the same iteration count; stats carries iterations,
 * visited_pairs, te, reach_count and the per-level counts.  One-shot:
 * workspaces are allocated and freed inside the call. */
RPQ_API int rpq_ssr_wide(rpq_graph* g, int32_t nstates, int32_t ntrans, const int32_t* t_src,
                         const int32_t* t_label, const uint8_t* t_inv, const int32_t* t_dst,
                         int32_t nstarts, const int32_t* starts, int32_t nfinals, const int32_t* finals,
                         int32_t source, double timeout_s, uint32_t* out_bits, int64_t nwords,
                         rpq_stats* stats);

/* One-shot eval_ssr. */
RPQ_API int rpq_ssr(rpq_graph* g, int32_t nstates, int32_t ntrans, const int32_t* t_src,
            const int32_t* t_label, const uint8_t* t_inv, const int32_t* t_dst,
            int32_t nstarts, const int32_t* starts, int32_t nfinals, const int32_t* finals,
            int32_t source, double timeout_s, uint8_t* out_reach, rpq_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* RPQ_B200_H */
