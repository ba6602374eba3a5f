// ssr_kernel.cuh -- the persistent sm_100a kernel that evaluates one
// single-source 2-RPQ: the reference's whole evaluator loop
//   P <- seed; while M: M <- (sum_a (N^a)^T x M x G^a) <not P>; P <- P + M
// (rpq/engine.py:146-171, Alg. 1) in ONE cooperative launch, one
// grid barrier per BFS level.
//
// Layout:
//   slot s          = (label, inverted) symbol; A_s = forward[l] or backward[l]
//                     (graph_store.py:87-91) as uint32 rowptr + int32 columns;
//                     A_s^T (the other direction) is what pull levels scan.
//   group g         = (state q, slot s) with targets {q' : q -s-> q'}: one row
//                     of the transposed transition matrix (engine.py:102).
//   visited P       = |Q| bitmaps of |V| bits; frontier F_L = 3 rotating
//                     bitmaps of the same shape (read L%3, write (L+1)%3,
//                     zero (L+2)%3).
//   push work queue = row SEGMENTS (start, len, group) cut into BUNDLES of
//                     <= 32 edges, double-buffered by level parity, written
//                     by the warp that discovers a pair (sharded counters).
//
// Per level the direction is push (expand the queue) or pull (every
// unvisited (q', w) whose row w of A_s^T is non-empty -- read off a bitmap per
// slot, Params::ne_tab -- scans that row for a frontier member of the source
// state, early exit), chosen from the frontier's edge count against the
// unvisited edge estimate (Beamer's rule).  Either way the result is the
// same set: P only grows by (q', w) pairs with a frontier predecessor.
#pragma once

#include "checks.cuh"

namespace rpqk {
#ifndef RPQ_CUT_SHIFT_UP
#define RPQ_CUT_SHIFT_UP 1
#endif

// One CTA per SM; the thread count is a template parameter of the kernels:
// 768 (24 warps, 80 registers) for small state spaces, where fewer spills win,
// 1024 (32 warps, 64 registers) for large ones, where more warps in flight win
constexpr int kThreads = 768;         // small state spaces
constexpr int kThreadsLarge = 1024;   // large state spaces (and the batch kernel)
#ifndef RPQ_LARGE_PAIRS
#define RPQ_LARGE_PAIRS (8ll << 20)
#endif
constexpr long long kLargePairs = RPQ_LARGE_PAIRS;  // |Q| x |V| from which the large variant runs
constexpr int kMinBlocks = 1;
constexpr int kMaxWarps = kThreadsLarge / 32;
constexpr int kEdgesPerLane = 4;     // push: edges each lane expands per bundle
constexpr int kBundle = 32 * kEdgesPerLane;  // edges per bundle; an emission pass has
                                             // <= 32 segments, so a bundle spans <= 32
constexpr int kShards = 160;         // queue shards, one per CTA (+1 overflow shard)
static_assert(kShards <= 256, "the push shard search (two ballots of 32 x 8) covers 256 shards");
constexpr int kMaxStates = 256;
constexpr int kMaxGroups = 256;      // group id is 8 bits in a segment
constexpr int kMaxSlots = 128;
constexpr uint32_t kSegLenMax = (1u << 24) - 1;
#ifndef RPQ_FAST_GROUPS
#define RPQ_FAST_GROUPS 2
#endif
constexpr int kFastGroups = RPQ_FAST_GROUPS;       // emission: groups per state handled in one pass
// bundle = uint2 {x, y}; y bit 31 = inline, bits 0..6 = edges - 1,
//   inline  : x = column offset of the first edge, y bits 7..14 = group
//   indirect: x = index of the first segment, y bits 7..30 = offset into it
// a hole (bundle slot left empty by a spill) has y = 0xFFFFFFFF
constexpr uint32_t kHoleY = 0xFFFFFFFFu;
constexpr uint32_t kInline = 0x80000000u;
constexpr unsigned FULL = 0xffffffffu;
constexpr int kPullInline = 2;       // in-edges each lane tests before warp help
constexpr unsigned kSeedMinBundle = 4;  // seed level: smallest bundle (edges)

constexpr int ST_OVERFLOW = 100;
constexpr int ST_DEADLOCK = 101;

constexpr int DIR_PUSH = 0;
constexpr int DIR_PULL = 1;

struct Slot {
    const uint32_t* rowptr;
    const int32_t* col;
};

// Counters are never reset while anyone may still read them: queue counters
// rotate over 3 sets by barrier epoch e (produced in epoch e-1, read after
// barrier e, reset in epoch e+1), frontier statistics over 3 sets by level.
// Every CTA reads the same values after a barrier and so takes the same
// decision: no serial section, no broadcast.
struct QCnt {
    unsigned long long shard[kShards + 1];  // (segments << 32) | bundles
    unsigned long long edges;               // push-model edges emitted
    unsigned int overflow;
    unsigned int expire;                    // 1 + level whose deadline check failed
    unsigned long long emit_progress;       // edges emitted so far this level (reported in chunks)
    unsigned int emit_cut;                  // 1: the emission crossed View::cut_edges
    unsigned int big;                       // 1: some bundle of this queue holds more than 32 edges
};

struct FCnt {
    unsigned long long nnew;                // |F_L|
    unsigned int state[kMaxStates];         // |F_L| per state
};

struct Ctl {
    // ---- results prefix: the only part copied back to the host ------------
    unsigned int bar;        // barrier arrivals of this run (the last CTA out resets it to 0)
    int abort;
    unsigned long long t0;
    int status;              // written by CTA 0 only, as are the fields below
    int iterations;
    int levels;
    int pull_levels;
    unsigned long long te_push;
    unsigned long long te_exact;
    unsigned long long segments;
    unsigned long long pairs;
    unsigned long long reach_count;
    unsigned long long t_end;      // globaltimer when the last CTA left (device time = t_end - t0)
    unsigned int done_seq;         // RunArgs::run_seq, written to the host copy last (completion flag)
    unsigned int pad_done;
    unsigned long long ans_words;  // nonzero answer words (out_list runs)
    int ans_list;                  // 1: the host answer buffer holds (word index, word) pairs
    int pad_ans;
    long long level_new[64];
    long long level_edges[64];
    unsigned long long level_ns[64];
    unsigned long long work_ns[64];  // latest CTA finishing level L's work (from t0)
    unsigned long long bar_ns[64];   // CTA 0 leaving the barrier after level L
    int level_dir[64];
    // ---- working counters (zeroed by CTA 0 at the start of every run) -----
    QCnt qc[3];
    FCnt fc[3];
    // tail-bundle counter of the queue qc[i] while it is the current one
    // (reset with qc[i]); one 128-byte line each, away from the counters
    unsigned long long steal[3][16];
    unsigned int exits;  // CTAs past the epilogue (zero-copy results: the last one publishes)
    unsigned long long ans_cursor;  // list-mode answer: next free pair
};

// Per-run inputs, copied host->device with the automaton tables at the start
// of every run (so a captured CUDA graph replays without parameter updates).
struct RunArgs {
    int mode;  // 0: full evaluation from `source`; 1: one step from (M = F_0, P = visited) given
    int source;
    int dir_mode;  // 0 auto, 1 push only, 2 pull after the seed
    int count_te;
    float alpha;   // pull when m_f * alpha > m_u
    unsigned long long budget_ns;
    unsigned int bar_base;  // barrier counter value this run starts from
    int emit_mode;          // 0: emit F_{L+1}'s queue at discovery; 1: from F's bitmap
                            // in vertex order (plan epoch); 2: by frontier size
    unsigned int emit_inline_max;  // mode 2: inline while |F_L| < this
    unsigned int flags;            // RF_* push-path variants (tuning)
    long long own_w0, own_w1;      // step mode: owned word range of a partitioned rank (empty: all)
    float defer_alpha;             // emit at discovery unless mf_L * dmax * this > m_u (0: always emit)
    unsigned int run_seq;          // this run's number: the host polls Ctl::done_seq for it
    int out_list;                  // out_bits may receive a (word index, word) pair list when that is
                                   // smaller than the bitmap (sparse answers; Ctl::ans_list says which)
    uint32_t* out_bits;            // the caller's pinned answer bitmap (rpq_host_alloc), written by the
                                   // epilogue over PCIe, or null (then Params::host_bits)
};

constexpr unsigned RF_NO_PROBE = 1u;     // claim with atomicOr without reading P first
constexpr unsigned RF_PREFETCH = 2u;     // (retired: -30% on cfg4 in round 1; the bit is ignored)
constexpr unsigned RF_NO_CUT = 4u;       // never cut a push level's emission off (View::cut_edges)
constexpr unsigned RF_NO_CACHE = 16u;    // push without the shared-memory claim cache

struct Params {
    const RunArgs* run;
    const int32_t* tables;
    const Slot* slots;       // A_s, then A_s^T at [nslots, 2*nslots)
    const unsigned long long* slot_nnz;
    uint32_t* visited;
    uint32_t* fb[3];
    uint2* seg[2];
    uint2* bun[2];
    Ctl* ctl;
    Ctl* host_ctl;  // device view of the pinned host control block: the last CTA
                    // writes the results prefix there (no copy node), or null
    uint32_t* host_bits;  // device view of the pinned answer bitmap (written by the
                          // epilogue with the device one: no copy node), or null
    uint8_t* reach;
    uint32_t* reach_bits;  // the answer as a bitmap (same bits as reach)
    unsigned long long shard_segcap, shard_buncap, ovf_segcap, ovf_buncap;
    unsigned long long seg_alloc;
    unsigned long long bun_alloc;  // bundles per queue buffer (bounds checks)
    unsigned long long budget_ns;
    long long W;             // words per bitmap row (multiple of 4)
    int nv;
    int nstates, ngroups, nslots, ntargets, nstarts, nfinals, nin;
    int maxT;
    int table_ints;
    unsigned long long* trace;  // diagnostics: [level][cta][4] globaltimer stamps, or null
    float dmax_ne;              // the densest slot's mean degree over its non-empty rows (0: unknown)
    unsigned int* step_acc;     // step mode: [0] steps that found M non-empty, [1] sticky failure
                                // status of any step (zeroed by rpq_query_step_begin)
    int trace_levels;
    // per slot: the non-empty-row bitmap of A_s^T (bit v set when row v has
    // edges; W words), or null -- kept out of Slot (a 24-byte Slot cost the
    // push levels 15%: cfg3's dense one 70 -> 80 us)
    const uint32_t* const* ne_tab;
};

struct Smem {
    const int32_t* gbeg;     // [nstates+1]
    const int32_t* gslot;    // [ngroups]
    const int32_t* toff;     // [ngroups+1]
    const int32_t* targets;  // [ntargets]
    const int32_t* starts;
    const int32_t* finals;
    const int32_t* ibeg;     // [nstates+1] in-transitions (q -> q') per target q'
    const int32_t* isrc;     // [nin]
    const int32_t* islot;    // [nin]
    const Slot* slots;       // [2*nslots]
    const float* nnz;        // [nslots] edges of each slot (decision estimates)
    const uint32_t* const* ne;  // [nslots] non-empty-row bitmaps of the transposes (or null entries)
    const RunArgs* run;      // this run's inputs (shared-memory copy)
    uint64_t pf;             // L2 policy: evict first (graph, queues)
    uint64_t pl;             // L2 policy: evict last (P and F bitmaps)
};

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- L2 residency: the graph streams through L2 (evict-first); the P and F
// bitmaps, probed at random, should stay resident (evict-last) ------------
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* a, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* a, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ld_queue(const uint2* a, uint64_t pol) {  // written earlier in this kernel
    uint2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_queue(uint2* a, uint2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(a), "r"(v.x), "r"(v.y), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* a) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}
__device__ __forceinline__ uint32_t ld_bits(const uint32_t* a, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t or_bits(uint32_t* a, uint32_t b, uint64_t pol) {
    uint32_t v;
    asm volatile("atom.global.L2::cache_hint.or.b32 %0, [%1], %2, %3;" : "=r"(v) : "l"(a), "r"(b), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ void red_or_bits(uint32_t* a, uint32_t b, uint64_t pol) {
    asm volatile("red.global.L2::cache_hint.or.b32 [%0], %1, %2;" ::"l"(a), "r"(b), "l"(pol) : "memory");
}

// control-plane loads after a fence: L2 (coherence point), weak, pipelined
template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
    return __ldcg(p);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}
__device__ __forceinline__ unsigned long long warp_incl_scan_u64(unsigned long long v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long o = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t o = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

// largest lane j with key_j <= x (key non-decreasing across lanes, key_0 <= x)
__device__ __forceinline__ int warp_upper_lane(uint32_t key, uint32_t x) {
    int j = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        int cand = j + step;
        uint32_t k = __shfl_sync(FULL, key, cand & 31);
        if (cand < 32 && k <= x) j = cand;
    }
    return j;
}

// What every thread of a CTA needs to know after a barrier (warp 0 derives it
// from the global counters; all CTAs derive the same values).
struct View {
    int done;
    int dir;        // direction of the level about to run
    int plan;       // push level whose queue must first be emitted from F_L
    int defer;      // push level: do not emit F_{L+1}'s queue at discovery (the next level is likely pull)
    float mf;       // m_f of the last decided frontier (growth estimate)
    float dmax;     // the densest slot's mean degree, nnz / |V| (constant per query)
    int status;
    int iterations;
    unsigned long long nfront;  // |F_L|
    int qbig;                   // F_L's queue holds bundles of more than 32 edges (QCnt::big)
    float cut_edges;            // push level: once the emitted successor edges exceed this, the next
                                // level is pull whatever the rest emits (Beamer's m_f * alpha > m_u with
                                // this level's m_u, which only shrinks): stop emitting (0: never)
};

// Grid barrier for a cooperative launch over a monotonic arrival counter:
// barrier number e completes when e * gridDim.x arrivals are counted.
// Waiters spin on a relaxed load and fence once afterwards (acquire side; the
// fence also invalidates this SM's L1: CCTL.IVALL).
__device__ __forceinline__ void grid_barrier_on(unsigned* bar, int* abort, unsigned epoch, unsigned base) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        const unsigned target = base + epoch * gridDim.x;
        unsigned long long ts = 0;
        unsigned spins = 0;
        while ((int)(ld_relaxed_u32(bar) - target) < 0) {  // wrap-safe
            __nanosleep(16);
            if ((++spins & 4095u) == 0) {
                const unsigned long long now = globaltimer();
                if (ts == 0) {
                    ts = now;
                } else if (now - ts > 20000000000ull) {  // 20 s: cannot happen co-resident
                    atomicExch(abort, 1);
                    break;
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
}
__device__ __forceinline__ void grid_barrier(Ctl* ctl, unsigned epoch, unsigned base) {
    grid_barrier_on(&ctl->bar, &ctl->abort, epoch, base);
}

// Reservation of `nseg` segments and `nb` bundles (one lane).  Each CTA owns
// queue shard blockIdx.x and reserves in it with a shared-memory counter
// (published to the global shard counter once per epoch by flush_counts);
// a reservation that does not fit spills to the overflow shard through a
// global atomic, and the part of its bundle range inside the CTA's shard,
// [*hole_lo, *hole_hi), must then be filled with holes (y = kHoleY).
__device__ __forceinline__ bool reserve(const Params& p, unsigned long long* s_resv, QCnt* qc,
                                        uint32_t nseg, uint32_t nb, unsigned long long* seg_idx,
                                        unsigned long long* bun_idx, unsigned long long* hole_lo,
                                        unsigned long long* hole_hi) {
    const int shard = blockIdx.x;
    const unsigned long long inc = ((unsigned long long)nseg << 32) | nb;
    const unsigned long long old = atomicAdd(s_resv, inc);
    const unsigned long long s_loc = old >> 32, b_loc = old & 0xFFFFFFFFull;
    *hole_lo = *hole_hi = 0;
    if (s_loc + nseg <= p.shard_segcap && b_loc + nb <= p.shard_buncap) {
        *seg_idx = (unsigned long long)shard * p.shard_segcap + s_loc;
        *bun_idx = (unsigned long long)shard * p.shard_buncap + b_loc;
        return true;
    }
    if (b_loc < p.shard_buncap) {
        *hole_lo = (unsigned long long)shard * p.shard_buncap + b_loc;
        *hole_hi = (unsigned long long)shard * p.shard_buncap +
                   (b_loc + nb < p.shard_buncap ? b_loc + nb : p.shard_buncap);
    }
    const unsigned long long o2 = atomicAdd(&qc->shard[kShards], inc);
    const unsigned long long s2 = o2 >> 32, b2 = o2 & 0xFFFFFFFFull;
    if (s2 + nseg <= p.ovf_segcap && b2 + nb <= p.ovf_buncap) {
        *seg_idx = (unsigned long long)kShards * p.shard_segcap + s2;
        *bun_idx = (unsigned long long)kShards * p.shard_buncap + b2;
        return true;
    }
    return false;
}

// Where an epoch's emission goes.
struct Out {
    QCnt* qc;
    uint2* seg;
    uint2* bun;
    unsigned long long* s_resv;  // this CTA's shard fill: (segments << 32) | bundles
    uint32_t bsz;                // edges per emitted bundle (32..kBundle)
    float gain;                  // > 0: a pass emitting T edges of a group cuts them into bundles of
                                 // clamp(T * gain, bsz, kBundle) edges.  A level with few bundles emits
                                 // small ones so that its successor spreads over every warp -- but when
                                 // every pass emits thousands of edges (R-MAT grows 200x a level early
                                 // on) the successor has bundles to spare, and 32-edge ones cost it four
                                 // descriptors where one would do
};

// Warp-cooperative emission of the row segments of (state q, vertex w) pairs
// (one candidate per lane).  Returns the edges emitted.
__device__ __forceinline__ uint32_t emit_pairs(const Params& p, const Smem& S, const Out& o, bool valid,
                                               int q, int w, int lane) {
    if (valid && !RPQ_CHECK(q >= 0 && q < p.nstates && w >= 0 && w < p.nv, RPQ_F_SSR)) valid = false;
    const unsigned vmask = __ballot_sync(FULL, valid);
    if (vmask == 0) return 0;
    const int ng = valid ? (S.gbeg[q + 1] - S.gbeg[q]) : 0;
    int maxng = ng;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) maxng = max(maxng, __shfl_xor_sync(FULL, maxng, d));
    if (maxng <= kFastGroups) {
        // all groups' row pointers in flight together, one reservation
        uint32_t lo[kFastGroups], deg[kFastGroups];
        int g[kFastGroups];
#pragma unroll
        for (int k = 0; k < kFastGroups; ++k) {
            lo[k] = 0;
            deg[k] = 0;
            g[k] = 0;
            if (k < ng) {
                g[k] = S.gbeg[q] + k;
                const Slot sl = S.slots[S.gslot[g[k]]];
                lo[k] = ld_stream_u32(sl.rowptr + w, S.pf);
                deg[k] = ld_stream_u32(sl.rowptr + w + 1, S.pf);
            }
        }
        bool huge = false;
#pragma unroll
        for (int k = 0; k < kFastGroups; ++k) {
            deg[k] -= lo[k];
            huge |= deg[k] > kSegLenMax;
        }
        if (!__any_sync(FULL, huge)) {
            uint32_t excl[kFastGroups], T[kFastGroups], nb[kFastGroups], nseg[kFastGroups];
            bool anybig = false;
            // bundle size of a group's T edges (recomputed where needed: no register array)
            auto bsz_of = [&](uint32_t Tk) -> uint32_t {
                return o.gain > 0.0f ? min((uint32_t)kBundle, max(o.bsz, (uint32_t)((float)Tk * o.gain))) : o.bsz;
            };
            int rank[kFastGroups];
            uint32_t NS = 0, NB = 0, TT = 0;
#pragma unroll
            for (int k = 0; k < kFastGroups; ++k) {
                if (k < maxng) {
                    const unsigned m = __ballot_sync(FULL, deg[k] > 0);
                    rank[k] = __popc(m & lanemask_lt());
                    nseg[k] = (uint32_t)__popc(m);
                    const uint32_t incl = warp_incl_scan(deg[k], lane);
                    excl[k] = incl - deg[k];
                    T[k] = __shfl_sync(FULL, incl, 31);
                    const uint32_t bk = bsz_of(T[k]);
                    anybig |= bk > 32u && T[k] > 32u;
                    nb[k] = (T[k] + bk - 1) / bk;
                    NS += nseg[k];
                    NB += nb[k];
                    TT += T[k];
                } else {
                    rank[k] = 0;
                    nseg[k] = nb[k] = T[k] = excl[k] = 0;
                }
            }
            if (NB == 0) return 0;
            unsigned long long sbase = 0, bbase = 0, hlo = 0, hhi = 0;
            int ok = 1;
            if (lane == 0) ok = reserve(p, o.s_resv, o.qc, NS, NB, &sbase, &bbase, &hlo, &hhi) ? 1 : 0;
            ok = __shfl_sync(FULL, ok, 0);
            hlo = __shfl_sync(FULL, hlo, 0);
            hhi = __shfl_sync(FULL, hhi, 0);
            for (unsigned long long h = hlo + lane; h < hhi; h += 32)
                if (RPQ_CHECK(h < p.bun_alloc, RPQ_F_SSR)) o.bun[h] = make_uint2(0u, kHoleY);
            if (!ok) {
                if (lane == 0) atomicExch(&o.qc->overflow, 1u);
                return 0;
            }
            if (anybig && o.bsz <= 32u && lane == 0) o.qc->big = 1u;  // (same value from every writer)
            sbase = __shfl_sync(FULL, sbase, 0);
            bbase = __shfl_sync(FULL, bbase, 0);
#pragma unroll
            for (int k = 0; k < kFastGroups; ++k) {
                if (k >= maxng) break;
                if (nb[k] == 0) continue;
                bool need_seg = false;
                for (uint32_t kb0 = 0; kb0 < nb[k]; kb0 += 32) {
                    const uint32_t kb = kb0 + lane;
                    const uint32_t bk = bsz_of(T[k]);
                    const uint32_t pos = kb * bk;
                    const uint32_t cnt = kb < nb[k] ? min(bk, T[k] - pos) : 1u;
                    const uint32_t first = min(pos, T[k] - 1);
                    const int j = warp_upper_lane(excl[k], first);
                    const int jl = warp_upper_lane(excl[k], min(pos + cnt - 1, T[k] - 1));
                    const uint32_t exj = __shfl_sync(FULL, excl[k], j);
                    const int rj = __shfl_sync(FULL, rank[k], j);
                    const uint32_t loj = __shfl_sync(FULL, lo[k], j);
                    const int gj = __shfl_sync(FULL, g[k], j);
                    if (kb < nb[k]) {
                        uint2 bd;
                        if (j == jl) {  // within one row: carry the row offset inline
                            bd = make_uint2(loj + (pos - exj), kInline | ((uint32_t)gj << 7) | (cnt - 1));
                        } else {
                            bd = make_uint2((uint32_t)(sbase + rj), ((pos - exj) << 7) | (cnt - 1));
                            need_seg = true;
                        }
                        if (RPQ_CHECK(bbase + kb < p.bun_alloc, RPQ_F_SSR)) st_queue(o.bun + bbase + kb, bd, S.pf);
                    }
                }
                if (__any_sync(FULL, need_seg) && deg[k] > 0 && RPQ_CHECK(sbase + rank[k] < p.seg_alloc, RPQ_F_SSR))
                    st_queue(o.seg + sbase + rank[k], make_uint2(lo[k], (deg[k] << 8) | (uint32_t)g[k]), S.pf);
                sbase += nseg[k];
                bbase += nb[k];
            }
            return TT;
        }
    }
    uint32_t emitted = 0;
    for (int k = 0; k < maxng; ++k) {
        uint32_t lo = 0, deg = 0;
        int g = 0;
        if (k < ng) {
            g = S.gbeg[q] + k;
            const Slot sl = S.slots[S.gslot[g]];
            lo = ld_stream_u32(sl.rowptr + w, S.pf);
            deg = ld_stream_u32(sl.rowptr + w + 1, S.pf) - lo;
        }
        for (;;) {  // rows longer than a segment are split (rare)
            const uint32_t take = min(deg, kSegLenMax);
            const bool hs = take > 0;
            const unsigned m = __ballot_sync(FULL, hs);
            if (m == 0) break;
            const int rank = __popc(m & lanemask_lt());
            const uint32_t nseg = (uint32_t)__popc(m);
            const uint32_t incl = warp_incl_scan(take, lane);
            const uint32_t excl = incl - take;
            const uint32_t T = __shfl_sync(FULL, incl, 31);
            const uint32_t nb = (T + o.bsz - 1) / o.bsz;
            unsigned long long sbase = 0, bbase = 0, hlo = 0, hhi = 0;
            int ok = 1;
            if (lane == 0) ok = reserve(p, o.s_resv, o.qc, nseg, nb, &sbase, &bbase, &hlo, &hhi) ? 1 : 0;
            ok = __shfl_sync(FULL, ok, 0);
            hlo = __shfl_sync(FULL, hlo, 0);
            hhi = __shfl_sync(FULL, hhi, 0);
            for (unsigned long long h = hlo + lane; h < hhi; h += 32)
                if (RPQ_CHECK(h < p.bun_alloc, RPQ_F_SSR)) o.bun[h] = make_uint2(0u, kHoleY);
            if (!ok) {
                if (lane == 0) atomicExch(&o.qc->overflow, 1u);
                return emitted;
            }
            sbase = __shfl_sync(FULL, sbase, 0);
            bbase = __shfl_sync(FULL, bbase, 0);
            if (hs && RPQ_CHECK(sbase + rank < p.seg_alloc, RPQ_F_SSR))
                o.seg[sbase + rank] = make_uint2(lo, (take << 8) | (uint32_t)g);
            for (uint32_t kb0 = 0; kb0 < nb; kb0 += 32) {
                const uint32_t kb = kb0 + lane;
                const uint32_t pos = kb * o.bsz;
                const int j = warp_upper_lane(excl, min(pos, T - 1));
                const uint32_t exj = __shfl_sync(FULL, excl, j);
                const int rj = __shfl_sync(FULL, rank, j);
                if (kb < nb && RPQ_CHECK(bbase + kb < p.bun_alloc, RPQ_F_SSR)) {
                    const uint32_t cnt = min(o.bsz, T - pos);
                    o.bun[bbase + kb] = make_uint2((uint32_t)(sbase + rj), ((pos - exj) << 7) | (cnt - 1));
                }
            }
            emitted += T;
            lo += take;
            deg -= take;
        }
    }
    return emitted;
}

// Per-warp staging of discovered pairs so that emission passes are full
// (a pass emits 32).  stage_add keeps <= 63 staged; the push loop stages a
// whole bundle (stage_put, <= 31 + 32 x kEdgesPerLane) and drains it once, so
// its body holds one inlined emission instead of one per unrolled edge slot.
constexpr int kStageCap = 32 * kEdgesPerLane + 32;
// Per-warp dynamic shared memory: the push emission stage (with the warp's
// share of the claim cache behind it), or (pull epochs) the
// candidate queue: 768 vertex ids (736 + 32 found words in the step-loop variant).
constexpr int kWarpScratchWords = 776;
static_assert(kWarpScratchWords >= 2 * kStageCap, "the emission stage fits the warp scratch");
__host__ __device__ constexpr size_t kStageBytes(int nthreads) {
    return (size_t)(nthreads / 32) * kWarpScratchWords * 4;
}
struct Stage {
    int* q;  // smem [kStageCap]
    int* w;  // smem [kStageCap]
    int n;
};

__device__ __forceinline__ void stage_put(Stage& st, bool fresh, int q, int w, int lane) {
    const unsigned m = __ballot_sync(FULL, fresh);
    if (fresh) {
        const int pos = st.n + __popc(m & lanemask_lt());
        st.q[pos] = q;
        st.w[pos] = w;
    }
    st.n += __popc(m);
}

__device__ __forceinline__ uint32_t stage_add(const Params& p, const Smem& S, const Out& o, Stage& st,
                                              bool fresh, int q, int w, int lane) {
    const unsigned m = __ballot_sync(FULL, fresh);
    if (!m) return 0;
    if (fresh) {
        const int pos = st.n + __popc(m & lanemask_lt());
        st.q[pos] = q;
        st.w[pos] = w;
    }
    st.n += __popc(m);
    __syncwarp();
    uint32_t T = 0;
    if (st.n >= 32) {
        const int qq = st.q[lane], ww = st.w[lane];
        __syncwarp();
        T = emit_pairs(p, S, o, true, qq, ww, lane);
        const int rem = st.n - 32;
        int tq = 0, tw = 0;
        if (lane < rem) {
            tq = st.q[32 + lane];
            tw = st.w[32 + lane];
        }
        __syncwarp();
        if (lane < rem) {
            st.q[lane] = tq;
            st.w[lane] = tw;
        }
        st.n = rem;
        __syncwarp();
    }
    return T;
}

// emit every full pass of 32 staged pairs; keep the remainder (< 32)
__device__ __forceinline__ uint32_t stage_drain(const Params& p, const Smem& S, const Out& o, Stage& st,
                                                int lane) {
    if (st.n < 32) return 0;
    __syncwarp();
    uint32_t T = 0;
    int base = 0;
    for (; st.n - base >= 32; base += 32) {
        const int qq = st.q[base + lane], ww = st.w[base + lane];
        T += emit_pairs(p, S, o, true, qq, ww, lane);
    }
    const int rem = st.n - base;
    int tq = 0, tw = 0;
    if (lane < rem) {
        tq = st.q[base + lane];
        tw = st.w[base + lane];
    }
    __syncwarp();
    if (lane < rem) {
        st.q[lane] = tq;
        st.w[lane] = tw;
    }
    st.n = rem;
    __syncwarp();
    return T;
}

__device__ __forceinline__ uint32_t stage_flush(const Params& p, const Smem& S, const Out& o, Stage& st,
                                                int lane) {
    if (st.n == 0) return 0;
    const bool v = lane < st.n;
    const int qq = v ? st.q[lane] : 0, ww = v ? st.w[lane] : 0;
    __syncwarp();
    st.n = 0;
    return emit_pairs(p, S, o, v, qq, ww, lane);
}

// End-of-epoch flush of a CTA's counts: one atomic per CTA and counter.
__device__ __forceinline__ void flush_counts(unsigned long long* nnew_dst, const Out& o,
                                             unsigned int* state_dst, unsigned long long nnew,
                                             unsigned long long nedge, unsigned long long* red,
                                             unsigned int* s_state, int nstates) {
    unsigned long long* edges_dst = &o.qc->edges;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    nnew = warp_sum_u64(nnew);
    nedge = warp_sum_u64(nedge);
    if (lane == 0) {
        red[2 * wid] = nnew;
        red[2 * wid + 1] = nedge;
    }
    __syncthreads();
    if (wid == 0) {
        const int nwarp = (int)(blockDim.x >> 5);
        unsigned long long a = lane < nwarp ? red[2 * lane] : 0ull;
        unsigned long long c = lane < nwarp ? red[2 * lane + 1] : 0ull;
        a = warp_sum_u64(a);
        c = warp_sum_u64(c);
        if (lane == 0 && a && nnew_dst) atomicAdd(nnew_dst, a);
        if (lane == 0 && c) atomicAdd(edges_dst, c);
        if (lane == 0) {  // publish this CTA's shard fill (the local counter may exceed capacity)
            o.qc->shard[blockIdx.x] = *o.s_resv;
            *o.s_resv = 0;
        }
    }
    if (state_dst)
        for (int q = threadIdx.x; q < nstates; q += blockDim.x) {
            const unsigned int c = s_state[q];
            if (c) {
                atomicAdd(&state_dst[q], c);
                s_state[q] = 0;
            }
        }
}

// Totals of the queue produced in the previous epoch, and the per-shard
// bundle prefix the consumers index with.  Warp-cooperative (warp 0).
__device__ __forceinline__ void queue_scan(const Params& p, const QCnt* qc, int lane,
                                           unsigned long long* s_bpre, unsigned long long* nbun,
                                           unsigned long long* nseg) {
    // lane l owns shards [l*R, l*R + R): all loads in flight, a serial prefix
    // per lane, one warp scan of the lane totals
    constexpr int R = (kShards + 1 + 31) / 32;
    unsigned long long c[R];
    unsigned long long tot = 0, segs = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int sh = lane * R + r;
        const unsigned long long v = sh <= kShards ? ldcg(&qc->shard[sh]) : 0ull;
        const unsigned long long bcap = sh < kShards ? p.shard_buncap : p.ovf_buncap;
        const unsigned long long scap = sh < kShards ? p.shard_segcap : p.ovf_segcap;
        c[r] = min(v & 0xFFFFFFFFull, bcap);
        segs += min(v >> 32, scap);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) tot += c[r];
    const unsigned long long incl = warp_incl_scan_u64(tot, lane);
    unsigned long long run = incl - tot;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int sh = lane * R + r;
        if (sh <= kShards) s_bpre[sh] = run;
        run += c[r];
    }
    const unsigned long long total = __shfl_sync(FULL, incl, 31);
    if (lane == 0) s_bpre[kShards + 1] = total;
    *nbun = total;
    *nseg = warp_sum_u64(segs);
}

// Decision after frontier F_L has been produced (warp 0 of every CTA; every
// CTA reads the same counters and reaches the same result).  Mirrors the
// masked loop (engine.py:156-160): run while the frontier is non-empty,
// check the deadline, then step; and picks the direction of level L.
__device__ void decide_level(const Params& p, const Smem& S, unsigned e, int L, int prev_queued, int prev_dir,
                             int lane,
                             View* v, unsigned long long* s_bpre, unsigned long long* s_sv,
                             unsigned int* s_front) {
    Ctl* ctl = p.ctl;
    if (p.trace && L < p.trace_levels && lane == 0)  // diagnostics: decision entered
        p.trace[((long long)L * gridDim.x + blockIdx.x) * 8 + 6] = globaltimer() - ctl->t0;
    const QCnt* qc = &ctl->qc[e % 3];
    const FCnt* fc = &ctl->fc[L % 3];
    // every load of the decision in flight at once (one L2 round trip)
    constexpr int RS = kMaxStates / 32;
    unsigned int fst[RS];
#pragma unroll
    for (int r = 0; r < RS; ++r) fst[r] = 32 * r + lane < p.nstates ? ldcg(&fc->state[32 * r + lane]) : 0u;
    const unsigned long long nnew = ldcg(&fc->nnew);
    const unsigned long long nedge = ldcg(&qc->edges);
    const unsigned int overflow = ldcg(&qc->overflow);
    const unsigned int expire = ldcg(&qc->expire);
    const unsigned int emit_cut = ldcg(&qc->emit_cut);
    const unsigned int qbig = ldcg(&qc->big);
    const int abort = ldcg(&ctl->abort);
    unsigned long long nbun, nseg;
    queue_scan(p, qc, lane, s_bpre, &nbun, &nseg);
#pragma unroll
    for (int r = 0; r < RS; ++r) {
        const int q = 32 * r + lane;
        if (q < p.nstates) {
            s_front[q] = fst[r];
            s_sv[q] += fst[r];
        }
    }
    __syncwarp();
    if (p.trace && L < p.trace_levels && lane == 0)  // diagnostics: the decision's loads are back
        p.trace[((long long)L * gridDim.x + blockIdx.x) * 8 + 5] = globaltimer() - ctl->t0;
    // F_L's queue was emitted at discovery (exact m_f and bundles available)
    const int produced_by_push = prev_queued;
    int done = 0, iterations = 0, status = 0, next = DIR_PUSH, plan = 0;
    bool defer = false;
    float cut = 0.0f;
    long long ledges = -1;
    if (abort) {
        status = ST_DEADLOCK;
        done = 1;
    } else if (overflow) {
        status = ST_OVERFLOW;
        iterations = L;
        done = 1;
    } else if (expire) {
        status = RPQ_ETIMEOUT;
        iterations = (int)expire - 1;
        done = 1;
    } else if (nnew == 0) {
        iterations = L;
        done = 1;
    } else {
        if (S.run->dir_mode == 2) {
            next = DIR_PULL;
        } else if (S.run->dir_mode == 0) {
            // m_f: edges out of F_L (exact after a push level, estimated from
            // average degrees after a pull level); m_u: in-edges of unvisited
            // targets whose source state has a frontier.  Pull when
            // m_f * alpha > m_u (Beamer's rule; alpha tuned for these kernels).
            const float nv = (float)p.nv, inv_nv = __frcp_rn((float)p.nv);  // (no division subroutine)
            float mf = 0.0f, mu = 0.0f;
            int ntarget = 0;  // states a pull level would scan
            for (int q = lane; q < p.nstates; q += 32) {
                bool t = false;
                float unvis_frac = (nv - (float)s_sv[q]) * inv_nv;
                for (int k = S.ibeg[q]; k < S.ibeg[q + 1]; ++k)
                    if (s_front[S.isrc[k]]) {
                        t = true;
                        mu += S.nnz[S.islot[k]] * unvis_frac;
                    }
                ntarget += t ? 1 : 0;
                if (!produced_by_push && s_front[q]) {
                    const float fq = (float)s_front[q] * inv_nv;
                    for (int g = S.gbeg[q]; g < S.gbeg[q + 1]; ++g) mf += fq * S.nnz[S.gslot[g]];
                }
            }
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
                ntarget += __shfl_xor_sync(FULL, ntarget, d);
                mu += __shfl_xor_sync(FULL, mu, d);
                mf += __shfl_xor_sync(FULL, mf, d);
            }
            if (produced_by_push) mf = (float)nedge;
            // Emission cutoff for a push level: once its emitted successor
            // edges exceed m_u / alpha, the next level will almost surely be
            // pull (m_u only shrinks; the next frontier's states may read other
            // in-slots, so this is a heuristic -- a cut forces pull below,
            // which is always correct, only possibly slower)
            cut = (S.run->flags & RF_NO_CUT) ? 0.0f : mu * __frcp_rn(S.run->alpha) * 1.01f + 64.0f;
            // a push level whose successor frontier will likely warrant pull
            // does not emit that frontier's queue at discovery: a pull level
            // needs none (a push level re-emits it from the bitmap instead).
            // Predicted m_f(F_{L+1}) = m_f(F_L) x min(last growth, densest
            // slot's mean degree), tested like the real decision will be.
            if (S.run->defer_alpha > 0.0f) {
                const float dmax = v->dmax;  // densest slot's mean degree (per query, set at start)
                const float growth = __fdividef(mf, fmaxf(v->mf, 1.0f));
                defer = L > 0 && mf * fminf(growth, dmax) * S.run->defer_alpha > mu;
            }
            __syncwarp();  // every lane has read the previous m_f
            if (lane == 0) v->mf = mf;
            if (produced_by_push) {
                next = (mf * S.run->alpha > mu) ? DIR_PULL : DIR_PUSH;
            } else {
                // after a pull level stay in pull while the frontier is large
                // (Beamer: |F| > |V| / beta, beta = 24, with |V| counted once
                // per state the pull would scan); switching back costs a plan
                // epoch that re-emits F from its bitmap
                next = ((float)nnew * 24.0f > nv * (float)ntarget) ? DIR_PULL : DIR_PUSH;
            }
        }
        // a cut-off emission left F_L's queue incomplete: pull
        if (emit_cut && produced_by_push) next = DIR_PULL;
        if (next == DIR_PUSH) {
            if (produced_by_push) {
                ledges = (long long)nedge;
                if (nbun == 0) {  // nothing to expand: the next step is empty
                    iterations = L + 1;
                    done = 1;
                }
            } else {
                plan = 1;  // emit F_L's queue from its bitmap first
            }
        }
    }
    if (p.trace && L < p.trace_levels && lane == 0)
        p.trace[((long long)L * gridDim.x + blockIdx.x) * 8 + 7] = globaltimer() - ctl->t0;
    if (lane == 0) {
        v->done = done;
        v->dir = next;
        v->plan = plan;
        v->status = status;
        v->iterations = iterations;
        v->nfront = nnew;
        v->qbig = (int)qbig;
        v->defer = next == DIR_PUSH && defer;
        v->cut_edges = next == DIR_PUSH && !defer ? cut : 0.0f;
        if (blockIdx.x == 0) {  // results and statistics
            const unsigned long long now = globaltimer();
            atomicAdd(&ctl->pairs, nnew);  // fire-and-forget: no round trip on CTA 0's path
            if (L < 64) {
                ctl->level_new[L] = (long long)nnew;
                ctl->level_ns[L] = now - ctl->t0;
                ctl->level_edges[L] = ledges;
                ctl->level_dir[L] = next;
            }
            // count_te: a pull level L-1 also counted F_{L-1}'s push-model edges
            if (L >= 1 && L - 1 < 64 && prev_dir == DIR_PULL && S.run->count_te)
                ctl->level_edges[L - 1] = (long long)nedge;
            if (!done) {
                if (L > 0) ctl->levels = L;
                if (next == DIR_PULL) atomicAdd(&ctl->pull_levels, 1);
                if (next == DIR_PUSH && produced_by_push) {
                    atomicAdd(&ctl->te_push, nedge);
                    atomicAdd(&ctl->segments, nseg);
                }
                // _Clock.check at the top of iteration L (engine.py:87-89):
                // recorded now, acted upon at the next decision by every CTA
                if (now - ctl->t0 > S.run->budget_ns) ctl->qc[(e + 1) % 3].expire = (unsigned)L + 1;
            } else {
                ctl->status = status;
                ctl->iterations = iterations;
            }
        }
    }
}

// Decision after a plan epoch emitted F_L's queue.
__device__ void decide_plan(const Params& p, unsigned e, int L, int lane, View* v, unsigned long long* s_bpre) {
    Ctl* ctl = p.ctl;
    const QCnt* qc = &ctl->qc[e % 3];
    const unsigned long long nedge = ldcg(&qc->edges);
    const unsigned int overflow = ldcg(&qc->overflow);
    const unsigned int expire = ldcg(&qc->expire);
    const int abort = ldcg(&ctl->abort);
    unsigned long long nbun, nseg;
    queue_scan(p, qc, lane, s_bpre, &nbun, &nseg);
    int done = 0, status = 0, iterations = 0;
    if (abort) {
        status = ST_DEADLOCK;
        done = 1;
    } else if (overflow) {
        status = ST_OVERFLOW;
        iterations = L;
        done = 1;
    } else if (expire) {
        status = RPQ_ETIMEOUT;
        iterations = (int)expire - 1;
        done = 1;
    } else if (nbun == 0) {
        iterations = L + 1;
        done = 1;
    }
    if (lane == 0) {
        v->done = done;
        v->plan = 0;
        v->qbig = 0;  // (a plan epoch emits with gain 0)
        v->status = status;
        v->iterations = iterations;
        if (blockIdx.x == 0) {
            if (L < 64) ctl->level_edges[L] = (long long)nedge;
            ctl->te_push += nedge;
            ctl->segments += nseg;
            if (done) {
                ctl->status = status;
                ctl->iterations = iterations;
            }
        }
    }
}

__device__ __forceinline__ void reset_qc(Ctl* ctl, int k, int tid) {
    QCnt* qc = &ctl->qc[k];
    for (int i = tid; i <= kShards; i += blockDim.x) qc->shard[i] = 0;
    if (tid == 0) {
        ctl->steal[k][0] = 0;  // push tail
        ctl->steal[k][8] = 0;  // pull tail
        qc->edges = 0;
        qc->overflow = 0;
        qc->expire = 0;
        qc->emit_progress = 0;
        qc->emit_cut = 0;
        qc->big = 0;
    }
}

// Push-model edges out of frontier F (sum over its pairs of group degree x
// targets): this thread's share of a grid-stride sweep.  count_te only.
__device__ unsigned long long frontier_edges(const Params& p, const Smem& S, const uint32_t* f, long long gtid,
                                             long long gthreads, long long Wn) {
    unsigned long long te = 0;
    for (int q = 0; q < p.nstates; ++q) {
        if (S.gbeg[q + 1] == S.gbeg[q]) continue;
        for (long long i = gtid; i < Wn; i += gthreads) {
            uint32_t bits = __ldcg(f + (long long)q * p.W + i);
            while (bits) {
                const int v = (int)(i * 32 + __ffs(bits) - 1);
                bits &= bits - 1;
                for (int g = S.gbeg[q]; g < S.gbeg[q + 1]; ++g) {
                    const Slot sl = S.slots[S.gslot[g]];
                    te += (unsigned long long)(__ldg(sl.rowptr + v + 1) - __ldg(sl.rowptr + v)) *
                          (unsigned long long)(S.toff[g + 1] - S.toff[g]);
                }
            }
        }
    }
    return te;
}

// n / d and n % d for 32-bit n with inv = floor(2^32 / d) (d >= 2; d == 1: inv
// = 2^32 - 1): the estimate __umulhi(n, inv) is the quotient or one less.  A
// hardware-free 32-bit division is ~20 instructions, and the task dealing of
// the pull and plan epochs does two per task.
struct FastDiv {
    uint32_t d, inv;
    __device__ __forceinline__ explicit FastDiv(uint32_t d_) : d(d_), inv(d_ > 1 ? (uint32_t)(0x100000000ull / d_) : 0xFFFFFFFFu) {}
    __device__ __forceinline__ uint32_t div(uint32_t n, uint32_t* rem) const {
        uint32_t q = __umulhi(n, inv);
        uint32_t r = n - q * d;
        if (r >= d) {
            r -= d;
            ++q;
        }
        *rem = r;
        return q;
    }
};

#ifndef RPQ_PULL_CONT
#define RPQ_PULL_CONT 8
#endif
constexpr int kPullCont = RPQ_PULL_CONT;  // in-edges a lane probes on its own before the warp scans the row
#ifndef RPQ_PULL_STATIC_NUM
#define RPQ_PULL_STATIC_NUM 3  // static share of the pull tasks, in quarters
#endif


// Pull over the in-slots' non-empty-row bitmaps (Params::ne_tab).  Reading
// every row pointer of every unvisited vertex to learn which rows have
// in-edges (one in five to seven on R-MAT) cost ~250 instructions per
// 256-vertex task, and the pull levels were bound by instruction issue, not
// by bytes.  Here a task is TW words of vertices (32 on large graphs: 1,024
// vertices): lane l reads P's word and the bitmap's, candidates = ~P & ne, and
// only candidates' row pointers are ever loaded -- by the probing round, next
// to each other (a lane's candidates are queued consecutively, so adjacent
// lanes of a round read adjacent rows).  The queue holds vertex ids and
// outlives the task: rounds always probe 64 (two per lane, every load of a
// stage in flight together), whatever a single task contributes.  A
// discovery is a RED into P and F: the warp dealt the vertex is the only one
// looking at the pair this level.
// A target with several active in-slots (s_pk < 0) takes them one at a time:
// a slot's rounds finish (recording their hits in `found`) before the next
// slot looks at what is still missing.
#ifndef RPQ_NE_TW
#define RPQ_NE_TW 32  // words of vertices per pull task on large graphs
#endif
constexpr int kNECap = 736;  // queued vertices per warp; + 32 found words <= kWarpScratchWords
static_assert(kNECap + 32 <= kWarpScratchWords, "the vertex queue and the found words fit the warp scratch");

template <int TW>
__device__ __forceinline__ void pull_tasks_ne(const Params& p, const Smem& S, const uint32_t* fcur, uint32_t* fnext,
                                              long long pw0, long long pw1, int lane, unsigned* s_task,
                                              int s_nptarget, const int* s_ptarget, const int* s_pk,
                                              const unsigned int* s_front, unsigned int* s_state, unsigned int& nnew,
                                              unsigned long long* steal, uint32_t* ent, int first) {
    const long long nblk = (pw1 - pw0 + TW - 1) / TW;
    const long long ntask = (long long)s_nptarget * nblk;
    const long long G = gridDim.x;
    const long long nown = ntask >= 16 * G ? (ntask / 4 * RPQ_PULL_STATIC_NUM) / G * G : ntask;
    const FastDiv dblk((uint32_t)nblk), dG((uint32_t)G);
    const uint32_t G32 = (uint32_t)G;
    uint32_t* found = ent + kNECap;  // [32] hits of the current task (targets with several in-slots)
    int n = 0;              // queued vertices (warp-uniform)
    int qk = -1;            // the in-transition they belong to
    int qq2 = 0;            // its target state
    uint32_t qvb = 0;       // first vertex of the task whose hits `found` records
    bool qrec = false;      // record hits in `found`
    auto round = [&]() {
        const int np = min(n, 64);
        const int base = n - np;
        const Slot ps = S.slots[p.nslots + S.islot[qk]];
        const uint32_t* frow = fcur + (long long)S.isrc[qk] * p.W;
        uint32_t v[2], lo[2], hi[2], e[2];
        bool act[2], hit[2];
        int c0[2], c1[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int idx = base + 32 * u + lane;
            act[u] = idx < n;
            v[u] = act[u] ? ent[idx] : 0u;
            if (act[u] && !RPQ_CHECK(v[u] < (uint32_t)p.nv, RPQ_F_SSR)) act[u] = false;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            lo[u] = act[u] ? ld_stream_u32(ps.rowptr + v[u], S.pf) : 0u;
            hi[u] = act[u] ? ld_stream_u32(ps.rowptr + v[u] + 1, S.pf) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (act[u] && !RPQ_CHECK(lo[u] <= hi[u] && hi[u] <= p.slot_nnz[S.islot[qk] % p.nslots], RPQ_F_SSR))
                hi[u] = lo[u];
            if (lo[u] >= hi[u]) act[u] = false;  // (cannot happen for a bitmap built from these rows)
            c0[u] = act[u] ? ld_stream_i32(ps.col + lo[u], S.pf) : -1;
            c1[u] = act[u] && first > 1 && lo[u] + 1 < hi[u] ? ld_stream_i32(ps.col + lo[u] + 1, S.pf) : -1;
            if (act[u] && !RPQ_CHECK(c0[u] >= 0 && c0[u] < p.nv && c1[u] < p.nv, RPQ_F_SSR)) c0[u] = c1[u] = -1;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            hit[u] = (c0[u] >= 0 && ((ld_bits(frow + (c0[u] >> 5), S.pl) >> (c0[u] & 31)) & 1u)) ||
                     (c1[u] >= 0 && ((ld_bits(frow + (c1[u] >> 5), S.pl) >> (c1[u] & 31)) & 1u));
            e[u] = lo[u] + (uint32_t)first;
        }
        n = base;
        // misses continue lane-parallel, two in-edges per entry and round, up
        // to kPullCont edges of the row; longer rows are scanned by the warp
        for (;;) {
            bool go[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) go[u] = act[u] && !hit[u] && e[u] < min(hi[u], lo[u] + (uint32_t)kPullCont);
            if (!__ballot_sync(FULL, go[0] || go[1])) break;
            int d0[2], d1[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                d0[u] = go[u] ? ld_stream_i32(ps.col + e[u], S.pf) : -1;
                d1[u] = go[u] && e[u] + 1 < hi[u] ? ld_stream_i32(ps.col + e[u] + 1, S.pf) : -1;
                if (go[u] && !RPQ_CHECK(d0[u] >= 0 && d0[u] < p.nv && d1[u] < p.nv, RPQ_F_SSR)) d0[u] = d1[u] = -1;
            }
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (go[u]) {
                    hit[u] = (d0[u] >= 0 && ((ld_bits(frow + (d0[u] >> 5), S.pl) >> (d0[u] & 31)) & 1u)) ||
                             (d1[u] >= 0 && ((ld_bits(frow + (d1[u] >> 5), S.pl) >> (d1[u] & 31)) & 1u));
                    e[u] += 2;
                }
        }
        unsigned nhit = 0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            unsigned longs = __ballot_sync(FULL, act[u] && !hit[u] && e[u] < hi[u]);
            while (longs) {
                const int sl = __ffs(longs) - 1;
                longs &= longs - 1;
                const uint32_t rlo = __shfl_sync(FULL, e[u], sl), rhi = __shfl_sync(FULL, hi[u], sl);
                bool found_row = false;
                for (uint32_t ed = rlo; ed < rhi; ed += 128) {
                    int uu[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        uu[c] = ed + 32 * c + lane < rhi ? ld_stream_i32(ps.col + ed + 32 * c + lane, S.pf) : -1;
                    bool hh = false;
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (uu[c] >= 0 && RPQ_CHECK(uu[c] < p.nv, RPQ_F_SSR))
                            hh |= (ld_bits(frow + (uu[c] >> 5), S.pl) >> (uu[c] & 31)) & 1u;
                    if (__ballot_sync(FULL, hh)) {
                        found_row = true;
                        break;
                    }
                }
                if (found_row && lane == sl) hit[u] = true;
            }
            if (act[u] && hit[u]) {
                const long long off = (long long)qq2 * p.W + (v[u] >> 5);
                const uint32_t bit = 1u << (v[u] & 31u);
                red_or_bits(p.visited + off, bit, S.pl);
                red_or_bits(fnext + off, bit, S.pl);
                if (qrec) atomicOr(&found[((v[u] - qvb) >> 5) & 31u], bit);
                ++nnew;
            }
            nhit += __popc(__ballot_sync(FULL, act[u] && hit[u]));
        }
        if (lane == 0 && nhit) atomicAdd(&s_state[qq2], nhit);
        __syncwarp();  // (the queue's tail is rewritten by the next append)
    };
    // One loop, one call site of round() (it is ~500 instructions; inlined at
    // every drain it made the kernel 15% larger, and small levels pay for
    // code size in instruction fetches).  Every iteration first drains the
    // queue down to `limit`, then takes one step: APPEND the pending
    // candidates (`pend`, lane by lane, so a lane's candidates are consecutive
    // entries; a block with more than the queue holds goes in two halves of 16
    // lanes, <= 512 each), or PRODUCE the next (task, in-slot)'s candidates.
    uint32_t pend = 0, pvb = 0, pqvb = 0;  // pending candidates of this lane's word, their base vertex
    int pk = -1, pq2 = 0;                  // ... and their in-transition / target state
    bool prec = false, pfirst = false;     // ... recorded in `found` (several in-slots); first append of the slot
    int limit = kNECap;
    bool fin = false;
    int k_iter = -1, k_end = 0;            // inside a target with several in-slots: next in-transition to look at
    bool have_found = false;
    int q2 = 0;
    uint32_t need = 0, vb = 0;
    bool have = false;
    long long word = 0, word0 = 0;
    // APPEND: the pending candidates go on the queue, or `limit` asks for the
    // drain that must come first (the step is then retried)
    auto try_append = [&]() {
        if (n > 0 && (qk != pk || qrec || prec)) {  // another context's entries finish first
            limit = 0;
            return;
        }
        const uint32_t cnt = __popc(pend);
        const uint32_t incl = warp_incl_scan(cnt, lane);
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        int part = -1;  // -1: every lane; 0 / 1: lanes 0-15 / 16-31
        uint32_t half0 = 0;
        if (n + (int)total > kNECap) {
            if (n > 0) {
                limit = 0;
                return;
            }
            half0 = __shfl_sync(FULL, incl, 15);
            part = half0 > 0 ? 0 : 1;
        }
        const bool mine = part < 0 || (lane >> 4) == part;
        const uint32_t padd = part < 0 ? total : part == 0 ? half0 : total - half0;
        const uint32_t pbase = part == 1 ? half0 : 0u;
        if (prec && pfirst) {
            found[lane] = 0u;
            __syncwarp();
        }
        pfirst = false;
        qk = pk;
        qq2 = pq2;
        qrec = prec;
        qvb = pqvb;
        have_found = prec;
        int pos = n + (int)(incl - cnt - pbase);
        uint32_t m = mine ? pend : 0u;
        while (m) {
            ent[pos++] = pvb + (uint32_t)(__ffs(m) - 1);
            m &= m - 1;
        }
        if (mine) pend = 0u;
        n += (int)padd;
        __syncwarp();
        limit = prec ? 0 : 63;  // several in-slots: the slot's rounds finish; else fewer than a round stay queued
    };
    for (;;) {
        while (n > limit) round();
        if (fin) break;
        limit = kNECap;
        if (__ballot_sync(FULL, pend != 0)) {
            try_append();
            continue;
        }
        // ---- PRODUCE
        if (k_iter >= 0) {
            // a target with several in-slots; the previous slot's rounds are done (limit was 0)
            if (have_found) {
                need &= ~found[lane];
                have_found = false;
                __syncwarp();
            }
            int k = -1;
            if (__ballot_sync(FULL, need != 0))
                for (int kk = k_iter; kk < k_end; ++kk)
                    if (s_front[S.isrc[kk]]) {
                        k = kk;
                        break;
                    }
            if (k < 0) {
                k_iter = -1;
                continue;
            }
            k_iter = k + 1;
            pend = have ? need & ld_stream_u32(S.ne[S.islot[k]] + word, S.pf) : 0u;
            pvb = vb;
            pqvb = (uint32_t)(word0 << 5);
            pk = k;
            pq2 = q2;
            prec = true;
            pfirst = true;
            continue;
        }
        uint32_t task = 0;
        if (lane == 0) {
            const uint32_t i = atomicAdd(s_task, 1u);
            uint32_t rot;
            dG.div(blockIdx.x + i, &rot);
            task = i * G32 + rot;
            if (task >= (uint32_t)nown && nown < ntask) task = (uint32_t)nown + (uint32_t)atomicAdd(steal, 1ull);
        }
        task = __shfl_sync(FULL, task, 0);
        if ((long long)task >= ntask) {
            fin = true;
            limit = 0;
            continue;
        }
        uint32_t blk;
        const uint32_t tq = dblk.div(task, &blk);
        q2 = s_ptarget[tq];
        const int k1 = s_pk[tq];  // the target's only active in-transition, or -1: several
        word0 = pw0 + (long long)blk * TW;
        word = word0 + lane;
        have = lane < TW && word < pw1;
        vb = (uint32_t)(word << 5);
        need = have ? ~ld_bits(p.visited + (long long)q2 * p.W + word, S.pl) : 0u;
        if (k1 >= 0) {
            // (bits past |V| are clear in the bitmap)
            pend = have ? need & ld_stream_u32(S.ne[S.islot[k1]] + word, S.pf) : 0u;
            pvb = vb;
            pk = k1;
            pq2 = q2;
            prec = false;
            pfirst = false;
            if (__ballot_sync(FULL, pend != 0)) try_append();  // (the common step: no second iteration)
        } else {
            k_iter = S.ibeg[q2];
            k_end = S.ibeg[q2 + 1];
            have_found = false;
        }
    }
}

// The same pull for levels whose targets all have ONE active in-slot, on
// large graphs (32-word tasks), without the step loop above: straight-line
// task -> append -> rounds (cfg3's pull levels: 95 + 39 us against 102 + 41).
#ifndef RPQ_NE_PER_LANE
#define RPQ_NE_PER_LANE 2
#endif
constexpr int kNE1Cap = 768;
__device__ __forceinline__ void pull_tasks_ne1(const Params& p, const Smem& S, const uint32_t* fcur, uint32_t* fnext,
                                              long long pw0, long long pw1, int lane, unsigned* s_task,
                                              int s_nptarget, const int* s_ptarget, const int* s_pk,
                                              unsigned int* s_state, unsigned int& nnew,
                                              unsigned long long* steal, uint32_t* ent, int first) {
    const long long nblk = (pw1 - pw0 + 31) >> 5;
    const long long ntask = (long long)s_nptarget * nblk;
    const long long G = gridDim.x;
    const long long nown = ntask >= 16 * G ? (ntask / 4 * RPQ_PULL_STATIC_NUM) / G * G : ntask;
    const FastDiv dblk((uint32_t)nblk), dG((uint32_t)G);
    const uint32_t G32 = (uint32_t)G;
    constexpr int U = RPQ_NE_PER_LANE;  // candidates per lane and round
    int n = 0;    // queued vertices (warp-uniform)
    int qk = -1;  // the in-transition they belong to
    int qq2 = 0;  // its target state
    auto round = [&]() {
        const int np = min(n, 32 * U);
        const int base = n - np;
        const Slot ps = S.slots[p.nslots + S.islot[qk]];
        const uint32_t* frow = fcur + (long long)S.isrc[qk] * p.W;
        uint32_t v[U], lo[U], hi[U], e[U];
        bool act[U], hit[U];
        int c0[U], c1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int idx = base + 32 * u + lane;
            act[u] = idx < n;
            v[u] = act[u] ? ent[idx] : 0u;
            if (act[u] && !RPQ_CHECK(v[u] < (uint32_t)p.nv, RPQ_F_SSR)) act[u] = false;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            lo[u] = act[u] ? ld_stream_u32(ps.rowptr + v[u], S.pf) : 0u;
            hi[u] = act[u] ? ld_stream_u32(ps.rowptr + v[u] + 1, S.pf) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (act[u] && !RPQ_CHECK(lo[u] <= hi[u] && hi[u] <= p.slot_nnz[S.islot[qk] % p.nslots], RPQ_F_SSR))
                hi[u] = lo[u];
            if (lo[u] >= hi[u]) act[u] = false;  // (cannot happen for a bitmap built from these rows)
            c0[u] = act[u] ? ld_stream_i32(ps.col + lo[u], S.pf) : -1;
            c1[u] = act[u] && first > 1 && lo[u] + 1 < hi[u] ? ld_stream_i32(ps.col + lo[u] + 1, S.pf) : -1;
            if (act[u] && !RPQ_CHECK(c0[u] >= 0 && c0[u] < p.nv && c1[u] < p.nv, RPQ_F_SSR)) c0[u] = c1[u] = -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            hit[u] = (c0[u] >= 0 && ((ld_bits(frow + (c0[u] >> 5), S.pl) >> (c0[u] & 31)) & 1u)) ||
                     (c1[u] >= 0 && ((ld_bits(frow + (c1[u] >> 5), S.pl) >> (c1[u] & 31)) & 1u));
            e[u] = lo[u] + (uint32_t)first;
        }
        n = base;
        // misses continue lane-parallel, two in-edges per entry and round, up
        // to kPullCont edges of the row; longer rows are scanned by the warp
        for (;;) {
            bool go[U];
#pragma unroll
            for (int u = 0; u < U; ++u) go[u] = act[u] && !hit[u] && e[u] < min(hi[u], lo[u] + (uint32_t)kPullCont);
            bool anygo = false;
#pragma unroll
            for (int u = 0; u < U; ++u) anygo |= go[u];
            if (!__ballot_sync(FULL, anygo)) break;
            int d0[U], d1[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                d0[u] = go[u] ? ld_stream_i32(ps.col + e[u], S.pf) : -1;
                d1[u] = go[u] && e[u] + 1 < hi[u] ? ld_stream_i32(ps.col + e[u] + 1, S.pf) : -1;
                if (go[u] && !RPQ_CHECK(d0[u] >= 0 && d0[u] < p.nv && d1[u] < p.nv, RPQ_F_SSR)) d0[u] = d1[u] = -1;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (go[u]) {
                    hit[u] = (d0[u] >= 0 && ((ld_bits(frow + (d0[u] >> 5), S.pl) >> (d0[u] & 31)) & 1u)) ||
                             (d1[u] >= 0 && ((ld_bits(frow + (d1[u] >> 5), S.pl) >> (d1[u] & 31)) & 1u));
                    e[u] += 2;
                }
        }
        unsigned nhit = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            unsigned longs = __ballot_sync(FULL, act[u] && !hit[u] && e[u] < hi[u]);
            while (longs) {
                const int sl = __ffs(longs) - 1;
                longs &= longs - 1;
                const uint32_t rlo = __shfl_sync(FULL, e[u], sl), rhi = __shfl_sync(FULL, hi[u], sl);
                bool found_row = false;
                for (uint32_t ed = rlo; ed < rhi; ed += 128) {
                    int uu[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        uu[c] = ed + 32 * c + lane < rhi ? ld_stream_i32(ps.col + ed + 32 * c + lane, S.pf) : -1;
                    bool hh = false;
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (uu[c] >= 0 && RPQ_CHECK(uu[c] < p.nv, RPQ_F_SSR))
                            hh |= (ld_bits(frow + (uu[c] >> 5), S.pl) >> (uu[c] & 31)) & 1u;
                    if (__ballot_sync(FULL, hh)) {
                        found_row = true;
                        break;
                    }
                }
                if (found_row && lane == sl) hit[u] = true;
            }
            if (act[u] && hit[u]) {
                const long long off = (long long)qq2 * p.W + (v[u] >> 5);
                const uint32_t bit = 1u << (v[u] & 31u);
                red_or_bits(p.visited + off, bit, S.pl);
                red_or_bits(fnext + off, bit, S.pl);
                ++nnew;
            }
            nhit += __popc(__ballot_sync(FULL, act[u] && hit[u]));
        }
        if (lane == 0 && nhit) atomicAdd(&s_state[qq2], nhit);
        __syncwarp();  // (the queue's tail is rewritten by the next append)
    };
    for (;;) {
        uint32_t task = 0;
        if (lane == 0) {
            const uint32_t i = atomicAdd(s_task, 1u);
            uint32_t rot;
            dG.div(blockIdx.x + i, &rot);
            task = i * G32 + rot;
            if (task >= (uint32_t)nown && nown < ntask) task = (uint32_t)nown + (uint32_t)atomicAdd(steal, 1ull);
        }
        task = __shfl_sync(FULL, task, 0);
        if ((long long)task >= ntask) break;
        uint32_t blk;
        const uint32_t tq = dblk.div(task, &blk);
        const int q2 = s_ptarget[tq];
        const int k = s_pk[tq];
        const long long word = pw0 + (long long)blk * 32 + lane;
        uint32_t cm = 0;
        if (word < pw1) {
            const uint32_t pwv = ld_bits(p.visited + (long long)q2 * p.W + word, S.pl);
            const uint32_t nev = ld_stream_u32(S.ne[S.islot[k]] + word, S.pf);
            cm = ~pwv & nev;  // (bits past |V| are clear in the bitmap)
        }
        if (__ballot_sync(FULL, cm != 0) == 0) continue;
        if (qk != k)
            while (n > 0) round();
        qk = k;
        qq2 = q2;
        // append lane by lane (a lane's candidates are consecutive entries);
        // a block with more candidates than the queue has room for goes in
        // two halves of 16 lanes (<= 512 candidates each)
        const uint32_t cnt = __popc(cm);
        const uint32_t incl = warp_incl_scan(cnt, lane);
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        const uint32_t half0 = __shfl_sync(FULL, incl, 15);
        const bool split = n + (int)total > kNE1Cap;
        for (int part = 0; part < (split ? 2 : 1); ++part) {
            const bool mine = !split || (lane >> 4) == part;
            const uint32_t padd = !split ? total : part == 0 ? half0 : total - half0;
            const uint32_t pbase = split && part == 1 ? half0 : 0u;
            while (n > 0 && n + (int)padd > kNE1Cap) round();
            int pos = n + (int)(incl - cnt - pbase);
            uint32_t m = mine ? cm : 0u;
            const uint32_t vb = (uint32_t)(word << 5);
            while (m) {
                ent[pos++] = vb + (uint32_t)(__ffs(m) - 1);
                m &= m - 1;
            }
            n += (int)padd;
            __syncwarp();
            while (n >= 32 * U) round();
        }
    }
    while (n > 0) round();
}

// Diagnostic stamp k of level L for this CTA (thread 0): 0 level start (after
// the decision), 1 plan epoch done, 2 last warp done with the expansion,
// 3 past the barrier, 4 counters flushed.
__device__ __forceinline__ void stamp(const Params& p, int L, int k) {
    if (p.trace && L < p.trace_levels && threadIdx.x == 0)
        p.trace[((long long)L * gridDim.x + blockIdx.x) * 8 + k] = globaltimer() - p.ctl->t0;
}

template <int NT>
__global__ void __launch_bounds__(NT, kMinBlocks) ssr_kernel(const __grid_constant__ Params p) {
    constexpr int kWarps = NT / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_red[2 * kWarps];
    __shared__ unsigned long long s_bpre[kShards + 2];
    __shared__ unsigned long long s_sv[kMaxStates];  // |P| per state (same in every CTA)
    __shared__ unsigned int s_front[kMaxStates];     // |F_L| per state
    __shared__ unsigned int s_state[kMaxStates];     // this CTA's discoveries per state
    __shared__ int s_ptarget[kMaxStates];            // pull target states of this level
    __shared__ int s_nptarget;
    __shared__ int s_pmulti;  // some pull target of this level has several active in-slots
    __shared__ int s_pk[kMaxStates];  // first active in-transition of each pull target
    __shared__ View s_view;
    __shared__ unsigned long long s_resv;
    __shared__ unsigned s_task;  // next task index of this CTA in the current epoch
    __shared__ int s_cut;        // this level's emission was cut off (View::cut_edges)
    __shared__ unsigned long long s_emitted;  // edges this CTA emitted this level
    __shared__ unsigned long long s_wend;  // diagnostics: latest warp done with the epoch
    __shared__ RunArgs s_run;
    __shared__ float s_nnz[kMaxSlots];
    __shared__ const uint32_t* s_ne[kMaxSlots];

    // dynamic smem: [emission stages, kStageBytes(NT)] [slots] [tables]
    int* s_stage = reinterpret_cast<int*>(smem_raw);
    Slot* s_slots = reinterpret_cast<Slot*>(smem_raw + kStageBytes(NT));
    for (int i = threadIdx.x; i < p.nslots; i += blockDim.x) {
        s_nnz[i] = (float)p.slot_nnz[i];
        s_ne[i] = p.ne_tab ? p.ne_tab[i] : nullptr;
    }
    int32_t* s_tab = reinterpret_cast<int32_t*>(smem_raw + kStageBytes(NT) + sizeof(Slot) * 2 * p.nslots);
    for (int i = threadIdx.x; i < 2 * p.nslots; i += blockDim.x) s_slots[i] = p.slots[i];
    // the push path's hottest tables (gbeg, gslot, toff: the first three of
    // the block) also at compile-time shared addresses: with 64 registers
    // their run-time offsets were recomputed at every use (11% of cfg4's
    // instructions were address arithmetic).  Filled in the same pass (a second
    // round of global loads in the prologue cost every query 1-2 us).
    __shared__ int32_t s_gbeg[kMaxStates + 1], s_gslot[kMaxGroups], s_toff[kMaxGroups + 1];
    {
        const int o1 = p.nstates + 1, o2 = o1 + p.ngroups, o3 = o2 + p.ngroups + 1;
        for (int i = threadIdx.x; i < p.table_ints; i += blockDim.x) {
            const int32_t v = p.tables[i];
            s_tab[i] = v;
            if (i < o1) s_gbeg[i] = v;
            else if (i < o2) s_gslot[i - o1] = v;
            else if (i < o3) s_toff[i - o2] = v;
        }
    }
    if (threadIdx.x == 0) {
        s_resv = 0;
        s_wend = 0;
    }
    for (int i = threadIdx.x; i < kMaxStates; i += blockDim.x) {
        s_state[i] = 0;
        s_sv[i] = 0;
        s_front[i] = 0;
    }
    if (threadIdx.x == 0) {
        s_run = *p.run;
        s_view.mf = 0.0f;
        s_view.defer = 0;
        s_view.qbig = 0;
        s_view.cut_edges = 0.0f;
        float d = 0.0f;
        for (int sl = 0; sl < p.nslots; ++sl) d = fmaxf(d, (float)p.slot_nnz[sl]);
        // the defer prediction's degree: over non-empty rows when known (the
        // discovered vertices of a BFS are biased to rows with edges; on R-MAT
        // the mean over all rows underestimates their degree ~3x)
        s_view.dmax = p.dmax_ne > 0.0f ? p.dmax_ne : d * __frcp_rn((float)max(p.nv, 1));
    }
    Smem S;
    S.pf = policy_evict_first();
    S.pl = policy_evict_last();
    S.run = &s_run;
    S.slots = s_slots;
    S.nnz = s_nnz;
    S.ne = s_ne;
    S.gbeg = s_gbeg;
    S.gslot = s_gslot;
    S.toff = s_toff;
    S.targets = s_tab + (p.nstates + 1) + p.ngroups + (p.ngroups + 1);
    S.starts = S.targets + p.ntargets;
    S.finals = S.starts + p.nstarts;
    S.ibeg = S.finals + p.nfinals;
    S.isrc = S.ibeg + p.nstates + 1;
    S.islot = S.isrc + p.nin;

    Ctl* ctl = p.ctl;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long gthreads = (long long)gridDim.x * blockDim.x;
    const long long gwarp = (long long)blockIdx.x * kWarps + wid;
    const long long nwarps = (long long)gridDim.x * kWarps;
    const long long Wn = ((long long)p.nv + 31) >> 5;  // used words per bitmap row
    const long long nbits4 = (long long)p.nstates * p.W / 4;
    const bool cta0 = blockIdx.x == 0;
    // The bitmap level L+1 will write F_{L+2} into is F_{L-1}'s, free since
    // the barrier that ended level L-1: warps 1.. zero it while warp 0 takes
    // level L's decision (its loads are a 1.3 us round trip in which the CTA
    // had nothing else to do; the stores used to open the expand epoch).
    auto zero_next = [&](int L_) {
#ifndef RPQ_ZERO_IN_EXPAND
        uint4* z4 = reinterpret_cast<uint4*>(p.fb[(L_ + 2) % 3]);
        const long long zt = (long long)blockIdx.x * (NT - 32) + (threadIdx.x - 32);
        for (long long i = zt; i < nbits4; i += (long long)gridDim.x * (NT - 32)) z4[i] = make_uint4(0, 0, 0, 0);
#endif
    };
    __syncthreads();  // s_run, tables and counters above are read by every thread below
    Stage stage;
    stage.q = s_stage + wid * kWarpScratchWords;
    stage.w = s_stage + wid * kWarpScratchWords + kStageCap;
    stage.n = 0;
    // CTA 0 resets the control block (except the barrier counter, which only
    // grows); nobody else reads it before the first barrier
    if (cta0) {
        unsigned char* z = reinterpret_cast<unsigned char*>(ctl) + 8;  // keep bar, abort set below
        for (size_t i = threadIdx.x * 8; i + 8 <= sizeof(Ctl) - 8; i += (size_t)blockDim.x * 8)
            *reinterpret_cast<unsigned long long*>(z + i) = 0ull;
        if (threadIdx.x == 0) ctl->abort = 0;
        __syncthreads();
        if (threadIdx.x == 0) ctl->t0 = globaltimer();
    }

    unsigned e = 0;  // barriers passed

    const bool step_mode = s_run.mode == 1;  // step_update (engine.py:127-138)
    // ---- epoch 0: P <- 0, F <- 0 (step mode: P and F_0 = M come from the host)
    {
        uint4* v4 = reinterpret_cast<uint4*>(p.visited);
        if (!step_mode)
            for (long long i = gtid; i < nbits4; i += gthreads) v4[i] = make_uint4(0, 0, 0, 0);
        // step mode: F_0 = M is the caller's and only F_1 (the output) is
        // written; a full run clears F_0 and F_1 (level 0's expand epoch
        // clears F_2 before anything is written into it)
        for (int f = step_mode ? 1 : 0; f < 2; ++f) {
            uint4* f4 = reinterpret_cast<uint4*>(p.fb[f]);
            for (long long i = gtid; i < nbits4; i += gthreads) f4[i] = make_uint4(0, 0, 0, 0);
        }
    }
    grid_barrier(ctl, ++e, s_run.bar_base);

    // ---- epoch 1: seed P = M = {(q_s, source)} (engine.py:106-109, :154-155).
    // P was just cleared, so every start state is fresh: every CTA knows the
    // seed rows (the source's rows of each start state's groups) and writes a
    // share of their bundles -- a hub source's row (millions of edges) is not
    // emitted by one warp.  All seed bundles are inline (each lies in one row).
    if (!step_mode) {
        const Out o{&ctl->qc[(e + 1) % 3], p.seg[(e + 1) & 1], p.bun[(e + 1) & 1], &s_resv, 32u, 0.0f};
        if (cta0) reset_qc(ctl, (e + 2) % 3, threadIdx.x);
        unsigned long long nnew = 0, nedge = 0;
        const int src = S.run->source;
        if (cta0 && wid == 0) {  // claim the seed pairs
            for (int i = lane; i < p.nstarts; i += 32) {
                const int q = S.starts[i];
                const long long off = (long long)q * p.W + (src >> 5);
                const uint32_t bit = 1u << (src & 31);
                atomicOr(p.visited + off, bit);
                atomicOr(p.fb[0] + off, bit);
                atomicAdd(&s_state[q], 1u);
                nnew += 1;
            }
        }
        // the seed rows: one per (start state, group), in shared memory
        __shared__ uint32_t s_slo[kMaxGroups], s_sgrp[kMaxGroups];
        __shared__ unsigned long long s_sdeg[kMaxGroups + 1], s_sbun[kMaxGroups + 1];
        __shared__ int s_nrows;
        __shared__ uint32_t s_sbsz;
        if (threadIdx.x == 0) {
            int n = 0;
            unsigned long long edges = 0, bundles = 0;
            s_sdeg[0] = s_sbun[0] = 0;
            for (int i = 0; i < p.nstarts; ++i) {
                const int q = S.starts[i];
                for (int g = S.gbeg[q]; g < S.gbeg[q + 1] && n < kMaxGroups; ++g) {
                    const Slot sl = S.slots[S.gslot[g]];
                    const uint32_t lo = sl.rowptr[src], hi = sl.rowptr[src + 1];
                    s_slo[n] = lo;
                    s_sgrp[n] = (uint32_t)g;
                    edges += hi - lo;
                    s_sdeg[n + 1] = edges;
                    ++n;
                }
            }
            // small seed rows: 32-edge bundles spread the first level over more warps
            // about one bundle per warp (4..128 edges): the source's neighbours
            // are often hubs themselves (R-MAT: low ids), and each bundle's
            // warp emits its discoveries' rows -- few per warp spreads that out
            const unsigned long long per = (edges + nwarps - 1) / (unsigned long long)nwarps;
            const uint32_t bsz = (uint32_t)min(max(per, (unsigned long long)kSeedMinBundle), (unsigned long long)kBundle);
            for (int r = 0; r < n; ++r) {
                bundles += (s_sdeg[r + 1] - s_sdeg[r] + bsz - 1) / bsz;
                s_sbun[r + 1] = bundles;
            }
            s_nrows = n;
            s_sbsz = bsz;
            if (cta0) nedge = edges;
        }
        __syncthreads();
        {
            const int nrows = s_nrows;
            const uint32_t bsz = s_sbsz;
            const unsigned long long nb = s_sbun[nrows];
            // bundle b goes to shard b % G at index b / G (this CTA writes its shard)
            const unsigned long long mine = nb > blockIdx.x ? (nb - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
            if (mine > p.shard_buncap) {
                if (threadIdx.x == 0) atomicExch(&o.qc->overflow, 1u);
            } else {
                for (unsigned long long k = threadIdx.x; k < mine; k += blockDim.x) {
                    const unsigned long long b = blockIdx.x + k * gridDim.x;
                    int r = 0;
                    while (r + 1 < nrows && s_sbun[r + 1] <= b) ++r;  // few rows: linear
                    const unsigned long long pos = (b - s_sbun[r]) * bsz;
                    const unsigned long long deg = s_sdeg[r + 1] - s_sdeg[r];
                    const uint32_t cnt = (uint32_t)min((unsigned long long)bsz, deg - pos);
                    if (RPQ_CHECK((unsigned long long)blockIdx.x * p.shard_buncap + k < p.bun_alloc, RPQ_F_SSR))
                        o.bun[(unsigned long long)blockIdx.x * p.shard_buncap + k] =
                            make_uint2(s_slo[r] + (uint32_t)pos, kInline | (s_sgrp[r] << 7) | (cnt - 1));
                }
                if (threadIdx.x == 0) s_resv = ((cta0 ? (unsigned long long)nrows : 0ull) << 32) | mine;
            }
        }
        __syncthreads();
        flush_counts(&ctl->fc[0].nnew, o, ctl->fc[0].state, nnew, nedge, s_red, s_state, p.nstates);
    }
    if (!step_mode) {
        grid_barrier(ctl, ++e, s_run.bar_base);
        if (wid == 0) decide_level(p, S, e, 0, 1, DIR_PUSH, lane, &s_view, s_bpre, s_sv, s_front);
        else zero_next(0);
    } else {
        // one step from F_0 = M: count M per state (one epoch), then pull
        // (when M is dense against the owned targets) or push (emit M's rows
        // in a plan epoch, expand), and stop
        for (int q = 0; q < p.nstates; ++q) {
            unsigned c = 0;
            const uint32_t* row = p.fb[0] + (long long)q * p.W;
            for (long long i = gtid; i < Wn; i += gthreads) c += __popc(row[i]);
            c = (unsigned)warp_sum_u64(c);
            if (lane == 0 && c) atomicAdd(&ctl->fc[0].state[q], c);
        }
        grid_barrier(ctl, ++e, s_run.bar_base);
        if (threadIdx.x == 0) {
            unsigned long long nf = 0;
            for (int q = 0; q < p.nstates; ++q) {
                s_front[q] = ldcg(&ctl->fc[0].state[q]);
                nf += s_front[q];
            }
            if (cta0 && nf && p.step_acc) atomicAdd(p.step_acc, 1u);  // an iteration of the masked loop
            int ntarget = 0;
            for (int q2 = 0; q2 < p.nstates; ++q2) {
                bool t = false;
                for (int k = S.ibeg[q2]; k < S.ibeg[q2 + 1]; ++k) t |= s_front[S.isrc[k]] != 0;
                ntarget += t ? 1 : 0;
            }
            const long long own = (s_run.own_w1 > s_run.own_w0 ? s_run.own_w1 - s_run.own_w0 : Wn) * 32;
            int dir = s_run.dir_mode == 2 ? DIR_PULL : DIR_PUSH;
            if (s_run.dir_mode == 0 && (float)nf * 24.0f > (float)own * (float)ntarget) dir = DIR_PULL;
            s_view.done = nf == 0;
            s_view.dir = dir;
            s_view.plan = dir == DIR_PUSH;
            s_view.defer = 0;
        s_view.cut_edges = 0.0f;
            s_view.status = 0;
            s_view.iterations = 0;
            s_view.nfront = nf;
        }
    }
    __syncthreads();

#ifndef RPQ_NO_CLAIM_CACHE
    // Claim cache (push): a direct-mapped table in shared memory of P words
    // this CTA has seen, {word index + 1, bits known set}.  An edge whose
    // target bit is known set makes no claim.  On skewed graphs most edges of
    // a push level end on a few hub vertices whose P words share a handful of
    // 128-byte lines: their claims queue at one L2 slice and every warp waits
    // in that queue (cfg3: 2% of a level's claims hit one line).  Entries only
    // hold bits that are set in P (P only grows), so a stale or lost entry
    // costs a claim, never an answer.  One 64-bit shared access per entry:
    // tag and bits cannot tear.  The table lives in the part of each warp's
    // scratch the emission stage does not use (pull epochs overwrite it: it is
    // cleared before the next push epoch).
    constexpr int kPcPerWarp = 128;
    constexpr int kPcEntries = (kWarps >= 32 ? 32 : 16) * kPcPerWarp;  // a power of two
    constexpr int kPcShift = kWarps >= 32 ? 20 : 21;                    // 32 - log2(kPcEntries)
    static_assert(2 * kStageCap + 2 * kPcPerWarp <= kWarpScratchWords, "claim cache fits beside the stage");
    static_assert((2 * kStageCap) % 2 == 0 && kWarpScratchWords % 2 == 0, "8-byte aligned entries");
    auto pc_entry_at = [&](int i) -> unsigned long long* {
        return reinterpret_cast<unsigned long long*>(s_stage + (i >> 7) * kWarpScratchWords + 2 * kStageCap +
                                                     2 * (i & (kPcPerWarp - 1)));
    };
    auto pc_entry = [&](uint32_t tag) -> unsigned long long* {
        return pc_entry_at((int)((tag * 0x9E3779B1u) >> kPcShift));
    };
    const bool use_pc = (long long)p.nstates * p.W < 0xFFFFFFF0ll && !(s_run.flags & RF_NO_CACHE);
    bool pc_dirty = true;
#endif
    // ---- level loop -----------------------------------------------------------
    int L = 0;
    int dir = DIR_PUSH;
    uint32_t qbsz = kBundle;  // bundle size the current queue was emitted with (the seed's: not merged)
    for (;;) {
        if (s_view.done) break;
        stamp(p, L, 0);
        dir = s_view.dir;
        const uint32_t* fcur = p.fb[L % 3];
        uint32_t* fnext = p.fb[(L + 1) % 3];

        if (dir == DIR_PUSH && s_view.plan) {
            // ---- plan epoch: emit F_L's row segments from its bitmap (after pull)
            const uint32_t bsz = s_view.nfront < (unsigned long long)nwarps * 8 ? 32u : (uint32_t)kBundle;
            qbsz = bsz;
            const Out o{&ctl->qc[(e + 1) % 3], p.seg[(e + 1) & 1], p.bun[(e + 1) & 1], &s_resv, bsz, 0.0f};
            if (cta0) reset_qc(ctl, (e + 2) % 3, threadIdx.x);
            unsigned long long nedge = 0;
#ifndef RPQ_PLAN_STATIC
            // chunks of 32 words (1,024 vertices) of every state with a
            // frontier and out-groups, dealt like pull tasks: a rotation over
            // the CTAs, the last quarter from a grid-wide counter (a fixed
            // stride left the warps on F's dense stretches far behind)
            if (threadIdx.x == 0) {
                int n = 0;
                for (int q = 0; q < p.nstates; ++q)
                    if (s_front[q] && S.gbeg[q + 1] != S.gbeg[q]) s_ptarget[n++] = q;
                s_nptarget = n;
                s_task = 0;
            }
            __syncthreads();
            const uint32_t nchunk = (uint32_t)((Wn + 31) >> 5), G32 = gridDim.x;
            const uint32_t nptask = (uint32_t)s_nptarget * nchunk;
            const uint32_t npown = nptask >= 16 * G32 ? (nptask / 4 * 3) / G32 * G32 : nptask;
            unsigned long long* plan_steal = &ctl->steal[e % 3][0];
            const FastDiv dchunk(nchunk), dG(G32);
            for (;;) {
                uint32_t t = 0;
                if (lane == 0) {
                    const uint32_t i = atomicAdd(&s_task, 1u);
                    uint32_t rot;
                    dG.div(blockIdx.x + i, &rot);
                    t = i * G32 + rot;
                    if (t >= npown && npown < nptask) t = npown + (uint32_t)atomicAdd(plan_steal, 1ull);
                }
                t = __shfl_sync(FULL, t, 0);
                if (t >= nptask) break;
                uint32_t chunk;
                const uint32_t tq = dchunk.div(t, &chunk);
                const int q = s_ptarget[tq];
                const uint32_t* row = fcur + (long long)q * p.W;
                {
                    const long long w0 = (long long)chunk * 32;
#else
            for (int q = 0; q < p.nstates; ++q) {
                if (!s_front[q] || S.gbeg[q + 1] == S.gbeg[q]) continue;
                const uint32_t* row = fcur + (long long)q * p.W;
                for (long long w0 = gwarp * 32; w0 < Wn; w0 += nwarps * 32) {
#endif
                    // a word per lane; their set bits dealt 32 per round to the
                    // lanes (prefix over popcounts), so every stage_add is full
                    const long long wi = w0 + lane;
                    const uint32_t bits = wi < Wn ? row[wi] : 0u;
                    const uint32_t cnt = __popc(bits);
                    const uint32_t incl = warp_incl_scan(cnt, lane);
                    const uint32_t excl = incl - cnt;
                    const uint32_t total = __shfl_sync(FULL, incl, 31);
                    for (uint32_t r0 = 0; r0 < total; r0 += 32) {
                        const uint32_t x = r0 + lane;
                        const bool valid = x < total;
                        const int j = warp_upper_lane(excl, valid ? x : 0u);
                        const uint32_t wb = __shfl_sync(FULL, bits, j);
                        const uint32_t eb = __shfl_sync(FULL, excl, j);
                        const int v = valid ? (int)((w0 + j) * 32 + __fns(wb, 0, (int)(x - eb) + 1)) : 0;
                        const uint32_t T = stage_add(p, S, o, stage, valid, q, v, lane);
                        if (lane == 0) nedge += T;
                    }
                }
            }
            {
                const uint32_t T = stage_flush(p, S, o, stage, lane);
                if (lane == 0) nedge += T;
            }
            __syncthreads();
            flush_counts(nullptr, o, nullptr, 0, nedge, s_red, s_state, 0);
            grid_barrier(ctl, ++e, s_run.bar_base);
            if (wid == 0) decide_plan(p, e, L, lane, &s_view, s_bpre);
            __syncthreads();
            stamp(p, L, 1);
            if (s_view.done) break;
        }

        // ---- expand epoch of level L -------------------------------------------
        // small queues: emit small bundles so the next level spreads over more
        // warps (threshold: 4 bundles per warp, measured a hair better than 1)
        const uint32_t bsz = (dir == DIR_PUSH ? s_bpre[kShards + 1] : s_view.nfront / 8) <
                                     (unsigned long long)nwarps * 4
                                 ? 32u : (uint32_t)kBundle;
#ifndef RPQ_GAIN_BUNDLES
#define RPQ_GAIN_BUNDLES 4
#endif
#ifdef RPQ_NO_BUNDLE_GAIN
        const float gain = 0.0f;
#else
        // bundles the successor level wants: 4 per warp; this level has
        // s_bpre[kShards + 1] bundles, each the source of about one pass
        const float gain = dir == DIR_PUSH && bsz < (uint32_t)kBundle
                               ? (float)s_bpre[kShards + 1] / (float)(nwarps * RPQ_GAIN_BUNDLES) : 0.0f;
#endif
        const Out o{&ctl->qc[(e + 1) % 3], p.seg[(e + 1) & 1], p.bun[(e + 1) & 1], &s_resv, bsz, gain};
        const uint32_t qbsz_next = bsz;
        if (threadIdx.x == 0) {
            s_task = 0;
            s_cut = 0;
            s_emitted = 0;
        }
        if (cta0) {
            reset_qc(ctl, (e + 2) % 3, threadIdx.x);
            FCnt* fz = &ctl->fc[(L + 2) % 3];
            for (int q = threadIdx.x; q < kMaxStates; q += blockDim.x) fz->state[q] = 0;
            if (threadIdx.x == 0) fz->nnew = 0;
        }
#ifdef RPQ_ZERO_IN_EXPAND
        if (!step_mode) {  // zero the bitmap level L+1 will write F_{L+2} into
            uint4* z4 = reinterpret_cast<uint4*>(p.fb[(L + 2) % 3]);
            for (long long i = gtid; i < nbits4; i += gthreads) z4[i] = make_uint4(0, 0, 0, 0);
        }
#endif
#ifndef RPQ_NO_CLAIM_CACHE
        if (dir == DIR_PUSH && pc_dirty) {  // (CTA-uniform)
            for (int i = threadIdx.x; i < kPcEntries; i += NT) *pc_entry_at(i) = 0ull;
            pc_dirty = false;
        }
        if (dir == DIR_PULL) pc_dirty = true;  // the pull scratch overwrites the cache
#endif
        __syncthreads();  // s_task
        unsigned int nnew = 0;  // this thread's discoveries this level (< 2^32)
        unsigned long long nedge = 0;
        // emit F_{L+1}'s queue now (at discovery) or later from F's bitmap
        // (a step-mode run stops after this level: nobody expands F_{L+1}'s queue)
        // progress reports: about 4 per CTA before the cut
        // (a power of two, the next one up: the per-drain progress test below is
        // two shifts, not two 64-bit divisions; rounded down, the finer reports
        // cost cfg3 1%)
        const int cut_shift =
            s_view.cut_edges > 0.0f
                ? 63 - __clzll((unsigned long long)(s_view.cut_edges / (4.0f * (float)gridDim.x)) + 1ull) + RPQ_CUT_SHIFT_UP : -1;
        const unsigned long long cut_chunk = cut_shift >= 0 ? 1ull << cut_shift : 0ull;
        const bool emit_inline = dir == DIR_PUSH && !s_view.defer && !step_mode &&
                                 (s_run.emit_mode == 0 ||
                                  (s_run.emit_mode == 2 && s_view.nfront < s_run.emit_inline_max));
        const int queued = emit_inline ? 1 : 0;
        if (dir == DIR_PUSH) {
            // ---- push: expand the bundles of F_L's queue (produced last epoch)
            const unsigned long long nb = s_bpre[kShards + 1];
            const uint2* bun = p.bun[e & 1];
            const uint2* seg = p.seg[e & 1];
            // CTA-major dealing: consecutive bundles (often one row) land on different SMs
            const unsigned long long step = (unsigned long long)gridDim.x * kWarps;
            // CTA c owns bundles c, c + G, c + 2G, ... (a strided sample of the
            // queue, so heavy rows spread over SMs); its warps take them one at a
            // time from a shared counter, so fast warps do more of them
            (void)step;
            // On long queues (>= 64 bundles per CTA) the last eighth (past
            // nb_own, a multiple of G) is dealt from one grid-wide counter
            // instead: CTAs that finish their share early take the tail
            // instead of idling at the barrier.  Short queues stay CTA-local
            // (a global round trip per bundle costs more than the imbalance).
            const unsigned long long G = gridDim.x;
            const unsigned long long nb_own = nb >= 64 * G ? (nb - nb / 8) / G * G : nb;
            unsigned long long* steal = &ctl->steal[e % 3][0];
            // software pipeline: the next bundle's descriptor is in flight while
            // this one is expanded (one dependent round trip less per bundle)
            // descriptor of bundle b (b warp-uniform): its shard is
            // #{i in [1, kShards] : s_bpre[i] <= b} (s_bpre is non-decreasing):
            // lanes test every 8th entry, then the 7 inside the block found
            auto load_bundle = [&](unsigned long long b) -> uint2 {
                const int ci = 8 * (lane + 1);
                const int c = __popc(__ballot_sync(FULL, ci <= kShards && s_bpre[ci] <= b));
                const int fi = 8 * c + 1 + lane;
                const int sh = 8 * c + __popc(__ballot_sync(FULL, lane < 7 && fi <= kShards && s_bpre[fi] <= b));
                return ld_queue(bun + (unsigned long long)sh * p.shard_buncap + (b - s_bpre[sh]), S.pf);
            };
            auto grab = [&](uint2* d) -> unsigned long long {
                unsigned long long b = 0;
                if (lane == 0) {
                    b = (unsigned long long)atomicAdd(&s_task, 1u) * gridDim.x + blockIdx.x;
                    if (b >= nb_own && nb_own < nb) b = nb_own + atomicAdd(steal, 1ull);
                }
                b = __shfl_sync(FULL, b, 0);
                if (b < nb) *d = load_bundle(b);
                return b;
            };
            // A large queue of small bundles (a level whose predecessor was
            // small emits 32-edge bundles; R-MAT grows 200x a level early on):
            // a warp takes 4 bundles per grab, one per edge slot of its lanes,
            // instead of leaving three slots of every lane idle.
            const bool merge4 = qbsz <= 32u && !s_view.qbig && nb >= (unsigned long long)nwarps * 8;
            uint2 bd_next = make_uint2(0u, kHoleY);
            unsigned long long bi_next = merge4 ? 0ull : grab(&bd_next);
            for (;;) {
                int w[kEdgesPerLane], gj[kEdgesPerLane];
                if (merge4) {
                    // the CTA's own indices i4 .. i4+3; those past nb_own (a
                    // suffix) are replaced by as many from the grid-wide tail
                    unsigned long long i4 = 0, t4 = 0;
                    int u0 = kEdgesPerLane;  // first slot past nb_own
                    if (lane == 0) {
                        i4 = atomicAdd(&s_task, (unsigned)kEdgesPerLane);
                        if (nb_own < nb)
                            for (int u = kEdgesPerLane - 1; u >= 0; --u)
                                if ((i4 + u) * G + blockIdx.x >= nb_own) u0 = u;
                        if (u0 < kEdgesPerLane) t4 = nb_own + atomicAdd(steal, (unsigned long long)(kEdgesPerLane - u0));
                    }
                    i4 = __shfl_sync(FULL, i4, 0);
                    t4 = __shfl_sync(FULL, t4, 0);
                    u0 = __shfl_sync(FULL, u0, 0);
                    // lane u < 4 loads descriptor u (all four in flight); the
                    // decode below broadcasts them one at a time
                    const uint2* myaddr = nullptr;
                    bool anyb = false;
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        unsigned long long b = (i4 + u) * G + blockIdx.x;
                        if (u >= u0) b = t4 + (u - u0);
                        if (b < nb) {
                            const int ci = 8 * (lane + 1);
                            const int c = __popc(__ballot_sync(FULL, ci <= kShards && s_bpre[ci] <= b));
                            const int fi = 8 * c + 1 + lane;
                            const int sh =
                                8 * c + __popc(__ballot_sync(FULL, lane < 7 && fi <= kShards && s_bpre[fi] <= b));
                            if (lane == u) myaddr = bun + (unsigned long long)sh * p.shard_buncap + (b - s_bpre[sh]);
                            anyb = true;
                        }
                    }
                    if (!anyb) break;
                    const uint2 mybd = myaddr ? ld_queue(myaddr, S.pf) : make_uint2(0u, kHoleY);
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        const uint2 bdu = make_uint2(__shfl_sync(FULL, mybd.x, u), __shfl_sync(FULL, mybd.y, u));
                        gj[u] = -1;
                        w[u] = 0;
                        if (bdu.y == kHoleY) continue;  // warp-uniform
                        const uint32_t cu = (bdu.y & 127u) + 1;
                        if (bdu.y & kInline) {
                            const int g = (int)((bdu.y >> 7) & 0xFFu);
                            const bool okc = (uint32_t)lane < cu &&
                                             RPQ_CHECK(bdu.x + lane < p.slot_nnz[S.gslot[g] % p.nslots], RPQ_F_SSR);
                            gj[u] = okc ? g : -1;
                            w[u] = okc ? ld_stream_i32(S.slots[S.gslot[g]].col + bdu.x + lane, S.pf) : 0;
                        } else {
                            const uint32_t off = (bdu.y >> 7) & 0xFFFFFFu;
                            uint32_t my_start = 0, my_len = 0, my_grp = 0;
                            if ((unsigned long long)bdu.x + lane < p.seg_alloc) {
                                const uint2 sg = ld_queue(seg + bdu.x + lane, S.pf);
                                my_start = sg.x;
                                my_len = sg.y >> 8;
                                my_grp = sg.y & 0xFFu;
                            }
                            if (lane == 0) {
                                my_start += off;
                                my_len -= off;
                            }
                            const uint32_t incl = warp_incl_scan(my_len, lane);
                            const uint32_t excl = incl - my_len;
                            const bool active = (uint32_t)lane < cu;
                            const int j = warp_upper_lane(excl, active ? (uint32_t)lane : 0u);
                            const uint32_t sj = __shfl_sync(FULL, my_start, j);
                            const uint32_t exj = __shfl_sync(FULL, excl, j);
                            const int g = (int)__shfl_sync(FULL, my_grp, j);
                            const bool okc = active && RPQ_CHECK(g >= 0 && g < p.ngroups &&
                                                                     sj + ((uint32_t)lane - exj) <
                                                                         p.slot_nnz[S.gslot[g] % p.nslots],
                                                                 RPQ_F_SSR);
                            gj[u] = okc ? g : -1;
                            w[u] = okc ? ld_stream_i32(S.slots[S.gslot[g]].col + sj + ((uint32_t)lane - exj), S.pf)
                                       : 0;
                        }
                    }
                } else {
                const unsigned long long bi = bi_next;
                if (bi >= nb) break;
                const uint2 bd = bd_next;
                bi_next = grab(&bd_next);
                if (bd.y == kHoleY) continue;
                const uint32_t cnt = (bd.y & 127u) + 1;
                if (bd.y & kInline) {
                    // one row: columns bd.x .. bd.x + cnt - 1
                    const int g = (int)((bd.y >> 7) & 0xFFu);
                    const int32_t* col = S.slots[S.gslot[g]].col + bd.x;
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        const uint32_t ed = (uint32_t)(lane + 32 * u);
                        const bool okc = ed < cnt && RPQ_CHECK(bd.x + ed < p.slot_nnz[S.gslot[g] % p.nslots], RPQ_F_SSR);
                        gj[u] = okc ? g : -1;
                        w[u] = okc ? ld_stream_i32(col + ed, S.pf) : 0;
                    }
                } else {
                    const uint32_t s0 = bd.x;
                    const uint32_t off = (bd.y >> 7) & 0xFFFFFFu;
                    uint32_t my_start = 0, my_len = 0, my_grp = 0;
                    if ((unsigned long long)s0 + lane < p.seg_alloc) {
                        const uint2 sg = ld_queue(seg + s0 + lane, S.pf);
                        my_start = sg.x;
                        my_len = sg.y >> 8;
                        my_grp = sg.y & 0xFFu;
                    }
                    if (lane == 0) {
                        my_start += off;
                        my_len -= off;
                    }
                    const uint32_t incl = warp_incl_scan(my_len, lane);
                    const uint32_t excl = incl - my_len;
                    // edges lane, lane+32, ...: locate, then issue all column loads
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        const uint32_t ed = (uint32_t)(lane + 32 * u);
                        const bool active = ed < cnt;
                        const int j = warp_upper_lane(excl, active ? ed : 0u);
                        const uint32_t sj = __shfl_sync(FULL, my_start, j);
                        const uint32_t exj = __shfl_sync(FULL, excl, j);
                        const int g = (int)__shfl_sync(FULL, my_grp, j);
                        const bool okc = active && RPQ_CHECK(g >= 0 && g < p.ngroups &&
                                                                 sj + (ed - exj) < p.slot_nnz[S.gslot[g] % p.nslots],
                                                             RPQ_F_SSR);
                        gj[u] = okc ? g : -1;
                        w[u] = okc ? ld_stream_i32(S.slots[S.gslot[g]].col + sj + (ed - exj), S.pf) : 0;
                    }
                }
                }  // single bundle
                // probe P for every target, then claim with atomicOr
                for (int k = 0; k < p.maxT; ++k) {
                    uint32_t old[kEdgesPerLane];
                    int q2[kEdgesPerLane];
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        q2[u] = -1;
                        old[u] = 0xFFFFFFFFu;
                        if (gj[u] >= 0) {
                            const int t0 = S.toff[gj[u]];
                            if (t0 + k < S.toff[gj[u] + 1]) {
                                q2[u] = S.targets[t0 + k];
                                if (!(s_run.flags & RF_NO_PROBE))
                                    old[u] = ld_bits(p.visited + (long long)q2[u] * p.W + (w[u] >> 5), S.pl);
                                else
                                    old[u] = 0u;
#ifndef RPQ_NO_CLAIM_CACHE
                                if (use_pc) {
                                    const uint32_t tag = (uint32_t)((long long)q2[u] * p.W + (w[u] >> 5)) + 1u;
                                    const unsigned long long ent = *pc_entry(tag);
                                    if ((uint32_t)(ent >> 32) == tag) old[u] |= (uint32_t)ent;
                                }
#endif
                            }
                        }
                    }
                    unsigned claimed = 0;  // edge slots whose claim went to global memory
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        const uint32_t bit = 1u << (w[u] & 31);
                        if (q2[u] >= 0 && !RPQ_CHECK(q2[u] < p.nstates && w[u] >= 0 && w[u] < p.nv, RPQ_F_SSR))
                            q2[u] = -1;
                        if (q2[u] >= 0 && !(old[u] & bit)) {
                            const long long off2 = (long long)q2[u] * p.W + (w[u] >> 5);
                            old[u] = or_bits(p.visited + off2, bit, S.pl);
                            claimed |= 1u << u;
#ifdef RPQ_PUSH_SERIAL_CLAIMS
                            if (!(old[u] & bit)) red_or_bits(fnext + off2, bit, S.pl);
#endif
                        } else {
                            old[u] = 0xFFFFFFFFu;
                        }
                    }
#ifndef RPQ_PUSH_SERIAL_CLAIMS
                    // the F bits in a second pass: the claims above are volatile
                    // asm statements, kept in program order, so a RED between
                    // two of them would wait for the first claim's return before
                    // the second is issued (four serial L2 round trips per bundle)
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        const uint32_t bit = 1u << (w[u] & 31);
                        if (q2[u] >= 0 && !(old[u] & bit))
                            red_or_bits(fnext + (long long)q2[u] * p.W + (w[u] >> 5), bit, S.pl);
#ifndef RPQ_NO_CLAIM_CACHE
                        // what the claim returned is now known of the whole word
                        if (use_pc && ((claimed >> u) & 1u)) {
                            const uint32_t tag = (uint32_t)((long long)q2[u] * p.W + (w[u] >> 5)) + 1u;
                            *pc_entry(tag) = ((unsigned long long)tag << 32) | (old[u] | bit);
                        }
#endif
                    }
#endif
                    (void)claimed;
                    const bool emit_now = emit_inline && !*(volatile int*)&s_cut;
#pragma unroll
                    for (int u = 0; u < kEdgesPerLane; ++u) {
                        const bool fresh = q2[u] >= 0 && !(old[u] & (1u << (w[u] & 31)));
                        nnew += fresh ? 1 : 0;
#ifdef RPQ_PUSH_SERIAL_CLAIMS
                        if (fresh) atomicAdd(&s_state[q2[u]], 1u);
#else
                        // per-state counts: one shared atomic per distinct state among the
                        // fresh lanes (32 lanes on one shared address serialize)
                        unsigned fmk = __ballot_sync(FULL, fresh);
                        while (fmk) {
                            const int ld = __ffs(fmk) - 1;
                            const int qL = __shfl_sync(FULL, q2[u], ld);
                            const unsigned grp = __ballot_sync(FULL, fresh && q2[u] == qL);
                            if (lane == ld) atomicAdd(&s_state[qL], (unsigned)__popc(grp));
                            fmk &= ~grp;
                        }
#endif
                        if (emit_now) stage_put(stage, fresh, q2[u], w[u], lane);
                    }
                    if (emit_now) {
                        const uint32_t T = stage_drain(p, S, o, stage, lane);
                        if (lane == 0) {
                            nedge += T;
                            // report progress in chunks; past the cut, stop emitting
                            if (cut_chunk && T) {
                                const unsigned long long old_e = atomicAdd(&s_emitted, (unsigned long long)T);
                                const unsigned long long c0 = old_e >> cut_shift, c1 = (old_e + T) >> cut_shift;
                                if (c1 != c0) {
                                    const unsigned long long g =
                                        atomicAdd(&o.qc->emit_progress, (c1 - c0) << cut_shift) + ((c1 - c0) << cut_shift);
                                    if ((float)g >= s_view.cut_edges || ldcg(&o.qc->emit_cut)) {
                                        o.qc->emit_cut = 1u;
                                        s_cut = 1;
                                    }
                                }
                            }
                        }
                        if (__shfl_sync(FULL, *(volatile int*)&s_cut, 0)) stage.n = 0;  // drop what is staged
                    }
                }
            }
            if (emit_inline && !*(volatile int*)&s_cut) {
                const uint32_t T = stage_flush(p, S, o, stage, lane);
                if (lane == 0) nedge += T;
            }
            stage.n = 0;
        } else {
            // ---- pull: unvisited (q', w) scan A_s^T row w for a member of F_L[q]
            if (S.run->count_te)  // diagnostics: F_L's push-model edges (per-level roofline)
                nedge += frontier_edges(p, S, fcur, gtid, gthreads, Wn);
            if (threadIdx.x == 0) {
                int n = 0;
                int multi = 0;
                for (int q2 = 0; q2 < p.nstates; ++q2) {
                    int any = 0, kf = 0;
                    for (int k = S.ibeg[q2]; k < S.ibeg[q2 + 1]; ++k)
                        if (s_front[S.isrc[k]] != 0 && any++ == 0) kf = k;
                    if (any) {
                        s_pk[n] = any == 1 ? kf : -1;  // the only active in-transition, or -1: several
                        s_ptarget[n++] = q2;
                    }
                    multi |= any > 1;
                }
                s_nptarget = n;
                s_pmulti = multi;
            }
            __syncthreads();
            // targets: the owned word range (vertex-partitioned step), else all
            const long long pw0 = s_run.own_w1 > s_run.own_w0 ? s_run.own_w0 : 0;
            const long long pw1 = s_run.own_w1 > s_run.own_w0 ? min((long long)s_run.own_w1, Wn) : Wn;
            // A dense frontier (> 22% of |V| pairs) usually answers at the first
            // in-edge: a round probes one per candidate first, on a sparse one two.
            // Only in the large-state-space instance (measured on cfg3 and cfg5).
            const bool one_inline = NT == kThreadsLarge && (float)s_view.nfront > 0.22f * (float)p.nv;
            unsigned long long* pull_steal = &ctl->steal[e % 3][8];
            uint32_t* scratch = reinterpret_cast<uint32_t*>(s_stage) + (size_t)wid * kWarpScratchWords;
            const int first = one_inline ? 1 : kPullInline;
            // large graphs (>= 16 words of vertices per warp of the grid): 32-word
            // tasks; smaller ones: 8-word tasks, so that every warp has some
            const bool big = pw1 - pw0 >= (long long)nwarps * 16;
            if (big && !s_pmulti)
                pull_tasks_ne1(p, S, fcur, fnext, pw0, pw1, lane, &s_task, s_nptarget, s_ptarget, s_pk, s_state,
                               nnew, pull_steal, scratch, first);
            else if (big)
                pull_tasks_ne<RPQ_NE_TW>(p, S, fcur, fnext, pw0, pw1, lane, &s_task, s_nptarget, s_ptarget, s_pk, s_front,
                                  s_state, nnew, pull_steal, scratch, first);
            else
                pull_tasks_ne<8>(p, S, fcur, fnext, pw0, pw1, lane, &s_task, s_nptarget, s_ptarget, s_pk, s_front,
                                 s_state, nnew, pull_steal, scratch, first);
        }
        if (p.trace && lane == 0) atomicMax(&s_wend, globaltimer());  // this warp's work done
        __syncthreads();
        if (p.trace && L < p.trace_levels && threadIdx.x == 0) {
            p.trace[((long long)L * gridDim.x + blockIdx.x) * 8 + 2] = s_wend - ctl->t0;
            s_wend = 0;
        }
        if (threadIdx.x == 0 && L < 64) atomicMax(&ctl->work_ns[L], globaltimer() - ctl->t0);
        flush_counts(&ctl->fc[(L + 1) % 3].nnew, o, ctl->fc[(L + 1) % 3].state, nnew, nedge, s_red,
                     s_state, p.nstates);
        stamp(p, L, 4);
        grid_barrier(ctl, ++e, s_run.bar_base);
        stamp(p, L, 3);
        if (cta0 && threadIdx.x == 0 && L < 64) ctl->bar_ns[L] = globaltimer() - ctl->t0;
        ++L;
        qbsz = qbsz_next;
        if (step_mode) {
            if (threadIdx.x == 0) {
                s_view.done = 1;
                s_view.status = 1;  // (no answer projection in step mode)
                if (cta0) {
                    ctl->iterations = 1;
                    // no decision follows the step: record a barrier abort here
                    if (ldcg(&ctl->abort)) ctl->status = ST_DEADLOCK;
                }
            }
            __syncthreads();
            break;
        }
        if (wid == 0) decide_level(p, S, e, L, queued, dir, lane, &s_view, s_bpre, s_sv, s_front);
        else zero_next(L);
        __syncthreads();
    }

    // ---- epilogue: answer = OR of P's rows at final states (engine.py:112-114)
    // The answer bitmap only: the uint8[|V|] vector is expanded from it on
    // demand (reach_bytes_kernel, rpq_query_copy_reach), not on every run.
    stamp(p, L, 1);  // diagnostics: epilogue entered (row L's slots 1-4 are free: the loop broke before its stamps)
    int wrote_host = 0;  // this thread stored answer words to pinned host memory (over PCIe)
    if (s_view.status == 0) {
        unsigned long long cnt = 0, nzw = 0;
        uint32_t* const hb = s_run.out_bits ? s_run.out_bits : p.host_bits;
        const bool maybe_list = hb && s_run.out_list;
        for (long long i = gtid; i < Wn; i += gthreads) {
            uint32_t acc = 0;
            for (int f = 0; f < p.nfinals; ++f) acc |= __ldcg(p.visited + (long long)S.finals[f] * p.W + i);
            cnt += __popc(acc);
            nzw += acc != 0u;
            p.reach_bits[i] = acc;
            if (hb && !maybe_list) {
                hb[i] = acc;  // coalesced: 128 B per warp over PCIe
                wrote_host = 1;
            }
        }
        stamp(p, L, 2);  // diagnostics: projection written
        if (maybe_list) {
            // the host gets whichever is smaller: the bitmap, or the nonzero
            // words as (index, word) pairs -- an empty answer moves no bytes
            nzw = warp_sum_u64(nzw);
            if (lane == 0 && nzw) atomicAdd(&ctl->ans_words, nzw);
            grid_barrier(ctl, ++e, s_run.bar_base);
            const unsigned long long nz = ldcg(&ctl->ans_words);
            const bool list = 2 * nz < (unsigned long long)Wn;
            if (list) {
                for (long long i0 = gwarp * 32; i0 < Wn; i0 += nwarps * 32) {
                    const long long i = i0 + lane;
                    const uint32_t acc = i < Wn ? __ldcg(p.reach_bits + i) : 0u;
                    const unsigned m = __ballot_sync(FULL, acc != 0u);
                    if (!m) continue;
                    unsigned long long base = 0;
                    if (lane == 0) base = atomicAdd(&ctl->ans_cursor, (unsigned long long)__popc(m));
                    base = __shfl_sync(FULL, base, 0);
                    if (acc) {
                        const unsigned long long pos = base + __popc(m & lanemask_lt());
                        if (RPQ_CHECK(2 * pos + 1 < (unsigned long long)Wn, RPQ_F_SSR)) {
                            hb[2 * pos] = (uint32_t)i;
                            hb[2 * pos + 1] = acc;
                            wrote_host = 1;
                        }
                    }
                }
            } else {
                for (long long i = gtid; i < Wn; i += gthreads) {
                    hb[i] = __ldcg(p.reach_bits + i);
                    wrote_host = 1;
                }
            }
            if (cta0 && threadIdx.x == 0) ctl->ans_list = list ? 1 : 0;
            stamp(p, L, 3);  // diagnostics: answer transport written
        }
        // exact push-model TE = sum over (q, v) in P of q's group out-degrees x targets
        unsigned long long te = 0;
        if (S.run->count_te) {
            for (int q = 0; q < p.nstates; ++q) {
                if (S.gbeg[q + 1] == S.gbeg[q]) continue;
                for (long long i = gtid; i < Wn; i += gthreads) {
                    uint32_t bits = __ldcg(p.visited + (long long)q * p.W + i);
                    while (bits) {
                        const int v = (int)(i * 32 + __ffs(bits) - 1);
                        bits &= bits - 1;
                        for (int g = S.gbeg[q]; g < S.gbeg[q + 1]; ++g) {
                            const Slot sl = S.slots[S.gslot[g]];
                            te += (unsigned long long)(__ldg(sl.rowptr + v + 1) - __ldg(sl.rowptr + v)) *
                                  (unsigned long long)(S.toff[g + 1] - S.toff[g]);
                        }
                    }
                }
            }
        }
        // one atomic per CTA, not per warp (thousands on one address serialize)
        cnt = warp_sum_u64(cnt);
        te = warp_sum_u64(te);
        if (lane == 0) {
            s_red[2 * wid] = cnt;
            s_red[2 * wid + 1] = te;
        }
        __syncthreads();
        if (wid == 0) {
            cnt = warp_sum_u64(lane < kWarps ? s_red[2 * lane] : 0ull);
            te = warp_sum_u64(lane < kWarps ? s_red[2 * lane + 1] : 0ull);  // (kWarps <= 32)
            if (lane == 0 && cnt) atomicAdd(&ctl->reach_count, cnt);
            if (lane == 0 && te) atomicAdd(&ctl->te_exact, te);
        }
    }

    // The last CTA out: every CTA is past its last barrier, so it resets the
    // barrier counter for the next run on this query (runs on one query are
    // stream-ordered: no host round trip for the next run's barrier base);
    // zero-copy results: it copies the results prefix (everything before the
    // working counters) to pinned host memory; step mode: a failed step
    // latches its status for rpq_query_step_end.
    stamp(p, L, 4);  // diagnostics: epilogue done
    {
        __shared__ int s_last;
        // A system-scope fence costs ~20 us when all 148 CTAs issue one at
        // once (they serialize): only CTAs whose threads stored answer words
        // over PCIe pay it; everyone else orders its counters at GPU scope.
        wrote_host = __syncthreads_or(wrote_host);
        if (threadIdx.x == 0) {
            // this CTA's counter updates (and its answer words over PCIe, if
            // it wrote any) are visible before it counts itself out
            if (wrote_host) __threadfence_system();
            else __threadfence();
            s_last = atomicAdd(&ctl->exits, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (p.host_ctl && wid == 0) {
                // one warp copies the results prefix (~3 KB): one system fence
                // per writing warp, so as few writing warps as possible
                if (lane == 0) ctl->t_end = globaltimer();
                __syncwarp();
                constexpr int nw = (int)(offsetof(Ctl, qc) / 4);
                constexpr int iseq = (int)(offsetof(Ctl, done_seq) / 4);
                const unsigned* src = reinterpret_cast<const unsigned*>(ctl);
                unsigned* dst = reinterpret_cast<unsigned*>(p.host_ctl);
                for (int i = lane; i < nw; i += 32)
                    if (i != iseq) dst[i] = i == 0 ? 0u : __ldcg(src + i);
                __threadfence_system();
                __syncwarp();
                // the completion flag goes last: a host that sees it sees the
                // results prefix and every CTA's answer words
                if (lane == 0) {
                    *(volatile unsigned*)(dst + iseq) = s_run.run_seq;
                    __threadfence_system();
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                if (step_mode && p.step_acc) {
                    const int st = ldcg(&ctl->status);
                    if (st != 0) atomicCAS(p.step_acc + 1, 0u, (unsigned)st);
                }
                ctl->bar = 0;
                ctl->exits = 0;
            }
        }
    }
}

// Non-empty rows of a CSR (the defer predictor's mean degree), one atomic per warp.
__global__ void count_nonempty_kernel(const uint32_t* __restrict__ rowptr, long long nv,
                                      unsigned long long* __restrict__ out) {
    unsigned c = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x)
        c += rowptr[i + 1] > rowptr[i];
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// Non-empty-row bitmap of a CSR (Slot::ne): bit v of word v / 32 set when row v
// has edges; `words` words (bits past nv clear).  One ballot per 32 rows.
__global__ void nonempty_bitmap_kernel(const uint32_t* __restrict__ rowptr, long long nv, uint32_t* __restrict__ out,
                                       long long words) {
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < words * 32;
         v += (long long)gridDim.x * blockDim.x) {  // (warp-uniform trip count: bounds are multiples of 32)
        const bool ne = v < nv && rowptr[v + 1] > rowptr[v];
        const unsigned m = __ballot_sync(0xFFFFFFFFu, ne);
        if ((threadIdx.x & 31) == 0) out[v >> 5] = m;
    }
}

// uint8[nv] answer vector from the answer bitmap (bit v%32 of word v/32):
// 32 bytes per word, two 16-byte stores (the buffer holds W * 32 + 32 bytes).
__global__ void reach_bytes_kernel(const uint32_t* __restrict__ bits, uint8_t* __restrict__ out, long long words) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += (long long)gridDim.x * blockDim.x) {
        const uint32_t acc = bits[i];
        uint32_t b4[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t nib = (acc >> (4 * k)) & 0xFu;
            b4[k] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
        }
        uint4* dst = reinterpret_cast<uint4*>(out + i * 32);
        dst[0] = make_uint4(b4[0], b4[1], b4[2], b4[3]);
        dst[1] = make_uint4(b4[4], b4[5], b4[6], b4[7]);
    }
}

// Upload validation of a host CSR (the reference's SparseBoolMatrix checks its
// own structure, sparse_bool.py:60-73; a duck-typed graph may not): indptr
// non-decreasing within [0, nnz], columns within [0, nv).  *bad = 1 on failure.
template <typename I>
__global__ void validate_csr_kernel(const I* __restrict__ v, long long n, long long lo, long long hi, int monotone,
                                    int* __restrict__ bad) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long x = (long long)v[i];
        if (x < lo || x >= hi || (monotone && i + 1 < n && (long long)v[i + 1] < x)) *bad = 1;
    }
}

// int64 -> narrow copy used at upload (sparse_bool.py keeps int64 everywhere)
template <typename In, typename Out>
__global__ void narrow_kernel(const In* __restrict__ in, Out* __restrict__ out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (Out)in[i];
}

}  // namespace rpqk
