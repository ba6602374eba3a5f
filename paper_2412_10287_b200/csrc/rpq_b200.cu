// rpq_b200.cu -- B200-native (sm_100a) single-source 2-RPQ frontier BFS.
//
// Replaces the reference's per-level frontier step
//   M <- (sum_a (N^a)^T x M x G^a) <not P>;  P <- P + M      (Alg. 1;
//   rpq/engine.py:117-124 _step_sum, :146-171 eval_ssr_masked)
// with one persistent cooperative kernel per query.  See DESIGN.md for the
// layout; in short:
//
//   graph     per label and direction: uint32 row pointers + int32 columns
//             (forward[l] and backward[l] = transpose, graph_store.py:51-52)
//   automaton (state, slot) "groups": slot = (label, inverted) adjacency,
//             targets = the states reached on that symbol (transition matrix row)
//   P         |Q| bitmaps of |V| bits (visited), L2-resident for the configs
//   frontier  a work queue of row SEGMENTS (one per discovered (state, vertex)
//             pair and out-group with non-empty adjacency row) cut into
//             BUNDLES of <= 64 edges; producers emit the next level's
//             segments the moment they discover a pair, so each BFS level is
//             exactly one pass over the queue and one grid barrier.
//
// mask_complement + or_sum of the reference (engine.py:159, :165) are fused
// into the expansion: the first thread whose atomicOr sets a (state, vertex)
// bit owns the discovery.  np.unique's dedup (sparse_bool.py:250) is implicit
// in the bitmap.  The answer projection F x P (engine.py:112-114) is the
// kernel's epilogue.
#include "rpq_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    return fail(e == cudaErrorMemoryAllocation ? RPQ_ENOMEM : RPQ_ECUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                      \
    do {                                                    \
        cudaError_t e_ = (expr);                            \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
    } while (0)

constexpr int kThreads = 256;        // 8 warps per CTA
constexpr int kMinBlocks = 3;       // CTAs per SM the register budget is sized for
constexpr int kBundle = 32;          // edges per bundle (one per lane; <= 32 segments)
constexpr int kShards = 64;          // queue shards (+1 overflow shard), by CTA id
constexpr int kMaxStates = 1024;
constexpr int kMaxGroups = 256;      // group id is 8 bits in a segment
constexpr int kMaxSlots = 256;
constexpr uint32_t kSegLenMax = (1u << 24) - 1;
constexpr unsigned FULL = 0xffffffffu;

constexpr int ST_OVERFLOW = 100;     // internal: queue capacity exceeded
constexpr int ST_DEADLOCK = 101;     // internal: barrier spin limit hit

struct Slot {
    const uint32_t* rowptr;
    const int32_t* col;
};

struct Ctl {
    unsigned int bar_count;
    unsigned int bar_gen;
    int status;
    int done;
    int iterations;
    int levels;
    int overflow;
    int pad0;
    unsigned long long t0;
    // per queue buffer and shard: (segments << 32) | bundles
    unsigned long long shard_cnt[2][kShards + 1];
    unsigned long long new_cnt[2];
    unsigned long long edge_cnt[2];
    unsigned long long seg_total[2];
    unsigned long long te;
    unsigned long long segments;
    unsigned long long pairs;
    unsigned long long reach_count;
    long long level_new[RPQ_STATS_LEVELS];
    long long level_edges[RPQ_STATS_LEVELS];
};

// Kernel parameters.  Tables are small int32 arrays staged into shared memory:
//   gbeg[nstates+1]  groups of state q are [gbeg[q], gbeg[q+1])
//   gslot[ngroups]   slot of each group
//   toff[ngroups+1]  targets of group g are targets[toff[g] .. toff[g+1])
//   targets[ntargets]
//   starts[nstarts], finals[nfinals]
struct Params {
    const int32_t* tables;
    const Slot* slots;
    uint32_t* visited;
    uint2* seg[2];
    uint2* bun[2];
    Ctl* ctl;
    uint8_t* reach;
    unsigned long long shard_segcap;   // per regular shard
    unsigned long long shard_buncap;
    unsigned long long ovf_segcap;     // overflow shard (index kShards)
    unsigned long long ovf_buncap;
    unsigned long long seg_alloc;      // entries allocated per buffer
    unsigned long long bun_alloc;
    unsigned long long budget_ns;
    long long W;  // uint32 words per visited row (multiple of 4)
    int nv;
    int nstates, ngroups, nslots, ntargets, nstarts, nfinals;
    int maxT;  // max targets per group
    int source;
    int table_ints;
};

struct Smem {
    const int32_t* gbeg;
    const int32_t* gslot;
    const int32_t* toff;
    const int32_t* targets;
    const int32_t* starts;
    const int32_t* finals;
    const Slot* slots;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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
template <typename T>
__device__ __forceinline__ T ld_volatile(const T* p) {
    return *reinterpret_cast<const volatile T*>(p);
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

// Grid barrier for a cooperative launch.  The last CTA to arrive runs
// `serial` (one thread) before releasing everyone: per-level bookkeeping is
// thereby ordered after all CTAs' work and before any CTA's next level.
template <class F>
__device__ __forceinline__ void grid_sync(Ctl* ctl, F serial) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nblocks = gridDim.x;
        unsigned gen = ld_acquire_u32(&ctl->bar_gen);
        __threadfence();
        unsigned arrived = atomicAdd(&ctl->bar_count, 1u);
        if (arrived == nblocks - 1) {
            __threadfence();
            serial();
            ctl->bar_count = 0;
            __threadfence();
            st_release_u32(&ctl->bar_gen, gen + 1);
        } else {
            unsigned long long ts = 0;
            unsigned spins = 0;
            while (ld_acquire_u32(&ctl->bar_gen) == gen) {
                __nanosleep(32);
                if ((++spins & 4095u) == 0) {
                    unsigned long long now = globaltimer();
                    if (ts == 0) ts = now;
                    else if (now - ts > 20000000000ull) {  // 20 s: cannot happen co-resident
                        atomicExch(&ctl->status, ST_DEADLOCK);
                        atomicExch(&ctl->done, 1);
                        break;
                    }
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
}

constexpr uint32_t kHoleBundle = 0xFFFFFFFFu;  // bundle slot left empty by a spill

// Shard-local reservation of `nseg` segments and `nb` bundles in queue buffer
// `b` (called by one lane).  Regular shards are indexed by CTA; a reservation
// that does not fit spills to the overflow shard, and the part of its bundle
// range that lies inside the regular shard, [*hole_lo, *hole_hi), must be
// filled with kHoleBundle by the caller.  Returns false when even the
// overflow shard is full.
__device__ __forceinline__ bool reserve(const Params& p, int b, uint32_t nseg, uint32_t nb,
                                        unsigned long long* seg_idx, unsigned long long* bun_idx,
                                        unsigned long long* hole_lo, unsigned long long* hole_hi) {
    Ctl* ctl = p.ctl;
    const int shard = blockIdx.x % kShards;
    const unsigned long long inc = ((unsigned long long)nseg << 32) | nb;
    unsigned long long old = atomicAdd(&ctl->shard_cnt[b][shard], inc);
    unsigned long long s_loc = old >> 32, b_loc = old & 0xFFFFFFFFull;
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
    old = atomicAdd(&ctl->shard_cnt[b][kShards], inc);
    s_loc = old >> 32;
    b_loc = old & 0xFFFFFFFFull;
    if (s_loc + nseg <= p.ovf_segcap && b_loc + nb <= p.ovf_buncap) {
        *seg_idx = (unsigned long long)kShards * p.shard_segcap + s_loc;
        *bun_idx = (unsigned long long)kShards * p.shard_buncap + b_loc;
        return true;
    }
    return false;
}

// Warp-cooperative emission of the row segments of newly discovered
// (state q, vertex w) pairs (one candidate per lane) into queue buffer `b`.
// Returns the number of edges emitted (valid in every lane).
__device__ __forceinline__ uint32_t emit_pairs(const Params& p, const Smem& S, int b, bool valid,
                                            int q, int w, int lane) {
    const unsigned vmask = __ballot_sync(FULL, valid);
    if (vmask == 0) return 0;
    const int ng = valid ? (S.gbeg[q + 1] - S.gbeg[q]) : 0;
    int maxng = ng;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) maxng = max(maxng, __shfl_xor_sync(FULL, maxng, d));
    uint2* seg = p.seg[b];
    uint2* bun = p.bun[b];
    uint32_t emitted = 0;
    for (int k = 0; k < maxng; ++k) {
        uint32_t lo = 0, deg = 0;
        int g = 0;
        if (k < ng) {
            g = S.gbeg[q] + k;
            const Slot sl = S.slots[S.gslot[g]];
            lo = __ldg(sl.rowptr + w);
            deg = __ldg(sl.rowptr + w + 1) - lo;
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
            const uint32_t nb = (T + kBundle - 1) / kBundle;
            unsigned long long sbase = 0, bbase = 0, hlo = 0, hhi = 0;
            int ok = 1;
            if (lane == 0) ok = reserve(p, b, nseg, nb, &sbase, &bbase, &hlo, &hhi) ? 1 : 0;
            ok = __shfl_sync(FULL, ok, 0);
            hlo = __shfl_sync(FULL, hlo, 0);
            hhi = __shfl_sync(FULL, hhi, 0);
            for (unsigned long long h = hlo + lane; h < hhi; h += 32) bun[h] = make_uint2(kHoleBundle, 0);
            if (!ok) {
                if (lane == 0) atomicExch(&p.ctl->overflow, 1);
                return emitted;
            }
            sbase = __shfl_sync(FULL, sbase, 0);
            bbase = __shfl_sync(FULL, bbase, 0);
            if (hs) seg[sbase + rank] = make_uint2(lo, (take << 8) | (uint32_t)g);
            for (uint32_t kb0 = 0; kb0 < nb; kb0 += 32) {
                const uint32_t kb = kb0 + lane;
                const uint32_t pos = kb * kBundle;
                const int j = warp_upper_lane(excl, min(pos, T - 1));
                const uint32_t exj = __shfl_sync(FULL, excl, j);
                const int rj = __shfl_sync(FULL, rank, j);
                if (kb < nb) {
                    const uint32_t cnt = min((uint32_t)kBundle, T - pos);
                    bun[bbase + kb] = make_uint2((uint32_t)(sbase + rj), (pos - exj) | ((cnt - 1) << 24));
                }
            }
            emitted += T;
            lo += take;
            deg -= take;
        }
    }
    return emitted;
}

// Per-CTA flush of the level's statistics (one atomic per CTA and counter).
__device__ __forceinline__ void flush_counts(Ctl* ctl, int b, unsigned long long nnew,
                                             unsigned long long nedge, unsigned long long* red) {
    // red: 2 * (kThreads/32) shared slots
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        nnew += __shfl_xor_sync(FULL, nnew, d);
        nedge += __shfl_xor_sync(FULL, nedge, d);
    }
    if (lane == 0) {
        red[2 * wid] = nnew;
        red[2 * wid + 1] = nedge;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, c = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            a += red[2 * i];
            c += red[2 * i + 1];
        }
        if (a) atomicAdd(&ctl->new_cnt[b], a);
        if (c) atomicAdd(&ctl->edge_cnt[b], c);
    }
    __syncthreads();
}

// Bookkeeping after frontier F_L (queue buffer L&1) has been produced.
// Mirrors the masked loop exactly (engine.py:156-160): the loop runs while the
// frontier is non-empty, checks the deadline first, then steps.
__device__ __forceinline__ void level_bookkeeping(const Params& p, int L) {
    Ctl* ctl = p.ctl;
    const int b = L & 1;
    const unsigned long long nnew = ld_volatile(&ctl->new_cnt[b]);
    const unsigned long long nedge = ld_volatile(&ctl->edge_cnt[b]);
    unsigned long long nbun = 0, nseg = 0;
    for (int s = 0; s <= kShards; ++s) {
        const unsigned long long c = ld_volatile(&ctl->shard_cnt[b][s]);
        const unsigned long long bc = c & 0xFFFFFFFFull, sc = c >> 32;
        const unsigned long long bcap = s < kShards ? p.shard_buncap : p.ovf_buncap;
        const unsigned long long scap = s < kShards ? p.shard_segcap : p.ovf_segcap;
        nbun += bc < bcap ? bc : bcap;
        nseg += sc < scap ? sc : scap;
    }
    ctl->pairs += nnew;
    if (L < RPQ_STATS_LEVELS) ctl->level_new[L] = (long long)nnew;
    if (ld_volatile(&ctl->overflow)) {
        ctl->status = ST_OVERFLOW;
        ctl->iterations = L;
        ctl->done = 1;
    } else if (ld_volatile(&ctl->status) != 0) {
        ctl->done = 1;
    } else if (nnew == 0) {
        ctl->iterations = L;
        ctl->done = 1;
    } else {
        if (L > 0) ctl->levels = L;
        if (globaltimer() - ctl->t0 > p.budget_ns) {
            ctl->status = RPQ_ETIMEOUT;
            ctl->iterations = L;
            ctl->done = 1;
        } else {
            if (L < RPQ_STATS_LEVELS) ctl->level_edges[L] = (long long)nedge;
            ctl->te += nedge;
            ctl->segments += nseg;
            if (nbun == 0) {  // nothing to expand: the next step is empty
                ctl->iterations = L + 1;
                ctl->done = 1;
            }
        }
    }
    // the other buffer is produced into during the next level
    for (int s = 0; s <= kShards; ++s) {
        ctl->shard_cnt[b ^ 1][s] = 0;
    }
    ctl->new_cnt[b ^ 1] = 0;
    ctl->edge_cnt[b ^ 1] = 0;
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) rpq_ssr_kernel(Params p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_red[2 * (kThreads / 32)];
    __shared__ unsigned long long s_bpre[kShards + 2];  // bundle prefix over shards
    __shared__ unsigned long long s_bbase[kShards + 1]; // bundle base index of each shard
    Slot* s_slots = reinterpret_cast<Slot*>(smem_raw);
    int32_t* s_tab = reinterpret_cast<int32_t*>(smem_raw + sizeof(Slot) * p.nslots);
    for (int i = threadIdx.x; i < p.nslots; i += blockDim.x) s_slots[i] = p.slots[i];
    for (int i = threadIdx.x; i < p.table_ints; i += blockDim.x) s_tab[i] = p.tables[i];
    Smem S;
    S.slots = s_slots;
    S.gbeg = s_tab;
    S.gslot = S.gbeg + p.nstates + 1;
    S.toff = S.gslot + p.ngroups;
    S.targets = S.toff + p.ngroups + 1;
    S.starts = S.targets + p.ntargets;
    S.finals = S.starts + p.nstarts;

    Ctl* ctl = p.ctl;
    const int lane = threadIdx.x & 31;
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long gthreads = (long long)gridDim.x * blockDim.x;
    if (gtid == 0) ctl->t0 = globaltimer();

    // ---- phase 0: P <- 0 --------------------------------------------------
    {
        uint4* v4 = reinterpret_cast<uint4*>(p.visited);
        const long long n4 = (long long)p.nstates * p.W / 4;
        for (long long i = gtid; i < n4; i += gthreads) v4[i] = make_uint4(0, 0, 0, 0);
    }
    grid_sync(ctl, [] {});

    // ---- seed: P = M = {(q_s, source)} (engine.py:106-109, :154-155) ------
    {
        unsigned long long nnew = 0, nedge = 0;
        if (blockIdx.x == 0 && threadIdx.x < 32) {
            for (int i0 = 0; i0 < p.nstarts; i0 += 32) {
                const int i = i0 + lane;
                bool fresh = false;
                int q = 0;
                if (i < p.nstarts) {
                    q = S.starts[i];
                    uint32_t* word = p.visited + (long long)q * p.W + (p.source >> 5);
                    const uint32_t bit = 1u << (p.source & 31);
                    fresh = !(atomicOr(word, bit) & bit);
                }
                nnew += fresh ? 1 : 0;
                const uint32_t T = emit_pairs(p, S, 0, fresh, q, p.source, lane);
                if (lane == 0) nedge += T;
            }
        }
        flush_counts(ctl, 0, nnew, nedge, s_red);
    }
    grid_sync(ctl, [&] { level_bookkeeping(p, 0); });

    // ---- level loop ---------------------------------------------------------
    const int wid = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    for (int L = 0;; ++L) {
        if (ld_volatile(&ctl->done)) break;
        const int cur = L & 1, nxt = cur ^ 1;
        // bundle prefix over shards (each shard's bundles are contiguous)
        if (threadIdx.x == 0) {
            unsigned long long run = 0;
            for (int s = 0; s <= kShards; ++s) {
                s_bpre[s] = run;
                s_bbase[s] = (unsigned long long)s * p.shard_buncap;
                unsigned long long c = ld_volatile(&ctl->shard_cnt[cur][s]) & 0xFFFFFFFFull;
                const unsigned long long cap = s < kShards ? p.shard_buncap : p.ovf_buncap;
                run += c < cap ? c : cap;
            }
            s_bpre[kShards + 1] = run;
        }
        __syncthreads();
        const unsigned long long nb = s_bpre[kShards + 1];
        const uint2* bun = p.bun[cur];
        const uint2* seg = p.seg[cur];
        unsigned long long nnew = 0, nedge = 0;
        // bundles are dealt round-robin over warps, CTA-major so that
        // consecutive bundles (often of one row) land on different SMs
        const unsigned long long step = (unsigned long long)gridDim.x * wpb;
        for (unsigned long long bi = (unsigned long long)wid * gridDim.x + blockIdx.x; bi < nb; bi += step) {
            int s = 0;
#pragma unroll
            for (int h = 64; h >= 1; h >>= 1)
                if (s + h <= kShards && s_bpre[s + h] <= bi) s += h;
            const uint2 bd = __ldcg(bun + s_bbase[s] + (bi - s_bpre[s]));
            if (bd.x == kHoleBundle) continue;
            const uint32_t s0 = bd.x;
            const uint32_t off = bd.y & 0xFFFFFFu;
            const uint32_t cnt = (bd.y >> 24) + 1;
            uint32_t my_start = 0, my_len = 0, my_grp = 0;
            if ((unsigned long long)s0 + lane < p.seg_alloc) {
                const uint2 sg = __ldcg(seg + s0 + lane);
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
            const uint32_t e = lane;
            const bool active = e < cnt;
            const int j = warp_upper_lane(excl, active ? e : 0);
            const uint32_t sj = __shfl_sync(FULL, my_start, j);
            const uint32_t exj = __shfl_sync(FULL, excl, j);
            const int gj = (int)__shfl_sync(FULL, my_grp, j);
            int w = 0;
            int t0 = 0, t1 = 0;
            if (active) {
                const Slot sl = S.slots[S.gslot[gj]];
                w = __ldg(sl.col + sj + (e - exj));
                t0 = S.toff[gj];
                t1 = S.toff[gj + 1];
            }
            for (int k = 0; k < p.maxT; ++k) {
                bool fresh = false;
                int q2 = 0;
                if (active && t0 + k < t1) {
                    q2 = S.targets[t0 + k];
                    uint32_t* word = p.visited + (long long)q2 * p.W + (w >> 5);
                    const uint32_t bit = 1u << (w & 31);
                    if (!(*word & bit)) fresh = !(atomicOr(word, bit) & bit);
                }
                nnew += fresh ? 1 : 0;
                const uint32_t T = emit_pairs(p, S, nxt, fresh, q2, w, lane);
                if (lane == 0) nedge += T;
            }
        }
        flush_counts(ctl, nxt, nnew, nedge, s_red);
        grid_sync(ctl, [&] { level_bookkeeping(p, L + 1); });
    }

    // ---- epilogue: answer = OR of P's rows at final states (engine.py:112-114)
    if (ld_volatile(&ctl->status) == 0) {
        const long long nwords = ((long long)p.nv + 31) >> 5;
        unsigned long long cnt = 0;
        for (long long i = gtid; i < nwords; i += gthreads) {
            uint32_t acc = 0;
            for (int f = 0; f < p.nfinals; ++f)
                acc |= __ldcg(p.visited + (long long)S.finals[f] * p.W + i);
            cnt += __popc(acc);
            uint8_t* out = p.reach + i * 32;
            if (i * 32 + 32 <= p.nv) {
                uint32_t bytes[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t nib = (acc >> (4 * k)) & 0xFu;
                    bytes[k] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
                }
                reinterpret_cast<uint4*>(out)[0] = make_uint4(bytes[0], bytes[1], bytes[2], bytes[3]);
                reinterpret_cast<uint4*>(out)[1] = make_uint4(bytes[4], bytes[5], bytes[6], bytes[7]);
            } else {
                for (int k = 0; i * 32 + k < p.nv; ++k) out[k] = (acc >> k) & 1u;
            }
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) cnt += __shfl_xor_sync(FULL, cnt, d);
        if (lane == 0 && cnt) atomicAdd(&ctl->reach_count, cnt);
    }
}

// int64 -> narrow copy used at upload (sparse_bool.py keeps int64 everywhere)
template <typename In, typename Out>
__global__ void narrow_kernel(const In* __restrict__ in, Out* __restrict__ out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (Out)in[i];
}

}  // namespace

// ===========================================================================
// host side
// ===========================================================================

struct LabelDev {
    bool resident = false;
    uint32_t* rowptr[2] = {nullptr, nullptr};
    int32_t* col[2] = {nullptr, nullptr};
    int64_t nnz[2] = {0, 0};
};

struct rpq_graph {
    int device = 0;
    int32_t nv = 0;
    int32_t nl = 0;
    int sm_count = 0;
    std::vector<LabelDev> labels;
    std::mutex mu;
    int64_t bytes = 0;
};

struct rpq_query {
    rpq_graph* g = nullptr;
    int32_t nstates = 0;
    std::vector<int32_t> tables;  // host copy
    std::vector<Slot> slots;
    int ngroups = 0, nslots = 0, ntargets = 0, nstarts = 0, nfinals = 0, maxT = 0;
    int32_t* d_tables = nullptr;
    Slot* d_slots = nullptr;
    uint32_t* d_visited = nullptr;
    uint2* d_seg[2] = {nullptr, nullptr};
    uint2* d_bun[2] = {nullptr, nullptr};
    Ctl* d_ctl = nullptr;
    Ctl* h_ctl = nullptr;  // pinned
    uint8_t* d_reach = nullptr;
    unsigned long long shard_segcap = 0, shard_buncap = 0, ovf_segcap = 0, ovf_buncap = 0;
    unsigned long long seg_alloc = 0, bun_alloc = 0;
    long long W = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t last_stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int grid = 0;
    size_t smem = 0;
    bool ran = false;
    std::mutex mu;
};

namespace {

template <typename I>
int upload_csr(rpq_graph* g, LabelDev& L, int dir, int64_t nnz, const I* indptr, const I* indices) {
    const int64_t nv = g->nv;
    if (nnz < 0 || nnz > 0xFFFFFFFFll) return fail(RPQ_EINVAL, "label nnz must be < 2^32");
    if (!indptr || (nnz > 0 && !indices)) return fail(RPQ_EINVAL, "null CSR pointer");
    if ((int64_t)indptr[0] != 0 || (int64_t)indptr[nv] != nnz)
        return fail(RPQ_EINVAL, "CSR indptr must start at 0 and end at nnz");
    const int64_t n_items = std::max<int64_t>(nv + 1, nnz);
    void* staging = nullptr;
    CUDA_TRY(cudaMalloc(&staging, (size_t)n_items * sizeof(I)));
    CUDA_TRY(cudaMalloc(&L.rowptr[dir], (size_t)(nv + 1) * sizeof(uint32_t)));
    CUDA_TRY(cudaMalloc(&L.col[dir], (size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t)));
    CUDA_TRY(cudaMemcpy(staging, indptr, (size_t)(nv + 1) * sizeof(I), cudaMemcpyHostToDevice));
    narrow_kernel<I, uint32_t><<<1184, 256>>>((const I*)staging, L.rowptr[dir], nv + 1);
    CUDA_TRY(cudaGetLastError());
    if (nnz > 0) {
        CUDA_TRY(cudaMemcpy(staging, indices, (size_t)nnz * sizeof(I), cudaMemcpyHostToDevice));
        narrow_kernel<I, int32_t><<<1184, 256>>>((const I*)staging, L.col[dir], nnz);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaFree(staging));
    L.nnz[dir] = nnz;
    g->bytes += (nv + 1) * 4 + std::max<int64_t>(nnz, 1) * 4;
    return RPQ_OK;
}

void free_label(LabelDev& L) {
    for (int d = 0; d < 2; ++d) {
        if (L.rowptr[d]) cudaFree(L.rowptr[d]);
        if (L.col[d]) cudaFree(L.col[d]);
        L.rowptr[d] = nullptr;
        L.col[d] = nullptr;
    }
    L.resident = false;
}

template <typename I>
int set_label_impl(rpq_graph* g, int32_t label, int64_t fn, const I* fp, const I* fi, int64_t bn,
                   const I* bp, const I* bi) {
    if (!g) return fail(RPQ_EINVAL, "null graph");
    if (label < 0 || label >= g->nl) return fail(RPQ_EINVAL, "label index out of range");
    std::lock_guard<std::mutex> lk(g->mu);
    LabelDev& L = g->labels[label];
    if (L.resident) return RPQ_OK;
    if (cudaSetDevice(g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice failed");
    int rc = upload_csr<I>(g, L, 0, fn, fp, fi);
    if (rc == RPQ_OK) rc = upload_csr<I>(g, L, 1, bn, bp, bi);
    if (rc != RPQ_OK) {
        free_label(L);
        return rc;
    }
    L.resident = true;
    return RPQ_OK;
}

void free_query_buffers(rpq_query* q) {
    if (q->d_tables) cudaFree(q->d_tables);
    if (q->d_slots) cudaFree(q->d_slots);
    if (q->d_visited) cudaFree(q->d_visited);
    for (int b = 0; b < 2; ++b) {
        if (q->d_seg[b]) cudaFree(q->d_seg[b]);
        if (q->d_bun[b]) cudaFree(q->d_bun[b]);
    }
    if (q->d_ctl) cudaFree(q->d_ctl);
    if (q->h_ctl) cudaFreeHost(q->h_ctl);
    if (q->d_reach) cudaFree(q->d_reach);
    if (q->ev0) cudaEventDestroy(q->ev0);
    if (q->ev1) cudaEventDestroy(q->ev1);
    if (q->own_stream) cudaStreamDestroy(q->own_stream);
}

}  // namespace

extern "C" {

int rpq_abi_version(void) { return RPQ_ABI_VERSION; }

const char* rpq_last_error(void) { return g_last_error.c_str(); }

int rpq_device_info(int32_t device, int32_t* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes) {
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (l2_bytes) *l2_bytes = prop.l2CacheSize;
    if (hbm_bytes) *hbm_bytes = (int64_t)prop.totalGlobalMem;
    return RPQ_OK;
}

int rpq_graph_create(int32_t num_vertices, int32_t num_labels, int32_t device, rpq_graph** out) {
    if (!out) return fail(RPQ_EINVAL, "null output handle");
    *out = nullptr;
    if (num_vertices < 0 || num_labels < 0) return fail(RPQ_EINVAL, "negative graph dimensions");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(RPQ_EINVAL, "device index out of range");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(RPQ_ECUDA, "this build targets sm_100a (B200) only");
    rpq_graph* g = new rpq_graph();
    g->device = device;
    g->nv = num_vertices;
    g->nl = num_labels;
    g->sm_count = prop.multiProcessorCount;
    g->labels.resize(num_labels);
    *out = g;
    return RPQ_OK;
}

int rpq_graph_set_label(rpq_graph* g, int32_t label, int64_t fwd_nnz, const int64_t* fwd_indptr,
                        const int64_t* fwd_indices, int64_t bwd_nnz, const int64_t* bwd_indptr,
                        const int64_t* bwd_indices) {
    return set_label_impl<int64_t>(g, label, fwd_nnz, fwd_indptr, fwd_indices, bwd_nnz, bwd_indptr,
                                   bwd_indices);
}

int rpq_graph_set_label_i32(rpq_graph* g, int32_t label, int64_t fwd_nnz, const int32_t* fwd_indptr,
                            const int32_t* fwd_indices, int64_t bwd_nnz, const int32_t* bwd_indptr,
                            const int32_t* bwd_indices) {
    return set_label_impl<int32_t>(g, label, fwd_nnz, fwd_indptr, fwd_indices, bwd_nnz, bwd_indptr,
                                   bwd_indices);
}

int rpq_graph_label_resident(const rpq_graph* g, int32_t label) {
    if (!g || label < 0 || label >= g->nl) return 0;
    return g->labels[label].resident ? 1 : 0;
}

int64_t rpq_graph_device_bytes(const rpq_graph* g) { return g ? g->bytes : 0; }

int rpq_graph_destroy(rpq_graph* g) {
    if (!g) return RPQ_OK;
    cudaSetDevice(g->device);
    for (auto& L : g->labels) free_label(L);
    delete g;
    return RPQ_OK;
}

int rpq_query_create(rpq_graph* g, int32_t nstates, int32_t ntrans, const int32_t* t_src,
                     const int32_t* t_label, const uint8_t* t_inv, const int32_t* t_dst,
                     int32_t nstarts, const int32_t* starts, int32_t nfinals, const int32_t* finals,
                     rpq_query** out) {
    if (!out) return fail(RPQ_EINVAL, "null output handle");
    *out = nullptr;
    if (!g) return fail(RPQ_EINVAL, "null graph");
    if (nstates < 1 || nstates > kMaxStates)
        return fail(RPQ_EINVAL, "nstates must be in [1, " + std::to_string(kMaxStates) + "]");
    if (ntrans < 0 || nstarts < 0 || nfinals < 0) return fail(RPQ_EINVAL, "negative count");
    if ((ntrans && (!t_src || !t_label || !t_inv || !t_dst)) || (nstarts && !starts) ||
        (nfinals && !finals))
        return fail(RPQ_EINVAL, "null automaton array");

    // usable transitions -> slots (label, inv) and (state, slot) groups
    std::map<std::pair<int, int>, int> slot_of;
    std::map<std::pair<int, int>, std::set<int>> group_targets;  // (state, slot) -> targets
    std::vector<std::pair<int, int>> slot_keys;
    {
        std::set<std::pair<int, int>> keys;
        for (int i = 0; i < ntrans; ++i) {
            if (t_src[i] < 0 || t_src[i] >= nstates || t_dst[i] < 0 || t_dst[i] >= nstates)
                return fail(RPQ_EINVAL, "transition state out of range");
            if (t_label[i] < 0) return fail(RPQ_EINVAL, "negative label index");
            if (t_label[i] >= g->nl) continue;  // engine.py:100-101
            keys.insert({t_label[i], t_inv[i] ? 1 : 0});
        }
        for (auto& k : keys) {
            slot_of[k] = (int)slot_keys.size();
            slot_keys.push_back(k);
        }
        for (int i = 0; i < ntrans; ++i) {
            if (t_label[i] >= g->nl) continue;
            int s = slot_of[{t_label[i], t_inv[i] ? 1 : 0}];
            group_targets[{t_src[i], s}].insert(t_dst[i]);
        }
    }
    if ((int)slot_keys.size() > kMaxSlots) return fail(RPQ_EINVAL, "too many distinct symbols");
    if ((int)group_targets.size() > kMaxGroups)
        return fail(RPQ_EINVAL, "automaton has more than 256 (state, symbol) groups");
    for (auto& k : slot_keys)
        if (!g->labels[k.first].resident)
            return fail(RPQ_ENOLABEL, "label " + std::to_string(k.first) + " is not resident");

    rpq_query* q = new rpq_query();
    q->g = g;
    q->nstates = nstates;
    std::vector<int32_t> gbeg(nstates + 1, 0), gslot, toff, targets;
    std::vector<int> gcount(nstates, 0);
    for (auto& kv : group_targets) gcount[kv.first.first]++;
    for (int s = 0; s < nstates; ++s) gbeg[s + 1] = gbeg[s] + gcount[s];
    // std::map iterates (state, slot) in order, so groups of a state are contiguous
    int maxT = 0;
    toff.push_back(0);
    uint64_t seg_per_vertex = 0, edge_bound = 0;
    for (auto& kv : group_targets) {
        gslot.push_back(kv.first.second);
        for (int t : kv.second) targets.push_back(t);
        toff.push_back((int32_t)targets.size());
        maxT = std::max<int>(maxT, (int)kv.second.size());
        const auto& key = slot_keys[kv.first.second];
        const int64_t nnz = g->labels[key.first].nnz[key.second];
        seg_per_vertex += 1;
        edge_bound += (uint64_t)nnz;
    }
    std::set<int> sset, fset;
    for (int i = 0; i < nstarts; ++i)
        if (starts[i] >= 0 && starts[i] < nstates) sset.insert(starts[i]);
    for (int i = 0; i < nfinals; ++i)
        if (finals[i] >= 0 && finals[i] < nstates) fset.insert(finals[i]);
    q->ngroups = (int)gslot.size();
    q->nslots = (int)slot_keys.size();
    q->ntargets = (int)targets.size();
    q->nstarts = (int)sset.size();
    q->nfinals = (int)fset.size();
    q->maxT = maxT;
    q->tables.insert(q->tables.end(), gbeg.begin(), gbeg.end());
    q->tables.insert(q->tables.end(), gslot.begin(), gslot.end());
    q->tables.insert(q->tables.end(), toff.begin(), toff.end());
    q->tables.insert(q->tables.end(), targets.begin(), targets.end());
    q->tables.insert(q->tables.end(), sset.begin(), sset.end());
    q->tables.insert(q->tables.end(), fset.begin(), fset.end());
    for (auto& k : slot_keys) {
        const LabelDev& L = g->labels[k.first];
        q->slots.push_back(Slot{L.rowptr[k.second], L.col[k.second]});
    }
    // queue capacities: every (state, vertex) pair is discovered at most once,
    // so a level holds at most |V| segments per group (+ splits of huge rows);
    // bundles are at most one partial per emission plus edges / kBundle.
    const uint64_t nv = (uint64_t)g->nv;
    // bound = worst case of one level; regular shards get 1/kShards of it
    // with headroom, the overflow shard the whole bound
    const unsigned long long segbound = nv * seg_per_vertex + edge_bound / kSegLenMax + 64;
    const unsigned long long bunbound = segbound + edge_bound / kBundle + 64;
    q->shard_segcap = segbound / kShards + segbound / (4 * kShards) + 1024;
    q->shard_buncap = bunbound / kShards + bunbound / (4 * kShards) + 1024;
    q->ovf_segcap = segbound;
    q->ovf_buncap = bunbound;
    q->seg_alloc = q->shard_segcap * kShards + q->ovf_segcap + 32;
    q->bun_alloc = q->shard_buncap * kShards + q->ovf_buncap;
    if (q->seg_alloc >= 0xFFFFFFFFull || q->shard_buncap >= 0xFFFFFFFFull || q->ovf_buncap >= 0xFFFFFFFFull) {
        delete q;
        return fail(RPQ_EINVAL, "segment queue would exceed 2^32 entries");
    }
    q->W = (((long long)g->nv + 31) / 32 + 3) / 4 * 4;

    auto bail = [&](int rc) {
        free_query_buffers(q);
        delete q;
        return rc;
    };
    if (cudaSetDevice(g->device) != cudaSuccess) return bail(fail(RPQ_ECUDA, "cudaSetDevice"));
#define QTRY(expr)                                                  \
    do {                                                            \
        cudaError_t e_ = (expr);                                    \
        if (e_ != cudaSuccess) return bail(cuda_fail(e_, #expr));   \
    } while (0)
    QTRY(cudaMalloc(&q->d_tables, std::max<size_t>(q->tables.size(), 1) * sizeof(int32_t)));
    QTRY(cudaMalloc(&q->d_slots, std::max<size_t>(q->slots.size(), 1) * sizeof(Slot)));
    QTRY(cudaMalloc(&q->d_visited, (size_t)q->W * nstates * sizeof(uint32_t)));
    for (int b = 0; b < 2; ++b) {
        QTRY(cudaMalloc(&q->d_seg[b], (size_t)q->seg_alloc * sizeof(uint2)));
        QTRY(cudaMalloc(&q->d_bun[b], (size_t)q->bun_alloc * sizeof(uint2)));
        // segments beyond a bundle's own are read (and ignored) by the
        // consumer's 32-wide load; keep them finite so its scan cannot wrap
        QTRY(cudaMemset(q->d_seg[b], 0, (size_t)q->seg_alloc * sizeof(uint2)));
    }
    QTRY(cudaMalloc(&q->d_ctl, sizeof(Ctl)));
    QTRY(cudaMallocHost(&q->h_ctl, sizeof(Ctl)));
    QTRY(cudaMalloc(&q->d_reach, (size_t)(q->W * 32 + 32)));
    QTRY(cudaStreamCreateWithFlags(&q->own_stream, cudaStreamNonBlocking));
    QTRY(cudaEventCreate(&q->ev0));
    QTRY(cudaEventCreate(&q->ev1));
    if (!q->tables.empty())
        QTRY(cudaMemcpy(q->d_tables, q->tables.data(), q->tables.size() * sizeof(int32_t),
                        cudaMemcpyHostToDevice));
    if (!q->slots.empty())
        QTRY(cudaMemcpy(q->d_slots, q->slots.data(), q->slots.size() * sizeof(Slot),
                        cudaMemcpyHostToDevice));
    q->smem = q->slots.size() * sizeof(Slot) + q->tables.size() * sizeof(int32_t) + 16;
    if (q->smem > 48 * 1024)
        QTRY(cudaFuncSetAttribute(rpq_ssr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)q->smem));
    int per_sm = 0;
    QTRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rpq_ssr_kernel, kThreads, q->smem));
    if (per_sm < 1) return bail(fail(RPQ_ECUDA, "step kernel cannot be resident"));
    q->grid = g->sm_count * per_sm;
#undef QTRY
    *out = q;
    return RPQ_OK;
}

int rpq_query_run(rpq_query* q, int32_t source, double timeout_s, void* stream) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (source < 0 || source >= q->g->nv)
        return fail(RPQ_ERANGE, "vertex index " + std::to_string(source) + " out of range");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    cudaStream_t st = stream ? (cudaStream_t)stream : q->own_stream;
    Params p{};
    p.tables = q->d_tables;
    p.slots = q->d_slots;
    p.visited = q->d_visited;
    for (int b = 0; b < 2; ++b) {
        p.seg[b] = q->d_seg[b];
        p.bun[b] = q->d_bun[b];
    }
    p.ctl = q->d_ctl;
    p.reach = q->d_reach;
    p.shard_segcap = q->shard_segcap;
    p.shard_buncap = q->shard_buncap;
    p.ovf_segcap = q->ovf_segcap;
    p.ovf_buncap = q->ovf_buncap;
    p.seg_alloc = q->seg_alloc;
    p.bun_alloc = q->bun_alloc;
    if (!(timeout_s >= 0) || std::isinf(timeout_s) || timeout_s > 1.0e9)
        p.budget_ns = ~0ull;
    else
        p.budget_ns = (unsigned long long)(timeout_s * 1e9);
    p.W = q->W;
    p.nv = q->g->nv;
    p.nstates = q->nstates;
    p.ngroups = q->ngroups;
    p.nslots = q->nslots;
    p.ntargets = q->ntargets;
    p.nstarts = q->nstarts;
    p.nfinals = q->nfinals;
    p.maxT = q->maxT;
    p.source = source;
    p.table_ints = (int)q->tables.size();
    CUDA_TRY(cudaEventRecord(q->ev0, st));
    CUDA_TRY(cudaMemsetAsync(q->d_ctl, 0, sizeof(Ctl), st));
    void* args[] = {&p};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)rpq_ssr_kernel, dim3(q->grid), dim3(kThreads),
                                         args, q->smem, st));
    CUDA_TRY(cudaEventRecord(q->ev1, st));
    CUDA_TRY(cudaMemcpyAsync(q->h_ctl, q->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    q->last_stream = st;
    q->ran = true;
    return RPQ_OK;
}

int rpq_query_wait(rpq_query* q, rpq_stats* stats) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (!q->ran) return fail(RPQ_EINVAL, "query has not been run");
    CUDA_TRY(cudaStreamSynchronize(q->last_stream));
    const Ctl& c = *q->h_ctl;
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, q->ev0, q->ev1));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->status = c.status;
        stats->iterations = c.iterations;
        stats->levels = c.levels;
        stats->grid = q->grid;
        stats->te = (int64_t)c.te;
        stats->segments = (int64_t)c.segments;
        stats->visited_pairs = (int64_t)c.pairs;
        stats->reach_count = (int64_t)c.reach_count;
        stats->device_ms = ms;
        for (int i = 0; i < RPQ_STATS_LEVELS; ++i) {
            stats->level_new[i] = c.level_new[i];
            stats->level_edges[i] = c.level_edges[i];
        }
    }
    if (c.status == ST_OVERFLOW) {
        if (stats) stats->status = RPQ_ECUDA;
        return fail(RPQ_ECUDA, "internal: frontier queue capacity exceeded");
    }
    if (c.status == ST_DEADLOCK) {
        if (stats) stats->status = RPQ_ECUDA;
        return fail(RPQ_ECUDA, "internal: grid barrier spin limit exceeded");
    }
    if (c.status == RPQ_ETIMEOUT) return fail(RPQ_ETIMEOUT, "query timed out");
    if (c.status != 0) return fail(RPQ_ECUDA, "kernel status " + std::to_string(c.status));
    return RPQ_OK;
}

int rpq_query_reach_device(rpq_query* q, uint8_t** d_reach) {
    if (!q || !d_reach) return fail(RPQ_EINVAL, "null argument");
    *d_reach = q->d_reach;
    return RPQ_OK;
}

int rpq_query_copy_reach(rpq_query* q, uint8_t* host_reach) {
    if (!q || !host_reach) return fail(RPQ_EINVAL, "null argument");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    if (q->g->nv == 0) return RPQ_OK;
    CUDA_TRY(cudaMemcpyAsync(host_reach, q->d_reach, (size_t)q->g->nv, cudaMemcpyDeviceToHost,
                             q->last_stream ? q->last_stream : q->own_stream));
    CUDA_TRY(cudaStreamSynchronize(q->last_stream ? q->last_stream : q->own_stream));
    return RPQ_OK;
}

int rpq_query_copy_visited(rpq_query* q, uint32_t* host_words, int64_t nwords) {
    if (!q || !host_words) return fail(RPQ_EINVAL, "null argument");
    const int64_t words = ((int64_t)q->g->nv + 31) / 32;
    if (nwords < words * q->nstates) return fail(RPQ_EINVAL, "output buffer too small");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    cudaStream_t st = q->last_stream ? q->last_stream : q->own_stream;
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaMemcpy2D(host_words, (size_t)words * 4, q->d_visited, (size_t)q->W * 4,
                          (size_t)words * 4, (size_t)q->nstates, cudaMemcpyDeviceToHost));
    return RPQ_OK;
}

int rpq_query_destroy(rpq_query* q) {
    if (!q) return RPQ_OK;
    cudaSetDevice(q->g->device);
    if (q->ran && q->last_stream) cudaStreamSynchronize(q->last_stream);
    free_query_buffers(q);
    delete q;
    return RPQ_OK;
}

int rpq_ssr(rpq_graph* g, int32_t nstates, int32_t ntrans, const int32_t* t_src,
            const int32_t* t_label, const uint8_t* t_inv, const int32_t* t_dst, int32_t nstarts,
            const int32_t* starts, int32_t nfinals, const int32_t* finals, int32_t source,
            double timeout_s, uint8_t* out_reach, rpq_stats* stats) {
    if (!g) return fail(RPQ_EINVAL, "null graph");
    if (source < 0 || source >= g->nv)
        return fail(RPQ_ERANGE, "vertex index " + std::to_string(source) + " out of range");
    rpq_query* q = nullptr;
    int rc = rpq_query_create(g, nstates, ntrans, t_src, t_label, t_inv, t_dst, nstarts, starts,
                              nfinals, finals, &q);
    if (rc != RPQ_OK) return rc;
    rc = rpq_query_run(q, source, timeout_s, nullptr);
    if (rc == RPQ_OK) rc = rpq_query_wait(q, stats);
    if (rc == RPQ_OK && out_reach) rc = rpq_query_copy_reach(q, out_reach);
    std::string err = g_last_error;
    rpq_query_destroy(q);
    g_last_error = err;
    return rc;
}

}  // extern "C"
