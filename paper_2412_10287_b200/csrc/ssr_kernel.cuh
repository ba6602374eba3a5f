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
// unvisited (q', w) scans A_s^T row w for a frontier member of the source
// state, early exit), chosen from the frontier's edge count against the
// unvisited edge estimate (Beamer's rule).  Either way the result is the
// same set: P only grows by (q', w) pairs with a frontier predecessor.
#pragma once

namespace rpqk {

constexpr int kThreads = 256;        // 8 warps per CTA
constexpr int kMinBlocks = 3;        // CTAs per SM the register budget targets
constexpr int kBundle = 32;          // edges per bundle (<= 32 segments)
constexpr int kShards = 64;          // queue shards (+1 overflow shard), by CTA
constexpr int kMaxStates = 256;
constexpr int kMaxGroups = 256;      // group id is 8 bits in a segment
constexpr int kMaxSlots = 128;
constexpr uint32_t kSegLenMax = (1u << 24) - 1;
constexpr uint32_t kHoleBundle = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xffffffffu;
constexpr int kPullInline = 4;       // in-edges each lane tests before warp help

constexpr int ST_OVERFLOW = 100;
constexpr int ST_DEADLOCK = 101;

constexpr int DIR_PUSH = 0;
constexpr int DIR_PULL = 1;

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
    int dir;   // direction of the level about to run
    int plan;  // 1: the push level about to run must first emit its queue from F
    int pad;
    unsigned long long t0;
    unsigned long long shard_cnt[2][kShards + 1];  // (segments << 32) | bundles
    unsigned long long new_cnt[2];
    unsigned long long edge_cnt[2];
    unsigned int state_front[2][kMaxStates];       // |F_L| per state, by parity of L
    unsigned long long state_vis[kMaxStates];      // |P| per state
    unsigned long long te_push;                    // edges expanded by push levels
    unsigned long long te_exact;                   // push-model TE over P (flag)
    unsigned long long segments;
    unsigned long long pairs;
    unsigned long long reach_count;
    long long level_new[64];
    long long level_edges[64];
    int level_dir[64];
};

struct Params {
    const int32_t* tables;
    const Slot* slots;       // A_s, then A_s^T at [nslots, 2*nslots)
    const unsigned long long* slot_nnz;
    uint32_t* visited;
    uint32_t* fb[3];
    uint2* seg[2];
    uint2* bun[2];
    Ctl* ctl;
    uint8_t* reach;
    unsigned long long shard_segcap, shard_buncap, ovf_segcap, ovf_buncap;
    unsigned long long seg_alloc;
    unsigned long long budget_ns;
    long long W;             // words per bitmap row (multiple of 4)
    int nv;
    int nstates, ngroups, nslots, ntargets, nstarts, nfinals, nin;
    int maxT;
    int source;
    int table_ints;
    int dir_mode;            // 0 auto, 1 push only, 2 pull after the seed
    int count_te;
    float alpha;             // pull when m_f * alpha > m_u
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

// Control words every thread needs after a barrier, broadcast through smem.
struct CtlView {
    int done;
    int dir;
    int plan;
};

// Grid barrier for a cooperative launch.  The last CTA to arrive runs
// `serial` (one thread) before releasing everyone, so per-level bookkeeping
// is ordered after all CTAs' work and before any CTA's next level.  Waiters
// spin on a relaxed load (no per-iteration L1 invalidation) and fence once.
template <class F>
__device__ __forceinline__ void grid_sync(Ctl* ctl, CtlView* view, F serial) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nblocks = gridDim.x;
        unsigned gen = ld_relaxed_u32(&ctl->bar_gen);
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
            while (ld_relaxed_u32(&ctl->bar_gen) == gen) {
                __nanosleep(20);
                if ((++spins & 4095u) == 0) {
                    unsigned long long now = globaltimer();
                    if (ts == 0) {
                        ts = now;
                    } else if (now - ts > 20000000000ull) {  // 20 s: cannot happen co-resident
                        atomicExch(&ctl->status, ST_DEADLOCK);
                        atomicExch(&ctl->done, 1);
                        break;
                    }
                }
            }
        }
        __threadfence();  // acquire side; also invalidates this SM's L1 (CCTL.IVALL)
        view->done = ld_volatile(&ctl->done);
        view->dir = ld_volatile(&ctl->dir);
        view->plan = ld_volatile(&ctl->plan);
    }
    __syncthreads();
}

// Shard-local reservation of `nseg` segments and `nb` bundles in queue buffer
// `b` (one lane).  A reservation that does not fit its CTA's shard spills to
// the overflow shard; the part of its bundle range inside the regular shard,
// [*hole_lo, *hole_hi), must then be filled with kHoleBundle by the caller.
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

// Warp-cooperative emission of the row segments of (state q, vertex w) pairs
// (one candidate per lane) into queue buffer `b`.  Returns the edges emitted.
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

// Per-CTA flush of a level's counters (one atomic per CTA and counter).
__device__ __forceinline__ void flush_counts(Ctl* ctl, int b, unsigned long long nnew,
                                             unsigned long long nedge, unsigned long long* red,
                                             unsigned int* s_state, int nstates) {
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
    for (int q = threadIdx.x; q < nstates; q += blockDim.x) {
        const unsigned int c = s_state[q];
        if (c) {
            atomicAdd(&ctl->state_front[b][q], c);
            s_state[q] = 0;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void count_state(unsigned int* s_state, bool fresh, int q) {
    if (fresh) atomicAdd(&s_state[q], 1u);
}

// Queue totals of buffer b (bundles / segments, clamped to shard capacity).
__device__ __forceinline__ void queue_totals(const Params& p, int b, unsigned long long* nbun,
                                             unsigned long long* nseg) {
    unsigned long long tb = 0, ts = 0;
    for (int s = 0; s <= kShards; ++s) {
        const unsigned long long c = ld_volatile(&p.ctl->shard_cnt[b][s]);
        const unsigned long long bc = c & 0xFFFFFFFFull, sc = c >> 32;
        const unsigned long long bcap = s < kShards ? p.shard_buncap : p.ovf_buncap;
        const unsigned long long scap = s < kShards ? p.shard_segcap : p.ovf_segcap;
        tb += bc < bcap ? bc : bcap;
        ts += sc < scap ? sc : scap;
    }
    *nbun = tb;
    *nseg = ts;
}

// Bookkeeping after frontier F_L has been produced (serial, one thread).
// Mirrors the masked loop (engine.py:156-160): run while the frontier is
// non-empty, check the deadline first, then step.  Also picks the direction
// of level L.
__device__ void level_bookkeeping(const Params& p, const Smem& S, int L) {
    Ctl* ctl = p.ctl;
    const int b = L & 1;
    const unsigned long long nnew = ld_volatile(&ctl->new_cnt[b]);
    const unsigned long long nedge = ld_volatile(&ctl->edge_cnt[b]);
    const int produced_by_push = (L == 0) || (ctl->dir == DIR_PUSH);
    unsigned long long nbun, nseg;
    queue_totals(p, b, &nbun, &nseg);
    ctl->pairs += nnew;
    for (int q = 0; q < p.nstates; ++q) ctl->state_vis[q] += ctl->state_front[b][q];
    if (L < 64) ctl->level_new[L] = (long long)nnew;
    if (ld_volatile(&ctl->overflow)) {
        ctl->status = ST_OVERFLOW;
        ctl->iterations = L;
        ctl->done = 1;
    } else if (ld_volatile(&ctl->status) != 0) {
        ctl->done = 1;
    } else if (nnew == 0) {
        ctl->iterations = L;
        ctl->done = 1;
    } else if (globaltimer() - ctl->t0 > p.budget_ns) {
        ctl->status = RPQ_ETIMEOUT;
        ctl->iterations = L;
        ctl->done = 1;
    } else {
        if (L > 0) ctl->levels = L;
        int next = DIR_PUSH;
        if (p.dir_mode == 2) {
            next = DIR_PULL;
        } else if (p.dir_mode == 0) {
            // m_f: edges out of F_L (exact after a push level, estimated from
            // average degrees after a pull level); m_u: in-edges of unvisited
            // targets whose source state has a frontier.  Beamer: pull when
            // m_f * alpha > m_u.
            double mf = 0.0, mu = 0.0;
            const double nv = (double)p.nv;
            if (produced_by_push) {
                mf = (double)nedge;
            } else {
                for (int q = 0; q < p.nstates; ++q) {
                    const unsigned int f = ctl->state_front[b][q];
                    if (!f) continue;
                    for (int g = S.gbeg[q]; g < S.gbeg[q + 1]; ++g)
                        mf += (double)f * (double)p.slot_nnz[S.gslot[g]] / nv;
                }
            }
            for (int q2 = 0; q2 < p.nstates; ++q2) {
                const double unvis = nv - (double)ctl->state_vis[q2];
                for (int k = S.ibeg[q2]; k < S.ibeg[q2 + 1]; ++k)
                    if (ctl->state_front[b][S.isrc[k]])
                        mu += (double)p.slot_nnz[S.islot[k]] * unvis / nv;
            }
            next = (mf * (double)p.alpha > mu) ? DIR_PULL : DIR_PUSH;
        }
        ctl->plan = 0;
        if (next == DIR_PUSH) {
            if (produced_by_push) {
                ctl->te_push += nedge;
                ctl->segments += nseg;
                if (L < 64) ctl->level_edges[L] = (long long)nedge;
                if (nbun == 0) {  // nothing to expand: the next step is empty
                    ctl->iterations = L + 1;
                    ctl->done = 1;
                }
            } else {
                ctl->plan = 1;  // emit F_L's queue from its bitmap first
            }
        } else if (L < 64) {
            ctl->level_edges[L] = -1;  // pull: edges scanned are not push-model edges
        }
        ctl->dir = next;
        if (L < 64) ctl->level_dir[L] = next;
    }
    // the other parity is produced into during level L
    for (int s = 0; s <= kShards; ++s) ctl->shard_cnt[b ^ 1][s] = 0;
    ctl->new_cnt[b ^ 1] = 0;
    ctl->edge_cnt[b ^ 1] = 0;
    for (int q = 0; q < p.nstates; ++q) ctl->state_front[b ^ 1][q] = 0;
}

// After a plan phase emitted F_L's queue into buffer L&1.
__device__ void plan_bookkeeping(const Params& p, int L) {
    Ctl* ctl = p.ctl;
    const int b = L & 1;
    unsigned long long nbun, nseg;
    queue_totals(p, b, &nbun, &nseg);
    const unsigned long long nedge = ld_volatile(&ctl->edge_cnt[b]);
    ctl->plan = 0;
    if (ld_volatile(&ctl->overflow)) {
        ctl->status = ST_OVERFLOW;
        ctl->iterations = L;
        ctl->done = 1;
        return;
    }
    ctl->te_push += nedge;
    ctl->segments += nseg;
    if (L < 64) ctl->level_edges[L] = (long long)nedge;
    if (nbun == 0) {
        ctl->iterations = L + 1;
        ctl->done = 1;
    }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) ssr_kernel(Params p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_red[2 * (kThreads / 32)];
    __shared__ unsigned long long s_bpre[kShards + 2];
    __shared__ unsigned int s_state[kMaxStates];     // per-state discoveries (flushed per level)
    __shared__ unsigned char s_active[kMaxStates];   // state has a non-empty current frontier
    __shared__ int s_ptarget[kMaxStates];            // pull target states of this level
    __shared__ int s_nptarget;
    __shared__ CtlView s_view;

    Slot* s_slots = reinterpret_cast<Slot*>(smem_raw);
    int32_t* s_tab = reinterpret_cast<int32_t*>(smem_raw + sizeof(Slot) * 2 * p.nslots);
    for (int i = threadIdx.x; i < 2 * p.nslots; i += blockDim.x) s_slots[i] = p.slots[i];
    for (int i = threadIdx.x; i < p.table_ints; i += blockDim.x) s_tab[i] = p.tables[i];
    for (int i = threadIdx.x; i < kMaxStates; i += blockDim.x) s_state[i] = 0;
    Smem S;
    S.slots = s_slots;
    S.gbeg = s_tab;
    S.gslot = S.gbeg + p.nstates + 1;
    S.toff = S.gslot + p.ngroups;
    S.targets = S.toff + p.ngroups + 1;
    S.starts = S.targets + p.ntargets;
    S.finals = S.starts + p.nstarts;
    S.ibeg = S.finals + p.nfinals;
    S.isrc = S.ibeg + p.nstates + 1;
    S.islot = S.isrc + p.nin;

    Ctl* ctl = p.ctl;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long gthreads = (long long)gridDim.x * blockDim.x;
    const long long gwarp = (long long)blockIdx.x * wpb + wid;
    const long long nwarps = (long long)gridDim.x * wpb;
    const long long Wn = ((long long)p.nv + 31) >> 5;  // used words per bitmap row
    if (gtid == 0) ctl->t0 = globaltimer();

    // ---- phase 0: P <- 0, F <- 0 --------------------------------------------
    {
        const long long n4 = (long long)p.nstates * p.W / 4;
        uint4* v4 = reinterpret_cast<uint4*>(p.visited);
        for (long long i = gtid; i < n4; i += gthreads) v4[i] = make_uint4(0, 0, 0, 0);
        for (int f = 0; f < 3; ++f) {
            uint4* f4 = reinterpret_cast<uint4*>(p.fb[f]);
            for (long long i = gtid; i < n4; i += gthreads) f4[i] = make_uint4(0, 0, 0, 0);
        }
    }
    __syncthreads();
    grid_sync(ctl, &s_view, [] {});

    // ---- seed: P = M = {(q_s, source)} (engine.py:106-109, :154-155) --------
    {
        unsigned long long nnew = 0, nedge = 0;
        if (blockIdx.x == 0 && wid == 0) {
            for (int i0 = 0; i0 < p.nstarts; i0 += 32) {
                const int i = i0 + lane;
                bool fresh = false;
                int q = 0;
                if (i < p.nstarts) {
                    q = S.starts[i];
                    const long long off = (long long)q * p.W + (p.source >> 5);
                    const uint32_t bit = 1u << (p.source & 31);
                    fresh = !(atomicOr(p.visited + off, bit) & bit);
                    if (fresh) atomicOr(p.fb[0] + off, bit);
                }
                nnew += fresh ? 1 : 0;
                count_state(s_state, fresh, q);
                const uint32_t T = emit_pairs(p, S, 0, fresh, q, p.source, lane);
                if (lane == 0) nedge += T;
            }
        }
        __syncthreads();
        flush_counts(ctl, 0, nnew, nedge, s_red, s_state, p.nstates);
    }
    grid_sync(ctl, &s_view, [&] { level_bookkeeping(p, S, 0); });

    // ---- level loop -----------------------------------------------------------
    for (int L = 0;; ++L) {
        if (s_view.done) break;
        const int cur = L & 1, nxt = cur ^ 1;
        const uint32_t* fcur = p.fb[L % 3];
        uint32_t* fnext = p.fb[(L + 1) % 3];

        if (s_view.dir == DIR_PUSH && s_view.plan) {
            // plan: emit F_L's row segments from its bitmap (after a pull level)
            for (int q = threadIdx.x; q < p.nstates; q += blockDim.x)
                s_active[q] = ld_volatile(&ctl->state_front[cur][q]) != 0;
            __syncthreads();
            unsigned long long nedge = 0;
            for (int q = 0; q < p.nstates; ++q) {
                if (!s_active[q] || S.gbeg[q + 1] == S.gbeg[q]) continue;
                const uint32_t* row = fcur + (long long)q * p.W;
                for (long long w0 = gwarp * 32; w0 < Wn; w0 += nwarps * 32) {
                    const long long wi = w0 + lane;
                    uint32_t bits = wi < Wn ? row[wi] : 0u;
                    unsigned any = __ballot_sync(FULL, bits != 0);
                    while (any) {
                        const int src_lane = __ffs(any) - 1;
                        any &= any - 1;
                        const uint32_t wb = __shfl_sync(FULL, bits, src_lane);
                        const bool valid = (wb >> lane) & 1u;
                        const int v = (int)((w0 + src_lane) * 32 + lane);
                        const uint32_t T = emit_pairs(p, S, cur, valid, q, v, lane);
                        if (lane == 0) nedge += T;
                    }
                }
            }
            flush_counts(ctl, cur, 0, nedge, s_red, s_state, 0);
            grid_sync(ctl, &s_view, [&] { plan_bookkeeping(p, L); });
            if (s_view.done) break;
        }

        // zero the bitmap level L+1 will write into F_{L+2}
        {
            uint4* z4 = reinterpret_cast<uint4*>(p.fb[(L + 2) % 3]);
            const long long n4 = (long long)p.nstates * p.W / 4;
            for (long long i = gtid; i < n4; i += gthreads) z4[i] = make_uint4(0, 0, 0, 0);
        }

        unsigned long long nnew = 0, nedge = 0;
        if (s_view.dir == DIR_PUSH) {
            // ---- push: expand the bundles of F_L's queue ------------------------
            if (threadIdx.x == 0) {
                unsigned long long run = 0;
                for (int s = 0; s <= kShards; ++s) {
                    s_bpre[s] = run;
                    const unsigned long long c = ld_volatile(&ctl->shard_cnt[cur][s]) & 0xFFFFFFFFull;
                    const unsigned long long cap = s < kShards ? p.shard_buncap : p.ovf_buncap;
                    run += c < cap ? c : cap;
                }
                s_bpre[kShards + 1] = run;
            }
            __syncthreads();
            const unsigned long long nb = s_bpre[kShards + 1];
            const uint2* bun = p.bun[cur];
            const uint2* seg = p.seg[cur];
            // CTA-major dealing: consecutive bundles (often one row) land on different SMs
            const unsigned long long step = (unsigned long long)gridDim.x * wpb;
            for (unsigned long long bi = (unsigned long long)wid * gridDim.x + blockIdx.x; bi < nb;
                 bi += step) {
                int s = 0;
#pragma unroll
                for (int h = 64; h >= 1; h >>= 1)
                    if (s + h <= kShards && s_bpre[s + h] <= bi) s += h;
                const uint2 bd = __ldcg(bun + (unsigned long long)s * p.shard_buncap + (bi - s_bpre[s]));
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
                const bool active = (uint32_t)lane < cnt;
                const int j = warp_upper_lane(excl, active ? (uint32_t)lane : 0u);
                const uint32_t sj = __shfl_sync(FULL, my_start, j);
                const uint32_t exj = __shfl_sync(FULL, excl, j);
                const int gj = (int)__shfl_sync(FULL, my_grp, j);
                int w = 0, t0 = 0, t1 = 0;
                if (active) {
                    const Slot sl = S.slots[S.gslot[gj]];
                    w = __ldg(sl.col + sj + ((uint32_t)lane - exj));
                    t0 = S.toff[gj];
                    t1 = S.toff[gj + 1];
                }
                for (int k = 0; k < p.maxT; ++k) {
                    bool fresh = false;
                    int q2 = 0;
                    if (active && t0 + k < t1) {
                        q2 = S.targets[t0 + k];
                        const long long off2 = (long long)q2 * p.W + (w >> 5);
                        const uint32_t bit = 1u << (w & 31);
                        if (!(p.visited[off2] & bit)) {
                            fresh = !(atomicOr(p.visited + off2, bit) & bit);
                            if (fresh) atomicOr(fnext + off2, bit);
                        }
                    }
                    nnew += fresh ? 1 : 0;
                    count_state(s_state, fresh, q2);
                    const uint32_t T = emit_pairs(p, S, nxt, fresh, q2, w, lane);
                    if (lane == 0) nedge += T;
                }
            }
        } else {
            // ---- pull: unvisited (q', w) scan A_s^T row w for a member of F_L[q]
            if (threadIdx.x == 0) {
                int n = 0;
                for (int q = 0; q < p.nstates; ++q)
                    s_active[q] = ld_volatile(&ctl->state_front[cur][q]) != 0;
                for (int q2 = 0; q2 < p.nstates; ++q2) {
                    bool any = false;
                    for (int k = S.ibeg[q2]; k < S.ibeg[q2 + 1]; ++k) any |= s_active[S.isrc[k]] != 0;
                    if (any) s_ptarget[n++] = q2;
                }
                s_nptarget = n;
            }
            __syncthreads();
            const long long ntask = (long long)s_nptarget * Wn;
            for (long long task = gwarp; task < ntask; task += nwarps) {
                const int q2 = s_ptarget[task / Wn];
                const long long word = task % Wn;
                const long long voff = (long long)q2 * p.W + word;
                const uint32_t vis = p.visited[voff];
                const int w = (int)(word * 32 + lane);
                const bool need = w < p.nv && !((vis >> lane) & 1u);
                if (__ballot_sync(FULL, need) == 0) continue;
                bool found = false;
                for (int k = S.ibeg[q2]; k < S.ibeg[q2 + 1]; ++k) {
                    const int q = S.isrc[k];
                    if (!s_active[q]) continue;
                    const bool look = need && !found;
                    if (__ballot_sync(FULL, look) == 0) break;
                    const Slot ps = S.slots[p.nslots + S.islot[k]];
                    const uint32_t* frow = fcur + (long long)q * p.W;
                    uint32_t lo = 0, hi = 0;
                    if (look) {
                        lo = __ldg(ps.rowptr + w);
                        hi = __ldg(ps.rowptr + w + 1);
                    }
                    // first kPullInline in-edges per lane, loads issued together
                    int u[kPullInline];
#pragma unroll
                    for (int i = 0; i < kPullInline; ++i)
                        u[i] = (look && lo + i < hi) ? __ldg(ps.col + lo + i) : -1;
#pragma unroll
                    for (int i = 0; i < kPullInline; ++i)
                        if (u[i] >= 0 && ((frow[u[i] >> 5] >> (u[i] & 31)) & 1u)) found = true;
                    // longer rows: the whole warp scans one row at a time
                    unsigned longrows = __ballot_sync(FULL, look && !found && hi - lo > kPullInline);
                    while (longrows) {
                        const int ln = __ffs(longrows) - 1;
                        longrows &= longrows - 1;
                        const uint32_t rlo = __shfl_sync(FULL, lo, ln) + kPullInline;
                        const uint32_t rhi = __shfl_sync(FULL, hi, ln);
                        bool hit = false;
                        for (uint32_t e = rlo; e < rhi; e += 32) {
                            bool h = false;
                            if (e + lane < rhi) {
                                const int uu = __ldg(ps.col + e + lane);
                                h = (frow[uu >> 5] >> (uu & 31)) & 1u;
                            }
                            if (__ballot_sync(FULL, h)) {
                                hit = true;
                                break;
                            }
                        }
                        if (hit && lane == ln) found = true;
                    }
                }
                const unsigned fmask = __ballot_sync(FULL, found);
                if (fmask) {
                    if (lane == 0) {
                        p.visited[voff] = vis | fmask;
                        fnext[voff] = fmask;
                        nnew += __popc(fmask);
                        atomicAdd(&s_state[q2], (unsigned)__popc(fmask));
                    }
                }
            }
        }
        flush_counts(ctl, nxt, nnew, nedge, s_red, s_state, p.nstates);
        grid_sync(ctl, &s_view, [&] { level_bookkeeping(p, S, L + 1); });
    }

    // ---- epilogue: answer = OR of P's rows at final states (engine.py:112-114)
    if (ld_volatile(&ctl->status) == 0) {
        unsigned long long cnt = 0;
        for (long long i = gtid; i < Wn; i += gthreads) {
            uint32_t acc = 0;
            for (int f = 0; f < p.nfinals; ++f) acc |= __ldcg(p.visited + (long long)S.finals[f] * p.W + i);
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
        // exact push-model TE = sum over (q, v) in P of the out-degrees of q's groups
        unsigned long long te = 0;
        if (p.count_te) {
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
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            cnt += __shfl_xor_sync(FULL, cnt, d);
            te += __shfl_xor_sync(FULL, te, d);
        }
        if (lane == 0 && cnt) atomicAdd(&ctl->reach_count, cnt);
        if (lane == 0 && te) atomicAdd(&ctl->te_exact, te);
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
