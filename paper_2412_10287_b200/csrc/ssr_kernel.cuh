// ssr_kernel.cuh -- the persistent sm_100a kernel that evaluates one
// single-source 2-RPQ: the reference's whole evaluator loop
//   P <- seed; while M: M <- (sum_a (N^a)^T x M x G^a) <not P>; P <- P + M
// (rpq/engine.py:146-171, Alg. 1) in ONE cooperative launch.
//
// Layout:
//   slot s    = (label, inverted) symbol; A_s = forward[l] or backward[l]
//               (graph_store.py:87-91) as uint32 row pointers + int32 columns;
//               A_s^T (the other direction) is what pull levels scan.
//   group g   = (state q, slot s) with targets {q' : q -s-> q'}: one row of
//               the transposed transition matrix (engine.py:102).
//   P         = |Q| bitmaps of |V| bits.
//   F_L       = 3 rotating bitmaps of the same shape (read L%3, write (L+1)%3,
//               zero (L+2)%3), plus the list of F_L's NON-EMPTY 32-bit WORDS:
//               whoever first sets a bit in a word of F_{L+1} appends the
//               word.  Push levels iterate that list, so sparse levels cost
//               O(|F|), and bitmaps give O(1) membership for pull levels.
//
// A level is one epoch (plus a chunk epoch when some rows are too long for
// one warp) and one grid barrier per epoch:
//   push: a warp takes 32 listed words, expands their set bits 32 frontier
//         items at a time -- row pointers of all groups in flight, then the
//         items' edges kEPL per lane -- and claims (q', w) with atomicOr on P.
//         Rows longer than kBigRow are cut into kChunk-edge chunks that every
//         warp shares in the chunk epoch.
//   pull: every unvisited (q', w) with a possible predecessor scans row w of
//         A_s^T for a member of F_L[q], early exit; rows longer than
//         kLongRow are chunked the same way.
// mask_complement + or_sum of the reference (engine.py:159, :165) are the
// atomicOr claim; np.unique's dedup (sparse_bool.py:250) is the bitmap.
// The direction of each level follows Beamer's rule on the exact out-edge
// count of the frontier (accumulated when pairs are discovered).
#pragma once

namespace rpqk {

constexpr int kThreads = 1024;       // 32 warps per CTA, one CTA per SM
constexpr int kMinBlocks = 1;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCtas = 160;
constexpr int kMaxStates = 256;
constexpr int kMaxGroups = 256;
constexpr int kMaxSlots = 128;
constexpr int kFastGroups = 4;       // groups per state expanded with all loads in flight
constexpr int kEPL = 4;              // push: edges per lane per sub-round
constexpr uint32_t kBigRow = 32;     // push rows longer than this become chunks
constexpr uint32_t kChunk = 512;     // edges per chunk
constexpr int kPullVerts = 4;        // pull: words (x32 vertices) per warp task
constexpr int kPullInline = 2;       // in-edges each lane tests first
constexpr int kPullStep = 4;         // in-edges per lane per medium-row step
constexpr uint32_t kLongRow = 32;    // pull rows longer than this (after inline) become chunks
constexpr unsigned FULL = 0xffffffffu;

constexpr int ST_OVERFLOW = 100;
constexpr int ST_DEADLOCK = 101;

constexpr int DIR_PUSH = 0;
constexpr int DIR_PULL = 1;

struct Slot {
    const uint32_t* rowptr;
    const int32_t* col;
};

// Per-frontier counters, rotating over 3 sets by level: the set of F_L is
// produced during level L-1, read by every CTA after the barrier that ends
// level L-1, and reset by CTA 0 during level L+1.  Every CTA reads the same
// values and so takes the same decisions: no serial section, no broadcast.
struct LCnt {
    unsigned long long nnew;      // |F_L|
    unsigned long long mf;        // sum over F_L of out-degree x targets (TE share)
    unsigned long long wl_ovf;    // entries in the word list's overflow region
    unsigned long long ch_ovf;    // chunks in the chunk buffer's overflow region
    unsigned int overflow;
    unsigned int expire;          // 1 + level whose deadline check failed
    unsigned int wl_cta[kMaxCtas];  // word-list fill of each CTA's region
    unsigned int ch_cta[kMaxCtas];  // chunk fill of each CTA's region
    unsigned int state[kMaxStates]; // |F_L| per state
};

struct Ctl {
    unsigned int bar;  // monotonic barrier arrivals
    int abort;
    unsigned long long t0;
    LCnt lc[3];
    // results, written by CTA 0 only
    int status;
    int iterations;
    int levels;
    int pull_levels;
    unsigned long long te;
    unsigned long long chunks;
    unsigned long long pairs;
    unsigned long long reach_count;
    long long level_new[64];
    long long level_edges[64];
    unsigned long long level_ns[64];
    unsigned long long work_ns[64];  // latest CTA finishing level L's main epoch (from t0)
    unsigned long long bar_ns[64];   // CTA 0 past the last barrier of level L
    int level_dir[64];
};

struct Params {
    const int32_t* tables;
    const Slot* slots;  // A_s, then A_s^T at [nslots, 2*nslots)
    const unsigned long long* slot_nnz;
    uint32_t* visited;
    uint32_t* fb[3];
    uint2* wl[2];       // word lists {q, word} by level parity
    uint4* chunks;      // long-row chunks of the current level (CTA regions + overflow)
    Ctl* ctl;
    uint8_t* reach;
    unsigned long long wl_cap;      // entries per CTA region
    unsigned long long wl_ovf_cap;  // entries in the overflow region
    unsigned long long ch_cap;      // chunks per CTA region
    unsigned long long ch_ovf_cap;  // chunks in the overflow region
    unsigned long long budget_ns;
    long long W;  // words per bitmap row (multiple of 4)
    int nv;
    int nstates, ngroups, nslots, ntargets, nstarts, nfinals, nin;
    int maxT;
    int source;
    int table_ints;
    int dir_mode;  // 0 auto, 1 push only, 2 pull only
    int count_te;  // kept for the ABI; TE is always exact now
    float alpha;   // pull when m_f * alpha > m_u
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

// What every thread of a CTA needs after a barrier (warp 0 derives it from
// the global counters; every CTA derives the same values).
struct View {
    int done;
    int dir;
    int status;
    int iterations;
    unsigned long long nwl;  // F_L's listed words (regions + overflow)
};

// Grid barrier for a cooperative launch over a monotonic arrival counter:
// barrier number e completes when e * gridDim.x arrivals are counted.
// Waiters spin on a relaxed load and fence once afterwards (acquire side; the
// fence also invalidates this SM's L1: CCTL.IVALL).
__device__ __forceinline__ void grid_barrier(Ctl* ctl, unsigned epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&ctl->bar, 1u);
        const unsigned target = epoch * gridDim.x;
        unsigned long long ts = 0;
        unsigned spins = 0;
        while (ld_relaxed_u32(&ctl->bar) < target) {
            __nanosleep(16);
            if ((++spins & 4095u) == 0) {
                const unsigned long long now = globaltimer();
                if (ts == 0) {
                    ts = now;
                } else if (now - ts > 20000000000ull) {  // 20 s: cannot happen co-resident
                    atomicExch(&ctl->abort, 1);
                    break;
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Per-CTA context of the frontier being built.
struct Ctx {
    LCnt* lc;           // counters of F_{L+1}
    uint2* wl;          // its word list
    uint32_t* fnext;    // its bitmap
    unsigned* s_wl;     // this CTA's word-list fill (smem)
    unsigned* s_ch;     // this CTA's chunk fill (smem)
    unsigned* s_state;  // this CTA's discoveries per state (smem)
};

// Warp-cooperative append of up to N (q, word) entries per lane (app[i]) to
// the word list: the CTA's region first, the overflow region for what does
// not fit.  One shared-memory atomic per call.
template <int N>
__device__ __forceinline__ void wl_append(const Params& p, const Ctx& c, const bool* app, const int* q,
                                          const int* w, int lane) {
    unsigned mine = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) mine += app[i] ? 1u : 0u;
    const unsigned incl = warp_incl_scan(mine, lane);
    const unsigned n = __shfl_sync(FULL, incl, 31);
    if (n == 0) return;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(c.s_wl, n);
    base = __shfl_sync(FULL, base, 0);
    const unsigned long long cap = p.wl_cap;
    const unsigned fit = base >= cap ? 0u : (unsigned)min((unsigned long long)n, cap - base);
    unsigned long long ob = 0;
    if (fit < n) {
        if (lane == 0) ob = atomicAdd(&c.lc->wl_ovf, (unsigned long long)(n - fit));
        ob = __shfl_sync(FULL, ob, 0);
        if (ob + (n - fit) > p.wl_ovf_cap) {
            if (lane == 0) atomicExch(&c.lc->overflow, 1u);
            return;
        }
    }
    unsigned r = incl - mine;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (!app[i]) continue;
        const uint2 ent = make_uint2((uint32_t)q[i], (uint32_t)(w[i] >> 5));
        if (r < fit)
            c.wl[(unsigned long long)blockIdx.x * cap + base + r] = ent;
        else
            c.wl[(unsigned long long)kMaxCtas * cap + ob + (r - fit)] = ent;
        ++r;
    }
}

// Out-degree x targets of (q[i], w[i]) over their groups, for N pairs per
// lane (q < 0: none), with every row-pointer load in flight together: each
// pair's share of TE / m_f.
template <int N>
__device__ __forceinline__ unsigned long long out_edges(const Smem& S, const int* q, const int* w) {
    unsigned long long s = 0;
    int ng[N];
    int maxg = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        ng[i] = q[i] >= 0 ? S.gbeg[q[i] + 1] - S.gbeg[q[i]] : 0;
        maxg = max(maxg, ng[i]);
    }
    constexpr int G = 2;  // groups per batch (register budget)
    for (int k0 = 0; k0 < maxg; k0 += G) {
        uint32_t lo[N][G], hi[N][G];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int k = 0; k < G; ++k) {
                lo[i][k] = hi[i][k] = 0;
                if (k0 + k < ng[i]) {
                    const Slot sl = S.slots[S.gslot[S.gbeg[q[i]] + k0 + k]];
                    lo[i][k] = __ldg(sl.rowptr + w[i]);
                    hi[i][k] = __ldg(sl.rowptr + w[i] + 1);
                }
            }
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int k = 0; k < G; ++k)
                if (k0 + k < ng[i]) {
                    const int g = S.gbeg[q[i]] + k0 + k;
                    s += (unsigned long long)(hi[i][k] - lo[i][k]) * (unsigned long long)(S.toff[g + 1] - S.toff[g]);
                }
    }
    return s;
}

// Bookkeeping of freshly claimed pairs (N per lane, fresh[i]): F bit (and a
// word-list entry when the word was empty), counts, out-edge total.  With
// set_f false the caller already wrote F and tells which words to list.
template <int N>
__device__ __forceinline__ void record_fresh(const Params& p, const Smem& S, const Ctx& c, const bool* fresh,
                                             const int* q, const int* w, int lane, unsigned long long& nnew,
                                             unsigned long long& mf) {
    bool app[N];
    int qq[N];
    uint32_t old[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        old[i] = 1;
        if (fresh[i]) old[i] = atomicOr(c.fnext + (long long)q[i] * p.W + (w[i] >> 5), 1u << (w[i] & 31));
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        app[i] = fresh[i] && old[i] == 0;
        qq[i] = fresh[i] ? q[i] : -1;
        if (fresh[i]) {
            nnew += 1;
            atomicAdd(&c.s_state[q[i]], 1u);
        }
    }
    mf += out_edges<N>(S, qq, w);
    wl_append<N>(p, c, app, q, w, lane);
}

// Claim every (target of group g[u], w[u]) not yet in P; kEPL edges per lane
// (g < 0: no edge).  Probes, claims and bookkeeping each keep all kEPL
// operations in flight.
__device__ __forceinline__ void claim_edges(const Params& p, const Smem& S, const Ctx& c, const int* w,
                                            const int* g, int lane, unsigned long long& nnew,
                                            unsigned long long& mf) {
    for (int k = 0; k < p.maxT; ++k) {
        uint32_t old[kEPL];
        int q2[kEPL];
#pragma unroll
        for (int u = 0; u < kEPL; ++u) {
            q2[u] = -1;
            old[u] = 0xFFFFFFFFu;
            if (g[u] >= 0) {
                const int t0 = S.toff[g[u]];
                if (t0 + k < S.toff[g[u] + 1]) {
                    q2[u] = S.targets[t0 + k];
                    old[u] = p.visited[(long long)q2[u] * p.W + (w[u] >> 5)];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kEPL; ++u) {
            const uint32_t bit = 1u << (w[u] & 31);
            if (q2[u] >= 0 && !(old[u] & bit))
                old[u] = atomicOr(p.visited + (long long)q2[u] * p.W + (w[u] >> 5), bit);
            else
                old[u] = 0xFFFFFFFFu;
        }
        bool fresh[kEPL];
#pragma unroll
        for (int u = 0; u < kEPL; ++u) fresh[u] = q2[u] >= 0 && !(old[u] & (1u << (w[u] & 31)));
        if (__any_sync(FULL, fresh[0] || fresh[1] || fresh[2] || fresh[3]))
            record_fresh<kEPL>(p, S, c, fresh, q2, w, lane, nnew, mf);
    }
}

// Warp-cooperative append of the kChunk-edge chunks of long rows (lanes with
// `big`): the CTA's region first, the overflow region for what does not fit.
__device__ __forceinline__ void add_chunks(const Params& p, const Ctx& c, bool big, uint32_t start, uint32_t len,
                                           uint32_t a, uint32_t b, int lane) {
    if (!__any_sync(FULL, big)) return;
    const unsigned mine = big ? (len + kChunk - 1) / kChunk : 0u;
    const unsigned incl = warp_incl_scan(mine, lane);
    const unsigned n = __shfl_sync(FULL, incl, 31);
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(c.s_ch, n);
    base = __shfl_sync(FULL, base, 0);
    const unsigned long long cap = p.ch_cap;
    const unsigned fit = base >= cap ? 0u : (unsigned)min((unsigned long long)n, cap - base);
    unsigned long long ob = 0;
    if (fit < n) {
        if (lane == 0) ob = atomicAdd(&c.lc->ch_ovf, (unsigned long long)(n - fit));
        ob = __shfl_sync(FULL, ob, 0);
        if (ob + (n - fit) > p.ch_ovf_cap) {
            if (lane == 0) atomicExch(&c.lc->overflow, 1u);
            return;
        }
    }
    unsigned r = incl - mine;
    for (unsigned i = 0; i < mine; ++i, ++r) {
        const uint32_t off = i * kChunk;
        const uint4 ent = make_uint4(start + off, min(kChunk, len - off), a, b);
        if (r < fit)
            p.chunks[(unsigned long long)blockIdx.x * cap + base + r] = ent;
        else
            p.chunks[(unsigned long long)kMaxCtas * cap + ob + (r - fit)] = ent;
    }
}

// End-of-epoch flush of a CTA's counts: one atomic per CTA and counter, and
// the CTA's word-list fill.  Call after __syncthreads().
__device__ __forceinline__ void flush_counts(const Ctx& c, unsigned long long nnew, unsigned long long mf,
                                             unsigned long long* red, int nstates) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    nnew = warp_sum_u64(nnew);
    mf = warp_sum_u64(mf);
    if (lane == 0) {
        red[2 * wid] = nnew;
        red[2 * wid + 1] = mf;
    }
    __syncthreads();
    if (wid == 0) {
        unsigned long long a = lane < kWarps ? red[2 * lane] : 0ull;
        unsigned long long b = lane < kWarps ? red[2 * lane + 1] : 0ull;
        a = warp_sum_u64(a);
        b = warp_sum_u64(b);
        if (lane == 0) {
            if (a) atomicAdd(&c.lc->nnew, a);
            if (b) atomicAdd(&c.lc->mf, b);
            c.lc->wl_cta[blockIdx.x] = *c.s_wl;
            c.lc->ch_cta[blockIdx.x] = *c.s_ch;
        }
    }
    for (int q = threadIdx.x; q < nstates; q += blockDim.x) {
        const unsigned int v = c.s_state[q];
        if (v) {
            atomicAdd(&c.lc->state[q], v);
            c.s_state[q] = 0;
        }
    }
}

// Exclusive prefix of per-CTA region fills (clamped to the region capacity)
// into s_pre[0..gridDim.x]; returns the total.  Warp-cooperative.
__device__ __forceinline__ unsigned region_prefix(const unsigned* fill, unsigned long long cap, unsigned* s_pre,
                                                  int lane) {
    constexpr int R = (kMaxCtas + 31) / 32;
    unsigned cnt[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int cc = 32 * r + lane;
        cnt[r] = cc < (int)gridDim.x ? (unsigned)min((unsigned long long)ldcg(&fill[cc]), cap) : 0u;
    }
    unsigned carry = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int cc = 32 * r + lane;
        const unsigned incl = warp_incl_scan(cnt[r], lane);
        if (cc <= (int)gridDim.x) s_pre[cc] = carry + incl - cnt[r];
        carry += __shfl_sync(FULL, incl, 31);
    }
    return carry;
}

// Region holding global index idx < s_pre[gridDim.x] (binary search in smem).
__device__ __forceinline__ int region_of(const unsigned* s_pre, unsigned long long idx) {
    int r = 0;
#pragma unroll
    for (int h = 128; h >= 1; h >>= 1)
        if (r + h < (int)gridDim.x && s_pre[r + h] <= idx) r += h;
    return r;
}

// Decision after F_L has been built (warp 0 of every CTA; every CTA reads the
// same counters and reaches the same result).  Mirrors the masked loop
// (engine.py:156-160): run while the frontier is non-empty, check the
// deadline, then step; and picks the direction of level L.
__device__ void decide_level(const Params& p, const Smem& S, int L, int lane, View* v, unsigned* s_wpre,
                             unsigned long long* s_sv, unsigned int* s_front) {
    Ctl* ctl = p.ctl;
    const LCnt* lc = &ctl->lc[L % 3];
    const unsigned long long nnew = ldcg(&lc->nnew);
    const unsigned long long mf = ldcg(&lc->mf);
    const unsigned long long wovf = ldcg(&lc->wl_ovf);
    const unsigned int overflow = ldcg(&lc->overflow);
    const unsigned int expire = ldcg(&lc->expire);
    const int abort = ldcg(&ctl->abort);
    const unsigned carry = region_prefix(lc->wl_cta, p.wl_cap, s_wpre, lane);
    for (int q = lane; q < p.nstates; q += 32) {
        const unsigned int f = ldcg(&lc->state[q]);
        s_front[q] = f;
        s_sv[q] += f;
    }
    __syncwarp();
    int done = 0, iterations = 0, status = 0, next = DIR_PUSH;
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
    } else if (mf == 0) {
        iterations = L + 1;  // nothing to expand: the next step is empty
        done = 1;
    } else {
        if (p.dir_mode == 2) {
            next = DIR_PULL;
        } else if (p.dir_mode == 0) {
            // m_u: in-edges of unvisited targets whose source state has a
            // frontier.  Pull when m_f * alpha > m_u (Beamer's rule).
            const double nv = (double)p.nv;
            double mu = 0.0;
            for (int q = lane; q < p.nstates; q += 32) {
                const double unvis = nv - (double)s_sv[q];
                for (int k = S.ibeg[q]; k < S.ibeg[q + 1]; ++k)
                    if (s_front[S.isrc[k]]) mu += (double)p.slot_nnz[S.islot[k]] * unvis / nv;
            }
            mu = warp_sum_f64(mu);
            next = ((double)mf * (double)p.alpha > mu) ? DIR_PULL : DIR_PUSH;
        }
    }
    if (lane == 0) {
        v->done = done;
        v->dir = next;
        v->status = status;
        v->iterations = iterations;
        v->nwl = (unsigned long long)carry + wovf;
        if (blockIdx.x == 0) {  // results and statistics
            const unsigned long long now = globaltimer();
            ctl->pairs += nnew;
            if (nnew && !status) ctl->te += mf;
            if (L < 64) {
                ctl->level_new[L] = (long long)nnew;
                ctl->level_ns[L] = now - ctl->t0;
                ctl->level_edges[L] = (long long)mf;
                ctl->level_dir[L] = next;
            }
            if (!done) {
                if (L > 0) ctl->levels = L;
                if (next == DIR_PULL) ctl->pull_levels += 1;
                // _Clock.check at the top of iteration L (engine.py:87-89):
                // recorded now, acted upon at the next decision by every CTA
                if (now - ctl->t0 > p.budget_ns) ctl->lc[(L + 1) % 3].expire = (unsigned)L + 1;
            } else {
                ctl->status = status;
                ctl->iterations = iterations;
            }
        }
    }
}

__device__ __forceinline__ void reset_lc(LCnt* lc, int tid) {
    for (int i = tid; i < kMaxCtas; i += kThreads) {
        lc->wl_cta[i] = 0;
        lc->ch_cta[i] = 0;
    }
    for (int i = tid; i < kMaxStates; i += kThreads) lc->state[i] = 0;
    if (tid == 0) {
        lc->nnew = 0;
        lc->mf = 0;
        lc->wl_ovf = 0;
        lc->ch_ovf = 0;
        lc->overflow = 0;
        lc->expire = 0;
    }
}

// One pull scan of a medium row / chunk: any member of F (bitmap row frow)
// among col[lo, hi)?  Warp-cooperative, 128 columns per step.
__device__ __forceinline__ bool warp_row_hit(const int32_t* col, uint32_t lo, uint32_t hi, const uint32_t* frow,
                                             int lane) {
    for (uint32_t ed = lo; ed < hi; ed += 128) {
        int uu[4];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) uu[cc] = ed + 32 * cc + lane < hi ? __ldg(col + ed + 32 * cc + lane) : -1;
        bool h = false;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
            if (uu[cc] >= 0) h |= (frow[uu[cc] >> 5] >> (uu[cc] & 31)) & 1u;
        if (__ballot_sync(FULL, h)) return true;
    }
    return false;
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) ssr_kernel(Params p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_red[2 * kWarps];
    __shared__ unsigned s_wpre[kMaxCtas + 1];       // F_L's word-list prefix over CTA regions
    __shared__ unsigned long long s_sv[kMaxStates];  // |P| per state (same in every CTA)
    __shared__ unsigned int s_front[kMaxStates];     // |F_L| per state
    __shared__ unsigned int s_state[kMaxStates];     // this CTA's discoveries per state
    __shared__ int s_ptarget[kMaxStates];            // pull target states of this level
    __shared__ int s_nptarget;
    __shared__ unsigned s_wl;                        // this CTA's word-list fill
    __shared__ unsigned s_ch;                        // this CTA's chunk fill
    __shared__ unsigned s_cpre[kMaxCtas + 1];        // chunk prefix over CTA regions
    __shared__ unsigned long long s_nch;
    __shared__ unsigned s_task;                      // push: next task in this CTA's range
    __shared__ View s_view;

    Slot* s_slots = reinterpret_cast<Slot*>(smem_raw);
    int32_t* s_tab = reinterpret_cast<int32_t*>(smem_raw + sizeof(Slot) * 2 * p.nslots);
    for (int i = threadIdx.x; i < 2 * p.nslots; i += blockDim.x) s_slots[i] = p.slots[i];
    for (int i = threadIdx.x; i < p.table_ints; i += blockDim.x) s_tab[i] = p.tables[i];
    for (int i = threadIdx.x; i < kMaxStates; i += blockDim.x) {
        s_state[i] = 0;
        s_sv[i] = 0;
        s_front[i] = 0;
    }
    if (threadIdx.x == 0) s_wl = s_ch = 0;
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
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long gthreads = (long long)gridDim.x * blockDim.x;
    const long long gwarp = (long long)blockIdx.x * kWarps + wid;
    const long long nwarps = (long long)gridDim.x * kWarps;
    const long long Wn = ((long long)p.nv + 31) >> 5;  // used words per bitmap row
    const long long nbits4 = (long long)p.nstates * p.W / 4;
    const bool cta0 = blockIdx.x == 0;
    if (gtid == 0) ctl->t0 = globaltimer();

    unsigned e = 0;  // barriers passed

    // ---- epoch 0: P <- 0, F <- 0 --------------------------------------------
    {
        uint4* v4 = reinterpret_cast<uint4*>(p.visited);
        for (long long i = gtid; i < nbits4; i += gthreads) v4[i] = make_uint4(0, 0, 0, 0);
        for (int f = 0; f < 3; ++f) {
            uint4* f4 = reinterpret_cast<uint4*>(p.fb[f]);
            for (long long i = gtid; i < nbits4; i += gthreads) f4[i] = make_uint4(0, 0, 0, 0);
        }
    }
    grid_barrier(ctl, ++e);

    // ---- epoch 1: seed F_0 = P = {(q_s, source)} (engine.py:106-109, :154-155)
    {
        const Ctx c{&ctl->lc[0], p.wl[0], p.fb[0], &s_wl, &s_ch, s_state};
        unsigned long long nnew = 0, mf = 0;
        if (cta0 && wid == 0) {
            for (int i0 = 0; i0 < p.nstarts; i0 += 32) {
                const int i = i0 + lane;
                bool fresh = false;
                int q = 0;
                if (i < p.nstarts) {
                    q = S.starts[i];
                    const uint32_t bit = 1u << (p.source & 31);
                    fresh = !(atomicOr(p.visited + (long long)q * p.W + (p.source >> 5), bit) & bit);
                }
                const bool fa[1] = {fresh};
                const int qa[1] = {q}, wa[1] = {p.source};
                record_fresh<1>(p, S, c, fa, qa, wa, lane, nnew, mf);
            }
        }
        __syncthreads();
        flush_counts(c, nnew, mf, s_red, p.nstates);
    }
    grid_barrier(ctl, ++e);
    if (wid == 0) decide_level(p, S, 0, lane, &s_view, s_wpre, s_sv, s_front);
    __syncthreads();

    // ---- level loop -----------------------------------------------------------
    int L = 0;
    for (;;) {
        if (s_view.done) break;
        const int dir = s_view.dir;
        const uint32_t* fcur = p.fb[L % 3];
        const Ctx c{&ctl->lc[(L + 1) % 3], p.wl[(L + 1) & 1], p.fb[(L + 1) % 3], &s_wl, &s_ch, s_state};
        if (threadIdx.x == 0) s_wl = s_ch = s_task = 0;
        if (cta0) reset_lc(&ctl->lc[(L + 2) % 3], threadIdx.x);
        {  // zero the bitmap level L+1 will write F_{L+2} into
            uint4* z4 = reinterpret_cast<uint4*>(p.fb[(L + 2) % 3]);
            for (long long i = gtid; i < nbits4; i += gthreads) z4[i] = make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
        unsigned long long nnew = 0, mf = 0;

        if (dir == DIR_PUSH) {
            // ---- push: expand the set bits of F_L's listed words -------------
            const unsigned long long nwl = s_view.nwl;
            const unsigned nreg = s_wpre[gridDim.x];
            const uint2* wl = p.wl[L & 1];
            // words per warp task: enough tasks for every warp while the list is short
            // the list is split into one contiguous range per CTA; the CTA's
            // warps take `span`-word tasks from it through a shared counter
            unsigned span = 8;
            while (span > 1 && (unsigned long long)span * nwarps > nwl) span >>= 1;
            const unsigned long long per_cta = (nwl + gridDim.x - 1) / gridDim.x;
            const unsigned long long r_lo = min(nwl, per_cta * blockIdx.x);
            const unsigned long long r_hi = min(nwl, r_lo + per_cta);
            for (;;) {
                unsigned long long c0 = 0;
                if (lane == 0) c0 = r_lo + (unsigned long long)atomicAdd(&s_task, span);
                c0 = __shfl_sync(FULL, c0, 0);
                if (c0 >= r_hi) break;
                const unsigned long long idx = c0 + lane;
                int q = 0;
                uint32_t word = 0, bits = 0;
                if ((unsigned)lane < span && idx < r_hi) {
                    uint2 ent;
                    if (idx < nreg) {
                        const int r = region_of(s_wpre, idx);
                        ent = __ldcg(wl + (unsigned long long)r * p.wl_cap + (idx - s_wpre[r]));
                    } else {
                        ent = __ldcg(wl + (unsigned long long)kMaxCtas * p.wl_cap + (idx - nreg));
                    }
                    q = (int)ent.x;
                    word = ent.y;
                    bits = fcur[(long long)q * p.W + word];
                }
                const uint32_t pc = __popc(bits);
                const uint32_t iincl = warp_incl_scan(pc, lane);
                const uint32_t iexcl = iincl - pc;
                const uint32_t NI = __shfl_sync(FULL, iincl, 31);
                for (uint32_t r0 = 0; r0 < NI; r0 += 32) {
                    // one frontier item (q, v) per lane
                    const uint32_t t = r0 + lane;
                    const bool act = t < NI;
                    const int j = warp_upper_lane(iexcl, act ? t : 0u);
                    const uint32_t bj = __shfl_sync(FULL, bits, j);
                    const int qv = __shfl_sync(FULL, q, j);
                    const uint32_t wj = __shfl_sync(FULL, word, j);
                    const uint32_t ej = __shfl_sync(FULL, iexcl, j);
                    const int v = act ? (int)(wj * 32 + __fns(bj, 0, (int)(t - ej) + 1)) : 0;
                    const int ng = act ? S.gbeg[qv + 1] - S.gbeg[qv] : 0;
                    int maxng = ng;
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) maxng = max(maxng, __shfl_xor_sync(FULL, maxng, d));
                    for (int k0 = 0; k0 < maxng; k0 += kFastGroups) {
                        // row pointers of up to kFastGroups groups in flight together
                        uint32_t lo[kFastGroups], deg[kFastGroups];
                        int g[kFastGroups];
#pragma unroll
                        for (int k = 0; k < kFastGroups; ++k) {
                            lo[k] = deg[k] = 0;
                            g[k] = -1;
                            if (k0 + k < ng) {
                                g[k] = S.gbeg[qv] + k0 + k;
                                const Slot sl = S.slots[S.gslot[g[k]]];
                                lo[k] = __ldg(sl.rowptr + v);
                                deg[k] = __ldg(sl.rowptr + v + 1);
                            }
                        }
#pragma unroll
                        for (int k = 0; k < kFastGroups; ++k) {
                            deg[k] -= lo[k];
                            if (k0 + k >= maxng) continue;
                            const bool big = deg[k] > kBigRow;  // long row: chunks for the chunk epoch
                            add_chunks(p, c, big, lo[k], deg[k], (uint32_t)g[k], 0u, lane);
                            if (big) deg[k] = 0;
                        }
#pragma unroll
                        for (int k = 0; k < kFastGroups; ++k) {
                            if (k0 + k >= maxng) break;
                            const uint32_t dincl = warp_incl_scan(deg[k], lane);
                            const uint32_t dexcl = dincl - deg[k];
                            const uint32_t T = __shfl_sync(FULL, dincl, 31);
                            for (uint32_t e0 = 0; e0 < T; e0 += 32 * kEPL) {
                                int w[kEPL], gg[kEPL];
#pragma unroll
                                for (int u = 0; u < kEPL; ++u) {
                                    const uint32_t ed = e0 + 32 * u + lane;
                                    const bool a = ed < T;
                                    const int jj = warp_upper_lane(dexcl, a ? ed : 0u);
                                    const uint32_t loj = __shfl_sync(FULL, lo[k], jj);
                                    const uint32_t exj = __shfl_sync(FULL, dexcl, jj);
                                    const int gj = __shfl_sync(FULL, g[k], jj);
                                    gg[u] = a ? gj : -1;
                                    w[u] = a ? __ldg(S.slots[S.gslot[gj]].col + loj + (ed - exj)) : 0;
                                }
                                claim_edges(p, S, c, w, gg, lane, nnew, mf);
                            }
                        }
                    }
                }
            }
        } else {
            // ---- pull: unvisited (q', w) scan A_s^T row w for a member of F_L[q]
            if (threadIdx.x == 0) {
                int n = 0;
                for (int q2 = 0; q2 < p.nstates; ++q2) {
                    bool any = false;
                    for (int k = S.ibeg[q2]; k < S.ibeg[q2 + 1]; ++k) any |= s_front[S.isrc[k]] != 0;
                    if (any) s_ptarget[n++] = q2;
                }
                s_nptarget = n;
            }
            __syncthreads();
            const long long nblk = (Wn + kPullVerts - 1) / kPullVerts;
            const long long ntask = (long long)s_nptarget * nblk;
            for (long long task = gwarp; task < ntask; task += nwarps) {
                const int q2 = s_ptarget[task / nblk];
                const long long word0 = (task % nblk) * kPullVerts;
                uint32_t vis[kPullVerts];
                bool need[kPullVerts], found[kPullVerts];
                int w[kPullVerts];
#pragma unroll
                for (int u = 0; u < kPullVerts; ++u)
                    vis[u] = word0 + u < Wn ? p.visited[(long long)q2 * p.W + word0 + u] : 0xFFFFFFFFu;
                bool any_need = false;
#pragma unroll
                for (int u = 0; u < kPullVerts; ++u) {
                    w[u] = (int)((word0 + u) * 32 + lane);
                    need[u] = w[u] < p.nv && !((vis[u] >> lane) & 1u);
                    found[u] = false;
                    any_need |= need[u];
                }
                if (__ballot_sync(FULL, any_need) == 0) continue;
                for (int k = S.ibeg[q2]; k < S.ibeg[q2 + 1]; ++k) {
                    const int q = S.isrc[k];
                    if (!s_front[q]) continue;
                    bool look[kPullVerts], any_look = false;
#pragma unroll
                    for (int u = 0; u < kPullVerts; ++u) {
                        look[u] = need[u] && !found[u];
                        any_look |= look[u];
                    }
                    if (__ballot_sync(FULL, any_look) == 0) break;
                    const Slot ps = S.slots[p.nslots + S.islot[k]];
                    const uint32_t* frow = fcur + (long long)q * p.W;
                    uint32_t lo[kPullVerts], hi[kPullVerts];
#pragma unroll
                    for (int u = 0; u < kPullVerts; ++u) {
                        lo[u] = look[u] ? __ldg(ps.rowptr + w[u]) : 0u;
                        hi[u] = look[u] ? __ldg(ps.rowptr + w[u] + 1) : 0u;
                    }
                    // the first kPullInline in-edges of every vertex, all loads in flight
                    int cand[kPullVerts][kPullInline];
#pragma unroll
                    for (int u = 0; u < kPullVerts; ++u)
#pragma unroll
                        for (int i = 0; i < kPullInline; ++i)
                            cand[u][i] = (lo[u] + i < hi[u]) ? __ldg(ps.col + lo[u] + i) : -1;
                    uint32_t fw[kPullVerts][kPullInline];
#pragma unroll
                    for (int u = 0; u < kPullVerts; ++u)
#pragma unroll
                        for (int i = 0; i < kPullInline; ++i)
                            fw[u][i] = cand[u][i] >= 0 ? frow[cand[u][i] >> 5] : 0u;
#pragma unroll
                    for (int u = 0; u < kPullVerts; ++u)
#pragma unroll
                        for (int i = 0; i < kPullInline; ++i)
                            if (cand[u][i] >= 0 && ((fw[u][i] >> (cand[u][i] & 31)) & 1u)) found[u] = true;
                    // the rest of the row: long rows become chunks; medium rows
                    // are scanned by their own lane, kPullStep columns of every
                    // vertex in flight per step, early exit
                    bool medium[kPullVerts];
                    uint32_t pos[kPullVerts];
#pragma unroll
                    for (int u = 0; u < kPullVerts; ++u) {
                        const bool more = look[u] && !found[u] && hi[u] - lo[u] > kPullInline;
                        const bool longrow = more && hi[u] - lo[u] - kPullInline > kLongRow;
                        add_chunks(p, c, longrow, lo[u] + kPullInline, hi[u] - lo[u] - kPullInline, (uint32_t)w[u],
                                   ((uint32_t)q2 << 16) | (uint32_t)k, lane);
                        medium[u] = more && !longrow;
                        pos[u] = lo[u] + kPullInline;
                    }
                    for (;;) {
                        bool any = false;
#pragma unroll
                        for (int u = 0; u < kPullVerts; ++u) any |= medium[u];
                        if (!any) break;
                        int cc[kPullVerts][kPullStep];
#pragma unroll
                        for (int u = 0; u < kPullVerts; ++u)
#pragma unroll
                            for (int i = 0; i < kPullStep; ++i)
                                cc[u][i] = medium[u] && pos[u] + i < hi[u] ? __ldg(ps.col + pos[u] + i) : -1;
#pragma unroll
                        for (int u = 0; u < kPullVerts; ++u) {
                            if (!medium[u]) continue;
#pragma unroll
                            for (int i = 0; i < kPullStep; ++i)
                                if (cc[u][i] >= 0 && ((frow[cc[u][i] >> 5] >> (cc[u][i] & 31)) & 1u)) found[u] = true;
                            pos[u] += kPullStep;
                            if (found[u] || pos[u] >= hi[u]) medium[u] = false;
                        }
                    }
                }
                bool app[kPullVerts];
                int qa[kPullVerts], qf[kPullVerts];
#pragma unroll
                for (int u = 0; u < kPullVerts; ++u) {
                    const unsigned fmask = __ballot_sync(FULL, found[u]);
                    app[u] = fmask != 0 && lane == 0;
                    qa[u] = q2;
                    qf[u] = found[u] ? q2 : -1;
                    if (app[u]) {  // this warp owns the word: plain stores
                        const long long voff = (long long)q2 * p.W + word0 + u;
                        p.visited[voff] = vis[u] | fmask;
                        c.fnext[voff] = fmask;
                        nnew += __popc(fmask);
                        atomicAdd(&c.s_state[q2], (unsigned)__popc(fmask));
                    }
                }
                if (__any_sync(FULL, found[0] || found[1] || found[2] || found[3])) {
                    mf += out_edges<kPullVerts>(S, qf, w);
                    wl_append<kPullVerts>(p, c, app, qa, w, lane);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && L < 64) atomicMax(&ctl->work_ns[L], globaltimer() - ctl->t0);
        flush_counts(c, nnew, mf, s_red, p.nstates);
        grid_barrier(ctl, ++e);

        // ---- chunk epoch: long rows cut into kChunk-edge pieces, all warps ----
        if (wid == 0) {
            const unsigned reg = region_prefix(c.lc->ch_cta, p.ch_cap, s_cpre, lane);
            const unsigned long long ovf = min(ldcg(&c.lc->ch_ovf), p.ch_ovf_cap);
            if (lane == 0) s_nch = reg + ovf;
        }
        __syncthreads();
        const unsigned long long nch = s_nch;
        if (nch) {
            unsigned long long cn = 0, cm = 0;
            if (cta0 && threadIdx.x == 0) ctl->chunks += nch;
            const unsigned creg = s_cpre[gridDim.x];
            // CTA-major dealing spreads one row's chunks over different SMs
            for (unsigned long long ci = (unsigned long long)wid * gridDim.x + blockIdx.x; ci < nch; ci += nwarps) {
                uint4 ch;
                if (ci < creg) {
                    const int r = region_of(s_cpre, ci);
                    ch = __ldcg(p.chunks + (unsigned long long)r * p.ch_cap + (ci - s_cpre[r]));
                } else {
                    ch = __ldcg(p.chunks + (unsigned long long)kMaxCtas * p.ch_cap + (ci - creg));
                }
                if (dir == DIR_PUSH) {
                    const int g = (int)ch.z;
                    const int32_t* col = S.slots[S.gslot[g]].col + ch.x;
                    for (uint32_t e0 = 0; e0 < ch.y; e0 += 32 * kEPL) {
                        int w[kEPL], gg[kEPL];
#pragma unroll
                        for (int u = 0; u < kEPL; ++u) {
                            const uint32_t ed = e0 + 32 * u + lane;
                            gg[u] = ed < ch.y ? g : -1;
                            w[u] = ed < ch.y ? __ldg(col + ed) : 0;
                        }
                        claim_edges(p, S, c, w, gg, lane, cn, cm);
                    }
                } else {
                    const int w = (int)ch.z;
                    const int q2 = (int)(ch.w >> 16), k = (int)(ch.w & 0xFFFFu);
                    const long long voff = (long long)q2 * p.W + (w >> 5);
                    const uint32_t bit = 1u << (w & 31);
                    if (p.visited[voff] & bit) continue;  // found by another row or chunk
                    const Slot ps = S.slots[p.nslots + S.islot[k]];
                    const bool hit =
                        warp_row_hit(ps.col, ch.x, ch.x + ch.y, fcur + (long long)S.isrc[k] * p.W, lane);
                    bool fresh[1] = {false};
                    if (hit && lane == 0) fresh[0] = !(atomicOr(p.visited + voff, bit) & bit);
                    const int qa[1] = {q2}, wa[1] = {w};
                    record_fresh<1>(p, S, c, fresh, qa, wa, lane, cn, cm);
                }
            }
            __syncthreads();
            flush_counts(c, cn, cm, s_red, p.nstates);
            grid_barrier(ctl, ++e);
        }
        if (cta0 && threadIdx.x == 0 && L < 64) ctl->bar_ns[L] = globaltimer() - ctl->t0;
        ++L;
        if (wid == 0) decide_level(p, S, L, lane, &s_view, s_wpre, s_sv, s_front);
        __syncthreads();
    }

    // ---- epilogue: answer = OR of P's rows at final states (engine.py:112-114)
    if (s_view.status == 0) {
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
        cnt = warp_sum_u64(cnt);
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

}  // namespace rpqk
