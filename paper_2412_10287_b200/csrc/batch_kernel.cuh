// batch_kernel.cuh -- up to 64 single-source 2-RPQs from different sources in
// ONE persistent launch, bit-sliced: every (state q, vertex v) pair carries a
// 64-bit word whose bit s says "(q, v) belongs to source s's set".  Per source
// this is exactly the masked evaluator (rpq/engine.py:146-171):
//   M_s <- step(M_s) <not P_s>;  P_s <- P_s + M_s
// but a frontier row v is read ONCE for all sources whose frontier holds
// (q, v) at that level, so adjacency traffic is shared across the batch
// (SURVEY.md §8(d) "batched sources", §8(e) regime 1).
//
// Layout:
//   vis[q][v]     64-bit source word: P, one row of nvp words per state
//   fw[L&1][q][v] 64-bit source word: M at level L.  A word is cleared when
//                 it is expanded, so fw[(L+1)&1] is all zero again when level
//                 L+1 starts writing it
//   act[L&1][q][b] one flag per 256-vertex block of M_L holding a non-empty
//                 word ("skip inactive (state, vertex-block)
//                 tiles"); raised by the discovery that first writes into it
//   heavy         row chunks (lo, hi, group, word) of rows longer than
//                 kLightDeg, expanded in a second phase of the level
// Per level: phase 1 sweeps the active blocks (a warp per block, coalesced
// word reads, 32 words per step), expands rows of <= kLightDeg edges
// warp-cooperatively (prefix over the items' degrees, kBEdges edges per lane
// in flight) and cuts longer rows into chunks; phase 2 (only when chunks
// exist) spreads the chunks over every warp.  Discoveries are fire-and-forget
// ORs (RED) into P and M_{L+1}: no atomic round trip, no work list.
#pragma once

namespace rpqk {

constexpr int kBatch = 64;             // sources per launch (bits of a source word)
using SW = unsigned long long;         // a source word: bit s = "in source s's set"
constexpr uint32_t kLightDeg = 64;     // rows up to this many edges stay in phase 1
constexpr uint32_t kChunk = 256;       // edges per heavy chunk
constexpr int kBlockShift = 8;         // activity flag per 2^8 vertices
constexpr int kBlockWords = 1 << kBlockShift;
constexpr int kBEdges = 4;             // edges per lane in flight per step (chunks)
constexpr int kBThreads = kThreadsLarge;  // batch state spaces are large: 32 warps per SM
constexpr int kBWarps = kBThreads / 32;
constexpr size_t kBWordsBytes = (size_t)kBWarps * (1 << 8) * sizeof(unsigned long long);  // 64 KB
constexpr int kGroups = 2;             // phase 1: groups of a state expanded together
constexpr int kGEdges = 2;             // phase 1: edges per lane and group per step

struct BCnt {
    unsigned int nact;         // 1 if some discovery produced M_L (0 iff M_L is empty)
    unsigned int nheavy;       // heavy chunks produced while expanding level L
    unsigned int overflow;
    unsigned int expire;       // the deadline check at the top of level L failed
    unsigned long long nnew;   // |M_L| summed over sources (from the items)
    unsigned long long items;  // (state, vertex) words of M_L that were non-empty
    SW active;                 // sources with a non-empty M_L
    unsigned int nlist;        // active blocks of M_L listed (the level's global block list)
    unsigned int pad2;
    unsigned long long steal;  // the list's grid-wide tail counter
};

struct BCtl {
    // ---- results prefix (copied back to the host) ------------------------
    unsigned int bar;  // monotonic barrier arrivals (runs continue from bar_base)
    int abort;
    unsigned long long t0;
    int status;
    int levels;
    unsigned long long te;     // sum over sources of product-graph edges expanded
    unsigned long long rows;   // edges read: sum over items of the row length (shared by a word's sources)
    unsigned long long pairs;  // sum over sources of |P_s|
    int last_level[kBatch];    // last level with a non-empty M_s
    unsigned long long reach_count[kBatch];
    unsigned long long level_items[64];
    unsigned long long level_new[64];
    unsigned long long level_ns[64];
    unsigned long long level_rows[64];  // edges read before level L starts (cumulative)
    SW level_active[64];
    // ---- working counters ------------------------------------------------
    BCnt bc[3];
};

struct BatchArgs {
    int nsrc;
    unsigned int bar_base;
    unsigned long long budget_ns;
    int sources[kBatch];
};

struct BHeavy {  // a heavy-row chunk: edges [a, b) of group g, for the sources of w
    uint32_t a, b, g, pad;
    SW w;
};

struct BParams {
    const BatchArgs* run;
    const int32_t* tables;
    const Slot* slots;
    SW* vis;
    SW* fw[2];
    uint32_t* act[2];  // [nstates][nblk] activity flags by level parity
    BHeavy* heavy;
    uint32_t* blist;  // [nstates * nblk] the level's active blocks
    BCtl* ctl;
    uint32_t* out;   // [kBatch][W] answer bitmaps
    long long nvp;   // words per state row of vis / fw (>= nv, multiple of kBlockWords)
    long long nblk;  // nvp / kBlockWords
    long long W;     // words per answer row (multiple of 4)
    unsigned long long heavy_cap;
    int nv, nstates, ngroups, nslots, ntargets, nstarts, nfinals, nin, table_ints;
};

// Source words w[c] reach (t[c], u[c]) (K edges per lane, loads overlapped):
// the sources not yet at (t, u) join P and M_{L+1}.  P is read first (from
// L2) and only ORed into where that read shows missing bits; the read may
// miss bits set earlier in this level, never bits of earlier levels, so the
// bits ORed into M_{L+1} are exactly the discoveries of this level (a bit may
// be discovered by several edges; ORs are idempotent).  Every discovery
// raises its 256-vertex block's activity flag for the next level (a plain
// store: idempotent, nothing to wait for) and counts toward M_{L+1}'s
// non-emptiness.
template <int K>
__device__ __forceinline__ void bvisit(const BParams& p, SW* fnext, uint32_t* anext, const bool (&act)[K],
                                       const int (&t)[K], const int (&u)[K], const SW (&w)[K],
                                       unsigned& nact) {
    long long off[K];
    SW seen[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        off[c] = (long long)t[c] * p.nvp + u[c];
        const bool ok = !act[c] || RPQ_CHECK(t[c] >= 0 && t[c] < p.nstates && u[c] >= 0 && u[c] < p.nv, RPQ_F_BATCH);
        seen[c] = act[c] && ok ? __ldcg(p.vis + off[c]) : ~0ull;
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
        const SW nw = w[c] & ~seen[c];
        if (nw) {
            atomicOr(p.vis + off[c], nw);  // results unused: RED
            atomicOr(fnext + off[c], nw);
            anext[(long long)t[c] * p.nblk + (u[c] >> kBlockShift)] = 1u;  // idempotent, no round trip
            ++nact;  // M_{L+1} is non-empty iff some discovery happened
        }
    }
}

// Rows longer than kLightDeg become chunks of kChunk edges for phase 2 (one
// atomic per warp); returns the degree phase 1 expands itself (0 if chunked).
__device__ __forceinline__ uint32_t split_heavy(const BParams& p, BCnt* cur, BCnt* nxt, int g, uint32_t lo,
                                                uint32_t deg, SW w, int lane) {
    const bool heavy = deg > kLightDeg;
    const uint32_t nch = heavy ? (deg + kChunk - 1) / kChunk : 0u;
    const uint32_t cincl = warp_incl_scan(nch, lane);
    const uint32_t ctot = __shfl_sync(FULL, cincl, 31);
    if (ctot) {
        unsigned cbase = 0;
        if (lane == 0) cbase = atomicAdd(&cur->nheavy, ctot);
        cbase = __shfl_sync(FULL, cbase, 0);
        if (heavy) {
            const unsigned long long c0 = (unsigned long long)cbase + cincl - nch;
            for (uint32_t c = 0; c < nch; ++c) {
                if (c0 + c < p.heavy_cap) {
                    const uint32_t a = lo + c * kChunk;
                    const uint32_t b = min(lo + deg, a + kChunk);
                    BHeavy hv;
                    hv.a = a;
                    hv.b = b;
                    hv.g = (uint32_t)g;
                    hv.pad = 0;
                    hv.w = w;
                    p.heavy[c0 + c] = hv;
                } else {
                    atomicExch(&nxt->overflow, 1u);
                }
            }
            return 0u;
        }
    }
    return deg;
}

// End of a phase: per-CTA sums into the counters.
__device__ __forceinline__ void bphase_end(const BParams& p, BCnt* nxt, unsigned nact, unsigned long long te,
                                           unsigned long long rows, unsigned long long nnew,
                                           unsigned long long items, SW act, BCnt* cnt,
                                           unsigned long long* s_red, SW* s_or) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned long long a = warp_sum_u64(nnew), b = warp_sum_u64(te), r = warp_sum_u64(rows);
    const unsigned long long it = warp_sum_u64(items), na = warp_sum_u64(nact);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) act |= __shfl_xor_sync(FULL, act, d);
    if (lane == 0) {
        s_red[5 * wid] = a;
        s_red[5 * wid + 1] = b;
        s_red[5 * wid + 2] = r;
        s_red[5 * wid + 3] = it;
        s_red[5 * wid + 4] = na;
        if (act) atomicOr(s_or, act);
    }
    __syncthreads();
    if (wid == 0) {
        unsigned long long v[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) v[k] = warp_sum_u64(lane < kBWarps ? s_red[5 * lane + k] : 0ull);
        if (lane == 0) {
            if (v[0]) atomicAdd(&cnt->nnew, v[0]);
            if (v[1]) atomicAdd(&p.ctl->te, v[1]);
            if (v[2]) atomicAdd(&p.ctl->rows, v[2]);
            if (v[3]) atomicAdd(&cnt->items, v[3]);
            if (v[4]) atomicOr(&nxt->nact, 1u);  // only non-emptiness matters (no 32-bit wrap)
            if (*s_or) atomicOr(&cnt->active, *s_or);
            *s_or = 0;
        }
    }
}

__global__ void __launch_bounds__(kBThreads, kMinBlocks) batch_kernel(BParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_red[5 * kBWarps];
    __shared__ SW s_or;
    __shared__ int s_single;  // every (state, symbol) group has exactly one target (a DFA)
    __shared__ BatchArgs s_run;

    // dynamic smem: [each warp's current block of M_L words: kBWords] [slots] [tables]
    SW* s_words = reinterpret_cast<SW*>(smem_raw);
    Slot* s_slots = reinterpret_cast<Slot*>(smem_raw + kBWordsBytes);
    int32_t* s_tab = reinterpret_cast<int32_t*>(smem_raw + kBWordsBytes + sizeof(Slot) * 2 * p.nslots);
    for (int i = threadIdx.x; i < 2 * p.nslots; i += blockDim.x) s_slots[i] = p.slots[i];
    for (int i = threadIdx.x; i < p.table_ints; i += blockDim.x) s_tab[i] = p.tables[i];
    if (threadIdx.x == 0) {
        s_run = *p.run;
        s_or = 0;
    }
    const int32_t* gbeg = s_tab;
    const int32_t* gslot = gbeg + p.nstates + 1;
    const int32_t* toff = gslot + p.ngroups;
    const int32_t* targets = toff + p.ngroups + 1;
    const int32_t* starts = targets + p.ntargets;
    const int32_t* finals = starts + p.nstarts;
    __syncthreads();
    if (threadIdx.x == 0) {
        int one = 1;
        for (int g = 0; g < p.ngroups; ++g) one &= (toff[g + 1] - toff[g]) == 1;
        s_single = one;
    }

    BCtl* ctl = p.ctl;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long gthreads = (long long)gridDim.x * blockDim.x;
    const bool cta0 = blockIdx.x == 0;
    if (cta0) {  // reset the control block (except the barrier counter)
        unsigned char* z = reinterpret_cast<unsigned char*>(ctl) + 8;
        for (size_t i = threadIdx.x * 8; i + 8 <= sizeof(BCtl) - 8; i += (size_t)blockDim.x * 8)
            *reinterpret_cast<unsigned long long*>(z + i) = 0ull;
        __syncthreads();
        if (threadIdx.x == 0) {
            ctl->abort = 0;
            ctl->t0 = globaltimer();
        }
        for (int s = threadIdx.x; s < kBatch; s += blockDim.x) ctl->last_level[s] = -1;
    }
    __syncthreads();
    const unsigned bar_base = s_run.bar_base;
    unsigned e = 0;
    const long long nbt = (long long)p.nstates * p.nblk;  // blocks over all states

    // ---- epoch 0: P <- 0, M <- 0, no active block, for every source
    {
        const long long n4 = (long long)p.nstates * p.nvp * (long long)sizeof(SW) / 16;  // uint4 units
        uint4* a = reinterpret_cast<uint4*>(p.vis);
        uint4* b = reinterpret_cast<uint4*>(p.fw[0]);
        uint4* c = reinterpret_cast<uint4*>(p.fw[1]);
        const uint4 z = make_uint4(0, 0, 0, 0);
        for (long long i = gtid; i < n4; i += gthreads) {
            a[i] = z;
            b[i] = z;
            c[i] = z;
        }
        for (long long i = gtid; i < nbt; i += gthreads) {
            p.act[0][i] = 0u;
            p.act[1][i] = 0u;
        }
    }
    grid_barrier_on(&ctl->bar, &ctl->abort, ++e, bar_base);

    // ---- epoch 1: seed P_s = M_s = {(q_s, source_s)} (engine.py:106-109)
    unsigned nact = 0;
    if (cta0 && threadIdx.x < s_run.nsrc) {  // source s = thread s (two warps)
        const int src = s_run.sources[threadIdx.x];
        for (int i = 0; i < p.nstarts; ++i) {
            const int q = starts[i];
            const long long off = (long long)q * p.nvp + src;
            atomicOr(p.vis + off, 1ull << threadIdx.x);
            atomicOr(p.fw[0] + off, 1ull << threadIdx.x);
            p.act[0][(long long)q * p.nblk + (src >> kBlockShift)] = 1u;
            ++nact;
        }
    }
    bphase_end(p, &ctl->bc[0], nact, 0ull, 0ull, 0ull, 0ull, 0ull, &ctl->bc[0], s_red, &s_or);
    nact = 0;
    grid_barrier_on(&ctl->bar, &ctl->abort, ++e, bar_base);

    // ---- level loop
    int status = 0;
    int L = 0;
    for (;;) {
        BCnt* cur = &ctl->bc[L % 3];
        BCnt* nxt = &ctl->bc[(L + 1) % 3];
        const unsigned ncur = ldcg(&cur->nact);
        const unsigned ovf = ldcg(&cur->overflow);
        const unsigned expire = ldcg(&cur->expire);
        const int abort = ldcg(&ctl->abort);
        if (abort) {
            status = ST_DEADLOCK;
            break;
        }
        if (ovf) {
            status = ST_OVERFLOW;
            break;
        }
        if (cta0 && threadIdx.x == 0) {
            const unsigned long long now = globaltimer();
            BCnt* old = &ctl->bc[(L + 2) % 3];  // level L-1's counters: statistics, then reset
            if (L > 0) {
                const SW act = ldcg(&old->active);
                const unsigned long long nn = ldcg(&old->nnew);
                for (int s = 0; s < kBatch; ++s)
                    if (act >> s & 1ull) ctl->last_level[s] = L - 1;
                ctl->pairs += nn;
                if (L - 1 < 64) {
                    ctl->level_new[L - 1] = nn;
                    ctl->level_items[L - 1] = ldcg(&old->items);
                    ctl->level_active[L - 1] = act;
                }
            }
            old->nact = 0;
            old->nheavy = 0;
            old->overflow = 0;
            old->expire = 0;
            old->nnew = 0;
            old->items = 0;
            old->active = 0;
            old->nlist = 0;
            old->steal = 0;
            if (L < 64) {
                ctl->level_ns[L] = now - ctl->t0;
                ctl->level_rows[L] = ldcg(&ctl->rows);
            }
            if (ncur) ctl->levels = L + 1;
            if (now - ctl->t0 > s_run.budget_ns) nxt->expire = 1;
        }
        if (ncur == 0) break;
        if (expire) {  // _Clock.check at the top of the iteration (engine.py:87-89)
            status = RPQ_ETIMEOUT;
            break;
        }
        uint32_t* acur = p.act[L & 1];
        uint32_t* anext = p.act[(L + 1) & 1];
        SW* fcur = p.fw[L & 1];
        SW* fnext = p.fw[(L + 1) & 1];
        // ---- phase 1: a warp per active block; light rows now, heavy rows as chunks
        unsigned long long te = 0, rows = 0, nnew = 0, items = 0;
        SW active = 0;
        // The level's active blocks are listed grid-wide first (one flag read
        // per block, coalesced; one atomic per warp), then dealt to every warp
        // of the grid: the first three quarters by a fixed stride, the rest
        // from one grid-wide counter, so the CTAs that finish early take the
        // tail (a per-CTA share of the blocks left 38% of the samples waiting
        // at the phase barriers).
        for (long long b0 = (long long)blockIdx.x * kBThreads; b0 < nbt; b0 += (long long)gridDim.x * kBThreads) {
            const long long b = b0 + threadIdx.x;
            const bool a = b < nbt && __ldcg(acur + b) != 0u;
            if (a) acur[b] = 0u;  // consumed (level L+2 raises it again)
            const unsigned m = __ballot_sync(FULL, a);
            if (m) {
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(&cur->nlist, (unsigned)__popc(m));
                base = __shfl_sync(FULL, base, 0);
                if (a) p.blist[base + __popc(m & lanemask_lt())] = (uint32_t)b;
            }
        }
        grid_barrier_on(&ctl->bar, &ctl->abort, ++e, bar_base);
        const unsigned long long nlisted = ldcg(&cur->nlist);
        const unsigned long long gwarp_b = (unsigned long long)blockIdx.x * kBWarps + wid;
        const unsigned long long nwarps_b = (unsigned long long)gridDim.x * kBWarps;
#ifndef RPQ_BATCH_STATIC_NUM
#define RPQ_BATCH_STATIC_NUM 2  // static share of the block list, in quarters (cfg5: 3/4 357, 2/4 369, 0 352 GTEPS)
#endif
        const unsigned long long nown = nlisted / 4 * RPQ_BATCH_STATIC_NUM;
        unsigned long long kk = gwarp_b;
        for (;;) {
            unsigned long long k = kk;
            if (k >= nown) {  // the stolen tail
                if (lane == 0) k = nown + atomicAdd(&cur->steal, 1ull);
                k = __shfl_sync(FULL, k, 0);
            }
            kk += nwarps_b;
            if (k >= nlisted) break;
            const long long blk = p.blist[k];
            const int q = (int)(blk / p.nblk);
            const long long v0 = (blk - (long long)q * p.nblk) * kBlockWords;
            SW* row = fcur + (long long)q * p.nvp;
            // the block's words, all loads in flight, parked in this warp's
            // shared slots (a register array indexed by the loop would be
            // selected element by element)
            SW* wsm = s_words + wid * kBlockWords;
            {
                SW wv[kBlockWords / 32];
#pragma unroll
                for (int r = 0; r < kBlockWords / 32; ++r) wv[r] = __ldcg(row + v0 + 32 * r + lane);
#pragma unroll
                for (int r = 0; r < kBlockWords / 32; ++r) wsm[32 * r + lane] = wv[r];
            }
            __syncwarp();
            const int ng = gbeg[q + 1] - gbeg[q];
#pragma unroll 1
            for (int r = 0; r < kBlockWords / 32; ++r) {
                const SW w = wsm[32 * r + lane];
                if (!__any_sync(FULL, w != 0ull)) continue;
                const int v = (int)(v0 + 32 * r + lane);
                if (w) {
                    row[v] = 0ull;        // fw[L&1] must be zero when level L+1 writes it
                    nnew += __popcll(w);  // M_L's (pair, source) members, each in exactly one word
                    ++items;
                    active |= w;
                }
                if (s_single) {
                    // a DFA: every group has one target.  Up to kGroups groups
                    // at once: their row pointers, then their column loads,
                    // in flight together
                    for (int kg0 = 0; kg0 < ng; kg0 += kGroups) {
                        uint32_t lo[kGroups], deg[kGroups], excl[kGroups], T[kGroups];
                        int tq[kGroups];
                        const int32_t* colk[kGroups];
#pragma unroll
                        for (int k = 0; k < kGroups; ++k) {
                            lo[k] = deg[k] = 0;
                            tq[k] = 0;
                            colk[k] = nullptr;
                            if (kg0 + k < ng) {
                                const int g = gbeg[q] + kg0 + k;
                                const Slot sl = s_slots[gslot[g]];
                                colk[k] = sl.col;
                                tq[k] = targets[toff[g]];
                                if (w) {
                                    lo[k] = sl.rowptr[v];
                                    deg[k] = sl.rowptr[v + 1];
                                }
                            }
                        }
                        uint32_t Tmax = 0;
#pragma unroll
                        for (int k = 0; k < kGroups; ++k) {
                            if (kg0 + k >= ng) {
                                T[k] = excl[k] = 0;
                                continue;
                            }
                            const int g = gbeg[q] + kg0 + k;
                            deg[k] -= lo[k];
                            te += (unsigned long long)deg[k] * __popcll(w);
                            rows += deg[k];
                            deg[k] = split_heavy(p, cur, nxt, g, lo[k], deg[k], w, lane);
                            const uint32_t incl = warp_incl_scan(deg[k], lane);
                            excl[k] = incl - deg[k];
                            T[k] = __shfl_sync(FULL, incl, 31);
                            Tmax = max(Tmax, T[k]);
                        }
                        for (uint32_t e0 = 0; e0 < Tmax; e0 += 32 * kGEdges) {
                            constexpr int K = kGroups * kGEdges;
                            bool act[K];
                            int tt[K], uu[K];
                            SW ww[K];
#pragma unroll
                            for (int k = 0; k < kGroups; ++k) {
#pragma unroll
                                for (int c = 0; c < kGEdges; ++c) {
                                    const int i = k * kGEdges + c;
                                    const uint32_t x = e0 + 32 * c + lane;
                                    const int j = warp_upper_lane(excl[k], x);
                                    const uint32_t lo_j = __shfl_sync(FULL, lo[k], j);
                                    const uint32_t ex_j = __shfl_sync(FULL, excl[k], j);
                                    ww[i] = __shfl_sync(FULL, w, j);
                                    act[i] = x < T[k];
                                    uu[i] = act[i] ? colk[k][lo_j + (x - ex_j)] : 0;
                                    tt[i] = tq[k];
                                }
                            }
                            bvisit<K>(p, fnext, anext, act, tt, uu, ww, nact);
                        }
                    }
                } else {
                    for (int kg = 0; kg < ng; ++kg) {
                        const int g = gbeg[q] + kg;
                        uint32_t lo = 0, deg = 0;
                        if (w) {
                            const Slot sl = s_slots[gslot[g]];
                            lo = sl.rowptr[v];
                            deg = sl.rowptr[v + 1] - lo;
                        }
                        te += (unsigned long long)deg * __popcll(w);
                        rows += deg;
                        deg = split_heavy(p, cur, nxt, g, lo, deg, w, lane);
                        const uint32_t incl = warp_incl_scan(deg, lane);
                        const uint32_t excl = incl - deg;
                        const uint32_t T = __shfl_sync(FULL, incl, 31);
                        const int32_t* col = s_slots[gslot[g]].col;
                        for (uint32_t e0 = 0; e0 < T; e0 += 32) {
                            const uint32_t x = e0 + lane;
                            const int j = warp_upper_lane(excl, x);
                            const uint32_t lo_j = __shfl_sync(FULL, lo, j);
                            const uint32_t ex_j = __shfl_sync(FULL, excl, j);
                            const SW w_j = __shfl_sync(FULL, w, j);
                            const bool a0 = x < T;
                            const int u = a0 ? col[lo_j + (x - ex_j)] : 0;
                            for (int t = toff[g]; t < toff[g + 1]; ++t) {
                                const bool act[1] = {a0};
                                const int tt[1] = {targets[t]};
                                const int uu[1] = {u};
                                const SW ww[1] = {w_j};
                                bvisit<1>(p, fnext, anext, act, tt, uu, ww, nact);
                            }
                        }
                    }
                }
            }
        }
        bphase_end(p, nxt, nact, te, rows, nnew, items, active, cur, s_red, &s_or);
        nact = 0;
        grid_barrier_on(&ctl->bar, &ctl->abort, ++e, bar_base);

        // ---- phase 2: heavy chunks, spread over every warp of the grid
        const unsigned nh = min((unsigned long long)ldcg(&cur->nheavy), p.heavy_cap);
        if (nh) {
            for (unsigned long long c = blockIdx.x + (unsigned long long)wid * gridDim.x; c < nh;
                 c += (unsigned long long)gridDim.x * kBWarps) {
                const BHeavy h = p.heavy[c];
                const int g = (int)h.g;
                const int32_t* col = s_slots[gslot[g]].col;
                const int t0 = toff[g], t1 = toff[g + 1];
                if (s_single) {
                    for (uint32_t a = h.a; a < h.b; a += 32 * kBEdges) {
                        bool act[kBEdges];
                        int tt[kBEdges], uu[kBEdges];
                        SW ww[kBEdges];
#pragma unroll
                        for (int c2 = 0; c2 < kBEdges; ++c2) {
                            const uint32_t x = a + 32 * c2 + lane;
                            act[c2] = x < h.b;
                            uu[c2] = act[c2] ? col[x] : 0;
                            tt[c2] = targets[t0];
                            ww[c2] = h.w;
                        }
                        bvisit<kBEdges>(p, fnext, anext, act, tt, uu, ww, nact);
                    }
                } else {
                    for (uint32_t a = h.a; a < h.b; a += 32) {
                        const bool a0 = a + lane < h.b;
                        const int u = a0 ? col[a + lane] : 0;
                        for (int t = t0; t < t1; ++t) {
                            const bool act[1] = {a0};
                            const int tt[1] = {targets[t]};
                            const int uu[1] = {u};
                            const SW ww[1] = {h.w};
                            bvisit<1>(p, fnext, anext, act, tt, uu, ww, nact);
                        }
                    }
                }
            }
            bphase_end(p, nxt, nact, 0ull, 0ull, 0ull, 0ull, 0ull, cur, s_red, &s_or);
            nact = 0;
            grid_barrier_on(&ctl->bar, &ctl->abort, ++e, bar_base);
        }
        ++L;
    }

    // ---- epilogue: answer_s = OR of P_s's rows at final states (engine.py:112-114),
    // transposed from source words to one bitmap per source
    if (status == 0) {
        const long long nblk = (p.nv + 127) / 128;
        const long long gwarp = (long long)blockIdx.x * kBWarps + wid;
        const long long nwarps = (long long)gridDim.x * kBWarps;
        unsigned long long cnt[2] = {0ull, 0ull};  // this lane's sources lane and 32 + lane
        for (long long b = gwarp; b < nblk; b += nwarps) {
            SW acc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const long long v = b * 128 + 32 * k + lane;
                acc[k] = 0;
                if (v < p.nv)
                    for (int f = 0; f < p.nfinals; ++f) acc[k] |= p.vis[(long long)finals[f] * p.nvp + v];
            }
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t mine[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    mine[k] = 0;
#pragma unroll 4
                    for (int s = 0; s < 32; ++s) {
                        const uint32_t bits = __ballot_sync(FULL, (acc[k] >> (32 * half + s)) & 1ull);
                        if (lane == s) mine[k] = bits;
                    }
                }
                const int src = 32 * half + lane;
                if (src < s_run.nsrc) {
                    *reinterpret_cast<uint4*>(p.out + (long long)src * p.W + b * 4) =
                        make_uint4(mine[0], mine[1], mine[2], mine[3]);
                    cnt[half] += __popc(mine[0]) + __popc(mine[1]) + __popc(mine[2]) + __popc(mine[3]);
                }
            }
        }
        // per source: shared-memory sums, then one global atomic per CTA
        if (threadIdx.x < kBatch) s_red[threadIdx.x] = 0ull;
        __syncthreads();
        for (int half = 0; half < 2; ++half)
            if (32 * half + lane < s_run.nsrc && cnt[half]) atomicAdd(&s_red[32 * half + lane], cnt[half]);
        __syncthreads();
        if (threadIdx.x < s_run.nsrc && s_red[threadIdx.x])
            atomicAdd(&ctl->reach_count[threadIdx.x], s_red[threadIdx.x]);
    }
    if (cta0 && threadIdx.x == 0) ctl->status = status;
}

}  // namespace rpqk
