// small_kernel.cuh -- one CTA evaluates a single-source 2-RPQ whose product
// state space fits in shared memory (|Q| x |V| <= kSmallMaxWords * 32 pairs,
// e.g. BASELINE cfg1: 2 x 10,000).  Same result, statistics and deadline
// semantics as ssr_kernel (the masked loop, engine.py:146-171), but P and the
// two frontier bitmaps live in shared memory and a level ends at a
// __syncthreads instead of a grid barrier: a level costs about one dependent
// chain of global loads (row pointers, columns) instead of barrier + decision
// + chain.  Push only: at this size a level's rows are few.
#pragma once

namespace rpqk {

constexpr int kSmallThreads = 1024;
constexpr int kSmallWarps = kSmallThreads / 32;
constexpr long long kSmallMaxWords = 12288;  // |Q| * W words per bitmap (3 bitmaps: 144 KB)

__global__ void __launch_bounds__(kSmallThreads, 1) small_kernel(Params p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ RunArgs s_run;
    __shared__ unsigned long long s_nnew, s_te;
    __shared__ int s_done, s_status, s_iters;

    Slot* s_slots = reinterpret_cast<Slot*>(smem_raw);
    int32_t* s_tab = reinterpret_cast<int32_t*>(smem_raw + sizeof(Slot) * 2 * p.nslots);
    const size_t tab_bytes = ((size_t)p.table_ints * 4 + 15) / 16 * 16;
    uint32_t* P = reinterpret_cast<uint32_t*>(smem_raw + sizeof(Slot) * 2 * p.nslots + tab_bytes);
    const long long nw = (long long)p.nstates * p.W;
    uint32_t* F[2] = {P + nw, P + 2 * nw};
    for (int i = threadIdx.x; i < 2 * p.nslots; i += blockDim.x) s_slots[i] = p.slots[i];
    for (int i = threadIdx.x; i < p.table_ints; i += blockDim.x) s_tab[i] = p.tables[i];
    for (long long i = threadIdx.x; i < 3 * nw; i += blockDim.x) P[i] = 0u;
    if (threadIdx.x == 0) s_run = *p.run;
    Ctl* ctl = p.ctl;
    {  // reset the control block, except the barrier counter (the grid kernel's)
        unsigned char* z = reinterpret_cast<unsigned char*>(ctl) + 8;
        for (size_t i = threadIdx.x * 8; i + 8 <= sizeof(Ctl) - 8; i += (size_t)blockDim.x * 8)
            *reinterpret_cast<unsigned long long*>(z + i) = 0ull;
    }
    __syncthreads();
    const int32_t* gbeg = s_tab;
    const int32_t* gslot = gbeg + p.nstates + 1;
    const int32_t* toff = gslot + p.ngroups;
    const int32_t* targets = toff + p.ngroups + 1;
    const int32_t* starts = targets + p.ntargets;
    const int32_t* finals = starts + p.nstarts;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // pull the push-direction adjacency of every slot into L2 up front (bulk
    // prefetch, 16 B granules): the level loop then pays L2, not DRAM, latency
    for (int s = wid; s < p.nslots; s += kSmallWarps) {
        const unsigned long long rp_bytes = ((unsigned long long)p.nv + 1) * 4ull;
        const unsigned long long col_bytes = p.slot_nnz[s] * 4ull;
        if (rp_bytes + col_bytes > (8ull << 20)) continue;
        const char* rp = reinterpret_cast<const char*>(s_slots[s].rowptr);
        const char* cl = reinterpret_cast<const char*>(s_slots[s].col);
        for (unsigned long long o = (unsigned long long)lane * 4096; o < rp_bytes; o += 32ull * 4096) {
            const unsigned n = (unsigned)min(4096ull, (rp_bytes - o) & ~15ull);
            if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rp + o), "r"(n) : "memory");
        }
        for (unsigned long long o = (unsigned long long)lane * 4096; o < col_bytes; o += 32ull * 4096) {
            const unsigned n = (unsigned)min(4096ull, (col_bytes - o) & ~15ull);
            if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cl + o), "r"(n) : "memory");
        }
    }
    const unsigned long long t0 = globaltimer();
    if (threadIdx.x == 0) {
        ctl->abort = 0;
        ctl->t0 = t0;
        s_nnew = 0;
        s_te = 0;
        s_done = 0;
        s_status = 0;
        s_iters = 0;
    }
    __syncthreads();
    // seed P = M = {(q_s, source)} (engine.py:106-109)
    if (threadIdx.x < p.nstarts) {
        const int q = starts[threadIdx.x];
        const long long off = (long long)q * p.W + (s_run.source >> 5);
        const uint32_t bit = 1u << (s_run.source & 31);
        if (!(atomicOr(P + off, bit) & bit)) {
            atomicOr(F[0] + off, bit);
            atomicAdd(&s_nnew, 1ull);
        }
    }
    __syncthreads();
    unsigned long long pairs = 0, te_total = 0;
    int L = 0, levels = 0;
    for (;; ++L) {
        const unsigned long long nnew = s_nnew;  // |F_L|
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long now = globaltimer();
            pairs += nnew;
            if (L < 64) {
                ctl->level_new[L] = (long long)nnew;
                ctl->level_ns[L] = now - t0;
                ctl->level_dir[L] = DIR_PUSH;
            }
            s_nnew = 0;
            s_te = 0;
            if (nnew == 0) {  // while m.nnz (engine.py:157)
                s_done = 1;
                s_iters = L;
            } else if (L > 0 && now - t0 > s_run.budget_ns) {  // _Clock.check
                s_done = 1;
                s_status = RPQ_ETIMEOUT;
                s_iters = L;
            }
            if (!s_done && L > 0) levels = L;
        }
        __syncthreads();
        if (s_done) break;
        uint32_t* fc = F[L & 1];
        uint32_t* fn = F[(L + 1) & 1];
        unsigned long long nnew_w = 0, te_w = 0;
        // each warp: 32 frontier words at a time; their set bits are dealt
        // 32 per round to the lanes (prefix over the words' popcounts)
        for (long long w0 = (long long)wid * 32; w0 < nw; w0 += (long long)kSmallWarps * 32) {
            const long long wi = w0 + lane;
            const uint32_t bits = wi < nw ? fc[wi] : 0u;
            const uint32_t cnt_l = __popc(bits);
            const uint32_t incl_b = warp_incl_scan(cnt_l, lane);
            const uint32_t excl_b = incl_b - cnt_l;
            const uint32_t nitems = __shfl_sync(FULL, incl_b, 31);
            for (uint32_t r0 = 0; r0 < nitems; r0 += 32) {
                const uint32_t x = r0 + lane;
                const bool valid = x < nitems;
                const int jb = warp_upper_lane(excl_b, valid ? x : 0u);
                const uint32_t wb = __shfl_sync(FULL, bits, jb);
                const uint32_t eb = __shfl_sync(FULL, excl_b, jb);
                int q = 0, v = 0;
                if (valid) {
                    const long long wj = w0 + jb;
                    q = (int)(wj / p.W);
                    v = (int)((wj - (long long)q * p.W) * 32 + __fns(wb, 0, (int)(x - eb) + 1));
                }
                const int ng = valid ? gbeg[q + 1] - gbeg[q] : 0;
                int maxng = ng;
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) maxng = max(maxng, __shfl_xor_sync(FULL, maxng, d));
                for (int kg0 = 0; kg0 < maxng; kg0 += kFastGroups) {
                    // row pointers of up to kFastGroups groups in flight together
                    uint32_t lo[kFastGroups], hi[kFastGroups];
#pragma unroll
                    for (int k = 0; k < kFastGroups; ++k) {
                        lo[k] = hi[k] = 0;
                        if (kg0 + k < ng) {
                            const Slot sl = s_slots[gslot[gbeg[q] + kg0 + k]];
                            lo[k] = sl.rowptr[v];
                            hi[k] = sl.rowptr[v + 1];
                        }
                    }
#pragma unroll
                    for (int k = 0; k < kFastGroups; ++k) {
                        if (kg0 + k >= maxng) break;
                        const int g = kg0 + k < ng ? gbeg[q] + kg0 + k : 0;
                        const uint32_t deg = hi[k] - lo[k];
                        if (deg) te_w += (unsigned long long)deg * (unsigned long long)(toff[g + 1] - toff[g]);
                        const uint32_t incl = warp_incl_scan(deg, lane);
                        const uint32_t excl = incl - deg;
                        const uint32_t T = __shfl_sync(FULL, incl, 31);
                        for (uint32_t e0 = 0; e0 < T; e0 += 32 * kEdgesPerLane) {
                            int uu[kEdgesPerLane], gg[kEdgesPerLane];
#pragma unroll
                            for (int c = 0; c < kEdgesPerLane; ++c) {  // column loads in flight together
                                const uint32_t xe = e0 + 32 * c + lane;
                                const int j = warp_upper_lane(excl, xe);
                                const uint32_t lo_j = __shfl_sync(FULL, lo[k], j);
                                const uint32_t ex_j = __shfl_sync(FULL, excl, j);
                                const int g_j = __shfl_sync(FULL, g, j);  // every lane: a sync shuffle
                                gg[c] = xe < T ? g_j : -1;
                                uu[c] = gg[c] >= 0 ? s_slots[gslot[gg[c]]].col[lo_j + (xe - ex_j)] : 0;
                            }
#pragma unroll
                            for (int c = 0; c < kEdgesPerLane; ++c) {
                                if (gg[c] < 0) continue;
                                const int u = uu[c];
                                const uint32_t bit = 1u << (u & 31);
                                for (int t = toff[gg[c]]; t < toff[gg[c] + 1]; ++t) {
                                    const long long off = (long long)targets[t] * p.W + (u >> 5);
                                    if (!(P[off] & bit) && !(atomicOr(P + off, bit) & bit)) {
                                        atomicOr(fn + off, bit);
                                        ++nnew_w;
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
        nnew_w = warp_sum_u64(nnew_w);
        te_w = warp_sum_u64(te_w);
        if (lane == 0) {
            if (nnew_w) atomicAdd(&s_nnew, nnew_w);
            if (te_w) atomicAdd(&s_te, te_w);
        }
        __syncthreads();
        for (long long i = threadIdx.x; i < nw; i += blockDim.x) fc[i] = 0u;  // F_{L+2} starts empty
        if (threadIdx.x == 0) {
            te_total += s_te;
            if (L < 64) ctl->level_edges[L] = (long long)s_te;
        }
    }
    // answer = OR of P's rows at final states (engine.py:112-114); P back to HBM
    const long long Wn = ((long long)p.nv + 31) >> 5;
    unsigned long long cnt = 0;
    for (long long i = threadIdx.x; i < Wn; i += blockDim.x) {
        uint32_t acc = 0;
        for (int f = 0; f < p.nfinals; ++f) acc |= P[(long long)finals[f] * p.W + i];
        if (i == Wn - 1 && (p.nv & 31)) acc &= (1u << (p.nv & 31)) - 1u;
        cnt += __popc(acc);
        p.reach_bits[i] = acc;
        uint32_t b4[8];  // 32 answer bytes of this word (the buffer has W * 32 + 32 bytes)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t nib = (acc >> (4 * k)) & 0xFu;
            b4[k] = (nib & 1u) | ((nib >> 1 & 1u) << 8) | ((nib >> 2 & 1u) << 16) | ((nib >> 3 & 1u) << 24);
        }
        uint4* dst = reinterpret_cast<uint4*>(p.reach + i * 32);
        dst[0] = make_uint4(b4[0], b4[1], b4[2], b4[3]);
        dst[1] = make_uint4(b4[4], b4[5], b4[6], b4[7]);
    }
    for (long long i = threadIdx.x; i < nw; i += blockDim.x) p.visited[i] = P[i];
    cnt = warp_sum_u64(cnt);
    if (lane == 0 && cnt) atomicAdd(&ctl->reach_count, cnt);
    if (threadIdx.x == 0) {
        ctl->status = s_status;
        ctl->iterations = s_iters;
        ctl->levels = levels;
        ctl->te_push = te_total;
        ctl->te_exact = te_total;
        ctl->pairs = pairs;
    }
}

}  // namespace rpqk
