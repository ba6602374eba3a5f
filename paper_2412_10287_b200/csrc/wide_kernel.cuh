// wide_kernel.cuh -- single-source 2-RPQ for automata beyond the persistent
// kernel's table limits (more than 256 states or (state, symbol) groups, or
// more than 128 symbols).  The reference evaluates any automaton
// (rpq/engine.py:146-171 loops over N.alphabet with numpy); the persistent
// kernel keeps its automaton tables in shared memory and packs group ids into
// 8 bits.  Here the transition list itself lives in global memory and every
// level is one launch of a plain push step: the same P / M sets level by
// level, so the answer and the masked loop's iteration count are the
// reference's.  Throughput is not the point of this path.
#pragma once

namespace rpqk {

struct WideTrans {
    const uint32_t* rowptr;  // A_s of the transition's symbol (forward[l] or backward[l])
    const int32_t* col;
    int32_t src, dst;
};

// One level: for every transition t = (q -s-> q') whose source state has a
// frontier, every (q, v) in F_L and every edge v -s-> w: claim (q', w) in P;
// the first setter puts it into F_{L+1}.  A warp per word of F_L[q]; the
// word's vertices one after the other, their rows lane-parallel.
__global__ void __launch_bounds__(256) wide_step_kernel(const WideTrans* __restrict__ trans, int ntrans,
                                                        uint32_t* __restrict__ visited,
                                                        const uint32_t* __restrict__ fcur,
                                                        uint32_t* __restrict__ fnext, long long W, int nv,
                                                        const unsigned int* __restrict__ cnt_cur,
                                                        unsigned int* __restrict__ cnt_next,
                                                        unsigned long long* __restrict__ totals) {
    const int lane = threadIdx.x & 31;
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long Wn = ((long long)nv + 31) >> 5;
    unsigned long long nnew = 0, te = 0;
    for (int t = 0; t < ntrans; ++t) {
        const WideTrans tr = trans[t];
        if (cnt_cur[tr.src] == 0) continue;
        const uint32_t* frow = fcur + (long long)tr.src * W;
        uint32_t* prow = visited + (long long)tr.dst * W;
        uint32_t* nrow = fnext + (long long)tr.dst * W;
        unsigned int found = 0;
        for (long long wi = gwarp; wi < Wn; wi += nwarps) {
            uint32_t bits = frow[wi];
            while (bits) {
                const long long v = wi * 32 + __ffs(bits) - 1;
                bits &= bits - 1;
                const uint32_t lo = tr.rowptr[v], hi = tr.rowptr[v + 1];
                if (lane == 0) te += hi - lo;
                for (uint32_t e = lo + lane; e < hi; e += 32) {
                    const int w = tr.col[e];
                    if (w < 0 || w >= nv) continue;  // (validated at upload)
                    const uint32_t bit = 1u << (w & 31);
                    if (prow[w >> 5] & bit) continue;
                    const uint32_t old = atomicOr(prow + (w >> 5), bit);
                    if (!(old & bit)) {
                        atomicOr(nrow + (w >> 5), bit);
                        ++found;
                    }
                }
            }
        }
        found = __reduce_add_sync(0xFFFFFFFFu, found);
        if (lane == 0 && found) atomicAdd(&cnt_next[tr.dst], found);
        nnew += found;
    }
    if (lane == 0) {
        if (nnew) atomicAdd(&totals[0], nnew);
        if (te) atomicAdd(&totals[1], te);
    }
}

// seed: P = M = {(q_s, source)} (engine.py:106-109)
__global__ void wide_seed_kernel(const int32_t* __restrict__ starts, int nstarts, int source, long long W,
                                 uint32_t* __restrict__ visited, uint32_t* __restrict__ f0,
                                 unsigned int* __restrict__ cnt, unsigned long long* __restrict__ totals) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nstarts; i += gridDim.x * blockDim.x) {
        const long long off = (long long)starts[i] * W + (source >> 5);
        const uint32_t bit = 1u << (source & 31);
        const uint32_t old = atomicOr(visited + off, bit);
        if (!(old & bit)) {  // (a start state listed twice seeds once)
            atomicOr(f0 + off, bit);
            atomicAdd(&cnt[starts[i]], 1u);
            atomicAdd(&totals[0], 1ull);
        }
    }
}

// answer = OR of P's rows at final states (engine.py:112-114); totals[2] += |answer|
__global__ void wide_project_kernel(const int32_t* __restrict__ finals, int nfinals, const uint32_t* __restrict__ visited,
                                    long long W, long long Wn, uint32_t* __restrict__ out,
                                    unsigned long long* __restrict__ totals) {
    unsigned long long cnt = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < Wn;
         i += (long long)gridDim.x * blockDim.x) {
        uint32_t acc = 0;
        for (int f = 0; f < nfinals; ++f) acc |= visited[(long long)finals[f] * W + i];
        out[i] = acc;
        cnt += __popc(acc);
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, (unsigned)cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&totals[2], cnt);
}

}  // namespace rpqk
