// ingest.cuh -- device-side graph ingest: an edge list (src, label, dst) is
// grouped by label on the device once; the canonical CSR of a label in either
// direction (rows sorted, duplicates collapsed, self-loops kept -- the layout
// of the reference's LabeledGraph: graph_store.py:161-176, sparse_bool.py:51-87)
// is built on first use by a radix sort of packed (row, col) keys.
#pragma once

#include <cub/cub.cuh>

namespace rpqk {

// label histogram (one atomic per edge into shared memory, then global)
__global__ void label_histogram_kernel(const int32_t* __restrict__ lab, long long n, int nl,
                                       unsigned long long* __restrict__ hist) {
    extern __shared__ unsigned int s_hist[];
    const bool local = nl <= 8192;
    if (local)
        for (int i = threadIdx.x; i < nl; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int l = lab[i];
        if (l < 0 || l >= nl) continue;
        if (local)
            atomicAdd(&s_hist[l], 1u);
        else
            atomicAdd(&hist[l], 1ull);
    }
    __syncthreads();
    if (local)
        for (int i = threadIdx.x; i < nl; i += blockDim.x)
            if (s_hist[i]) atomicAdd(&hist[i], (unsigned long long)s_hist[i]);
}

// scatter edges into their label's segment as packed (src << 32 | dst) keys.
// Labels with a shared-memory histogram (nl <= 8192): a block takes a chunk of
// edges, counts it per label in shared memory, reserves one range per label
// with a single global atomic, then places its edges with shared-memory
// cursors (no global atomic per edge: a few hot Zipf labels would serialize).
constexpr int kScatterChunk = 4096;
__global__ void label_scatter_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                     const int32_t* __restrict__ lab, long long n, int nl,
                                     unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ out) {
    extern __shared__ unsigned int s_cnt[];  // [nl] counts, then reused as cursors
    const bool local = nl <= 8192;
    if (!local) {  // many labels: one global atomic per edge
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x) {
            const int l = lab[i];
            if (l < 0 || l >= nl) continue;
            const unsigned long long pos = atomicAdd(&cursor[l], 1ull);
            out[pos] = ((unsigned long long)(uint32_t)src[i] << 32) | (uint32_t)dst[i];
        }
        return;
    }
    unsigned long long* s_base = reinterpret_cast<unsigned long long*>(s_cnt + ((nl + 1) & ~1));
    for (long long c0 = (long long)blockIdx.x * kScatterChunk; c0 < n; c0 += (long long)gridDim.x * kScatterChunk) {
        const long long c1 = min(n, c0 + (long long)kScatterChunk);
        for (int i = threadIdx.x; i < nl; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const int l = lab[i];
            if (l >= 0 && l < nl) atomicAdd(&s_cnt[l], 1u);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nl; i += blockDim.x) {
            const unsigned c = s_cnt[i];
            s_base[i] = c ? atomicAdd(&cursor[i], (unsigned long long)c) : 0ull;
            s_cnt[i] = 0;
        }
        __syncthreads();
        for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const int l = lab[i];
            if (l < 0 || l >= nl) continue;
            const unsigned long long pos = s_base[l] + atomicAdd(&s_cnt[l], 1u);
            out[pos] = ((unsigned long long)(uint32_t)src[i] << 32) | (uint32_t)dst[i];
        }
        __syncthreads();
    }
}

// keys (row << 32 | col) -> transposed keys (col << 32 | row)
__global__ void swap_halves_kernel(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out,
                                   long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = in[i];
        out[i] = (k << 32) | (k >> 32);
    }
}

// sorted unique keys -> row counts (atomic) and columns
__global__ void keys_to_csr_kernel(const unsigned long long* __restrict__ keys, long long n,
                                   uint32_t* __restrict__ rowcnt, int32_t* __restrict__ col) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        col[i] = (int32_t)(uint32_t)k;
        atomicAdd(&rowcnt[(uint32_t)(k >> 32) + 1], 1u);
    }
}

// Merged adjacency (rows of several slots concatenated per vertex): degree sums
__global__ void merge_degree_kernel(const uint32_t* const* __restrict__ rowptrs, int k, long long nv,
                                    uint32_t* __restrict__ deg) {
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        uint32_t d = 0;
        for (int s = 0; s < k; ++s) d += rowptrs[s][v + 1] - rowptrs[s][v];
        deg[v + 1] = d;
    }
}

// ... and the columns, one warp per vertex (coalesced segment copies)
__global__ void merge_copy_kernel(const uint32_t* const* __restrict__ rowptrs, const int32_t* const* __restrict__ cols,
                                  int k, long long nv, const uint32_t* __restrict__ mrow, int32_t* __restrict__ mcol) {
    const int lane = threadIdx.x & 31;
    for (long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nv;
         v += ((long long)gridDim.x * blockDim.x) >> 5) {
        uint32_t at = mrow[v];
        for (int s = 0; s < k; ++s) {
            const uint32_t lo = rowptrs[s][v], hi = rowptrs[s][v + 1];
            for (uint32_t e = lo + lane; e < hi; e += 32) mcol[at + (e - lo)] = cols[s][e];
            at += hi - lo;
        }
    }
}

}  // namespace rpqk
