// rpq_b200.cu -- host side of the B200-native (sm_100a) single-source 2-RPQ
// engine behind the C ABI of include/rpq_b200.h: graph residency (per-label
// CSR in both directions, graph_store.py:51-52), query compilation into the
// kernel's tables (_label_pairs, engine.py:92-103), workspaces, launch.
// The device code is in ssr_kernel.cuh.
#include "rpq_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "ssr_kernel.cuh"
#include "batch_kernel.cuh"
#include "small_kernel.cuh"
#include "wide_kernel.cuh"
#include "ingest.cuh"

using namespace rpqk;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? RPQ_ENOMEM : RPQ_ECUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                      \
    do {                                                    \
        cudaError_t e_ = (expr);                            \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
    } while (0)

// Checked build: a device bounds check that failed during the last run
// (checks.cuh) fails the run.  The site is reset for the next run.
int check_sites() {
#ifdef RPQ_CHECKED
    unsigned site = 0;
    if (cudaMemcpyFromSymbol(&site, rpqk::g_check_site, sizeof(site)) != cudaSuccess) {
        cudaGetLastError();
        return RPQ_OK;
    }
    if (site) {
        const unsigned zero = 0;
        cudaMemcpyToSymbol(rpqk::g_check_site, &zero, sizeof(zero));
        static const char* files[] = {"?", "ssr_kernel.cuh", "batch_kernel.cuh", "small_kernel.cuh"};
        const unsigned f = site / 100000u;
        return fail(RPQ_ECUDA, std::string("bounds check failed at ") + (f < 4 ? files[f] : "?") + ":" +
                                   std::to_string(site % 100000u));
    }
#endif
    return RPQ_OK;
}

// Pinned, mapped host blocks handed out by rpq_host_alloc: base -> bytes.
// A run whose answer buffer lies inside one has the kernel write the answer
// there directly (no copy node, no host memcpy).
std::mutex g_host_mu;
std::map<uintptr_t, size_t> g_host_blocks;

bool host_block_covers(const void* ptr, size_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host_blocks.upper_bound(a);
    if (it == g_host_blocks.begin()) return false;
    --it;
    return a >= it->first && a + bytes <= it->first + it->second;
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
    uint32_t* ne[2] = {nullptr, nullptr};  // non-empty-row bitmaps (Params::ne_tab), built on first use
    std::vector<uint32_t> h_ne[2];         // host copies, for the rows a query is seeded from (seed_ne)
};

struct rpq_graph {
    int device = 0;
    int32_t nv = 0;
    int32_t nl = 0;
    int sm_count = 0;
    std::vector<LabelDev> labels;
    std::mutex mu;
    int64_t bytes = 0;
    // device-ingested edge list (rpq_graph_create_coo): packed (src << 32 | dst)
    // keys grouped by label; labels are built from it on first use
    unsigned long long* d_coo = nullptr;
    std::vector<unsigned long long> coo_off;  // nl + 1 segment offsets
    // merged slots: the rows of several (label, inverted) symbols concatenated
    // per vertex, built when an automaton state reads them all into the same
    // targets (e.g. (a|b|c|d)*); keyed by the sorted symbol list
    std::map<std::vector<std::pair<int, int>>, LabelDev> merged;
};

struct rpq_query {
    rpq_graph* g = nullptr;
    int32_t nstates = 0;
    std::vector<int32_t> tables;  // kernel tables, layout of rpqk::Smem
    std::vector<Slot> slots;      // A_s for every slot, then A_s^T
    std::vector<unsigned long long> slot_nnz;
    int ngroups = 0, nslots = 0, ntargets = 0, nstarts = 0, nfinals = 0, nin = 0, maxT = 0;
    unsigned char* d_in = nullptr;  // per-run input block: RunArgs | slots | tables
    unsigned char* h_in = nullptr;  // its pinned host copy
    size_t in_bytes = 0, off_slots = 0, off_tables = 0;
    unsigned int bar_next = 0;      // barrier counter value the next run starts from
    unsigned long long* d_slot_nnz = nullptr;
    // Host copies of the non-empty-row bitmaps of the start states' push rows:
    // a source none of whose seed rows has an edge is answered without a
    // launch (query_eval).  Pointers into the labels' LabelDev::h_ne.
    std::vector<const uint32_t*> seed_ne;
    bool seed_ne_ok = false;
    bool start_is_final = false;
    int distinct_starts = 0;
    bool host_answered = false;  // the last query_eval did not run on the device (device state is stale)
    int32_t host_answered_source = 0;
    std::vector<const uint32_t*> ne_tab;   // per slot: non-empty-row bitmap of the transpose (Params::ne_tab)
    const uint32_t** d_ne_tab = nullptr;
    float dmax_ne = 0.0f;  // the densest slot's mean degree over non-empty rows
    int use_dmax_ne = 1;   // RPQ_TUNE_FLAGS bit 3 clears it (the round-1 all-rows mean)

    uint32_t* d_visited = nullptr;
    uint32_t* d_fb[3] = {nullptr, nullptr, nullptr};
    uint2* d_seg[2] = {nullptr, nullptr};
    uint2* d_bun[2] = {nullptr, nullptr};
    Ctl* d_ctl = nullptr;
    Ctl* h_ctl = nullptr;  // pinned
    Ctl* h_ctl_dev = nullptr;  // its device view (unified addressing)
    uint32_t* h_reach_bits_dev = nullptr;  // device view of h_reach_bits
    int zero_copy = 1;         // RPQ_TUNE_ZERO_COPY
    uint8_t* d_reach = nullptr;
    uint32_t* d_reach_bits = nullptr;
    uint32_t* h_reach_bits = nullptr;  // pinned; filled by run() when output_mode == 1
    int output_mode = 0;
    uint32_t* run_out_bits = nullptr;  // next run's caller-owned pinned answer buffer (rpq_query_eval)
    bool run_out_list = false;         // ... which may receive a (word index, word) pair list
    bool out_direct = false;           // the last run wrote its answer there, not to h_reach_bits
    bool reach_stale = true;           // d_reach (uint8) not yet expanded from d_reach_bits
    unsigned int run_seq = 0;          // number of the last rpq_query_run (Ctl::done_seq)
    bool last_zc = false;              // the last run's kernel writes the results prefix to the host

    cudaGraphExec_t graphs[4] = {nullptr, nullptr, nullptr, nullptr};  // captured run per variant
    cudaGraphExec_t graph = nullptr;  // the current variant's (one of graphs[])
    bool graph_failed = false;
    bool inflight = false;
    unsigned long long shard_segcap = 0, shard_buncap = 0, ovf_segcap = 0, ovf_buncap = 0;
    unsigned long long seg_alloc = 0, bun_alloc = 0;
    long long W = 0;
    int dir_mode = 0;
    int count_te = 0;
    int emit_mode = 0;
    unsigned int emit_inline_max = 1u << 16;
    unsigned int run_flags = RF_NO_PROBE;
    float defer_alpha = 1.5f;  // RPQ_TUNE_DEFER, with the non-empty-row degree (r02ab sweep: 3 mispredicts cfg5)
    long long own_w0 = 0, own_w1 = 0;  // owned word range (partitioned step); empty = all
    bool small_ok = false;    // |Q| x |V| fits the single-CTA kernel
    int allow_small = 1;      // RPQ_TUNE_SMALL
    size_t small_smem = 0;
    float alpha = 4.0f;
    cudaStream_t own_stream = nullptr;
    cudaStream_t last_stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int grid = 0;
    int nthreads = kThreads;  // ssr_kernel variant: kThreads or kThreadsLarge
    size_t smem = 0;
    bool ran = false;
    uint64_t edge_bound = 0;  // sum over groups of the slot's nnz
    unsigned long long* d_trace = nullptr;  // diagnostics (RPQ_TUNE_TRACE)
    unsigned int* d_step_acc = nullptr;     // step runs: non-empty steps, sticky failure status
    RunArgs step_ra{};                      // the input block of the last step_device run
    bool step_ra_valid = false;             // ... is what h_in holds (identical runs need no sync)
    int trace_levels = 0;

    // multi-source batch workspace (batch_kernel.cuh), allocated on first use
    SW* d_bvis = nullptr;
    SW* d_bfw[2] = {nullptr, nullptr};
    uint32_t* d_bact[2] = {nullptr, nullptr};
    BHeavy* d_bheavy = nullptr;
    size_t bsmem = 0;  // the batch kernel's dynamic shared memory
    uint32_t* d_blist = nullptr;  // the batch kernel's per-level active-block list
    BCtl* d_bctl = nullptr;
    BCtl* h_bctl = nullptr;  // pinned
    BatchArgs* d_bargs = nullptr;
    BatchArgs* h_bargs = nullptr;  // pinned
    uint32_t* d_bout = nullptr;
    long long bnvp = 0, bnblk = 0;
    unsigned long long bheavy_cap = 0;
    int bgrid = 0;
    int bnsrc = 0;
    unsigned int bbar_next = 0;
    bool binflight = false, bran = false;
    cudaStream_t blast_stream = nullptr;
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
    int* d_bad = nullptr;
    CUDA_TRY(cudaMalloc(&staging, (size_t)n_items * sizeof(I) + 16));
    d_bad = reinterpret_cast<int*>(reinterpret_cast<char*>(staging) + (size_t)n_items * sizeof(I));
    CUDA_TRY(cudaMemset(d_bad, 0, sizeof(int)));
    CUDA_TRY(cudaMalloc(&L.rowptr[dir], (size_t)(nv + 1) * sizeof(uint32_t)));
    CUDA_TRY(cudaMalloc(&L.col[dir], (size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t)));
    CUDA_TRY(cudaMemcpy(staging, indptr, (size_t)(nv + 1) * sizeof(I), cudaMemcpyHostToDevice));
    validate_csr_kernel<I><<<1184, 256>>>((const I*)staging, nv + 1, 0, nnz + 1, 1, d_bad);
    narrow_kernel<I, uint32_t><<<1184, 256>>>((const I*)staging, L.rowptr[dir], nv + 1);
    CUDA_TRY(cudaGetLastError());
    if (nnz > 0) {
        CUDA_TRY(cudaMemcpy(staging, indices, (size_t)nnz * sizeof(I), cudaMemcpyHostToDevice));
        validate_csr_kernel<I><<<1184, 256>>>((const I*)staging, nnz, 0, nv, 0, d_bad);
        narrow_kernel<I, int32_t><<<1184, 256>>>((const I*)staging, L.col[dir], nnz);
        CUDA_TRY(cudaGetLastError());
    }
    int bad = 0;
    CUDA_TRY(cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaFree(staging));
    if (bad) {
        cudaFree(L.rowptr[dir]);
        cudaFree(L.col[dir]);
        L.rowptr[dir] = nullptr;
        L.col[dir] = nullptr;
        return fail(RPQ_EINVAL, "CSR structure invalid: indptr must be non-decreasing and columns in [0, |V|)");
    }
    L.nnz[dir] = nnz;
    g->bytes += (nv + 1) * 4 + std::max<int64_t>(nnz, 1) * 4;
    return RPQ_OK;
}

void free_label(LabelDev& L) {
    for (int d = 0; d < 2; ++d) {
        if (L.rowptr[d]) cudaFree(L.rowptr[d]);
        if (L.col[d]) cudaFree(L.col[d]);
        if (L.ne[d]) cudaFree(L.ne[d]);
        L.h_ne[d].clear();
        L.rowptr[d] = nullptr;
        L.col[d] = nullptr;
        L.ne[d] = nullptr;
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

// Build label l's forward and backward CSR from the device edge list.
int materialize_label(rpq_graph* g, int32_t l) {
    LabelDev& L = g->labels[l];
    if (L.resident) return RPQ_OK;
    if (!g->d_coo) return fail(RPQ_ENOLABEL, "label " + std::to_string(l) + " is not resident");
    const unsigned long long lo = g->coo_off[l], n = g->coo_off[l + 1] - lo;
    const int64_t nv = g->nv;
    int bits = 1;
    while (bits < 32 && (1ll << bits) < nv) ++bits;
    unsigned long long *keys = nullptr, *tmp = nullptr;
    long long* d_nsel = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0, need = 0;
    auto cleanup = [&]() {
        if (keys) cudaFree(keys);
        if (tmp) cudaFree(tmp);
        if (d_nsel) cudaFree(d_nsel);
        if (temp) cudaFree(temp);
    };
#define MTRY(expr)                                                       \
    do {                                                                 \
        cudaError_t e_ = (expr);                                         \
        if (e_ != cudaSuccess) {                                         \
            cleanup();                                                   \
            free_label(L);                                               \
            return cuda_fail(e_, #expr);                                 \
        }                                                                \
    } while (0)
    const size_t nn = (size_t)std::max<unsigned long long>(n, 1);
    MTRY(cudaMalloc(&keys, nn * 8));
    MTRY(cudaMalloc(&tmp, nn * 8));
    MTRY(cudaMalloc(&d_nsel, sizeof(long long)));
    MTRY(cub::DeviceRadixSort::SortKeys(nullptr, need, keys, tmp, (int)0, 0, 64));
    temp_bytes = need;
    if (n > 0) {
        MTRY(cub::DeviceRadixSort::SortKeys(nullptr, need, keys, tmp, (long long)n, 0, 32 + bits));
        temp_bytes = std::max(temp_bytes, need);
        MTRY(cub::DeviceSelect::Unique(nullptr, need, tmp, keys, d_nsel, (long long)n));
        temp_bytes = std::max(temp_bytes, need);
    }
    MTRY(cudaMalloc(&temp, std::max<size_t>(temp_bytes, 16)));
    for (int dir = 0; dir < 2; ++dir) {
        long long m = 0;
        if (n > 0) {
            // keys of this direction into `keys`, sort into `tmp`, unique back into `keys`
            if (dir == 0)
                MTRY(cudaMemcpy(keys, g->d_coo + lo, n * 8, cudaMemcpyDeviceToDevice));
            else {
                swap_halves_kernel<<<1184, 256>>>(g->d_coo + lo, keys, (long long)n);
                MTRY(cudaGetLastError());
            }
            size_t tb = temp_bytes;
            MTRY(cub::DeviceRadixSort::SortKeys(temp, tb, keys, tmp, (long long)n, 0, 32 + bits));
            tb = temp_bytes;
            MTRY(cub::DeviceSelect::Unique(temp, tb, tmp, keys, d_nsel, (long long)n));
            long long nsel = 0;
            MTRY(cudaMemcpy(&nsel, d_nsel, sizeof(long long), cudaMemcpyDeviceToHost));
            m = nsel;
        }
        MTRY(cudaMalloc(&L.rowptr[dir], (size_t)(nv + 1) * sizeof(uint32_t)));
        MTRY(cudaMalloc(&L.col[dir], (size_t)std::max<long long>(m, 1) * sizeof(int32_t)));
        MTRY(cudaMemset(L.rowptr[dir], 0, (size_t)(nv + 1) * sizeof(uint32_t)));
        if (m > 0) {
            keys_to_csr_kernel<<<1184, 256>>>(keys, m, L.rowptr[dir], L.col[dir]);
            MTRY(cudaGetLastError());
            size_t tb = 0;
            MTRY(cub::DeviceScan::InclusiveSum(nullptr, tb, L.rowptr[dir], L.rowptr[dir], (int)(nv + 1)));
            void* t2 = nullptr;
            MTRY(cudaMalloc(&t2, std::max<size_t>(tb, 16)));
            cudaError_t e2 = cub::DeviceScan::InclusiveSum(t2, tb, L.rowptr[dir], L.rowptr[dir], (int)(nv + 1));
            cudaFree(t2);
            MTRY(e2);
        }
        L.nnz[dir] = m;
        g->bytes += (nv + 1) * 4 + std::max<long long>(m, 1) * 4;
    }
    MTRY(cudaDeviceSynchronize());
#undef MTRY
    cleanup();
    L.resident = true;
    return RPQ_OK;
}

// The merged adjacency of `syms` (each (label, inverted), resident) in both
// directions: direction d of the merged slot holds, per vertex, the rows of
// every symbol's direction-d matrix (its transpose for d = 1), concatenated.
// Duplicates across symbols are kept: a target reached twice is claimed once.
int build_merged(rpq_graph* g, const std::vector<std::pair<int, int>>& syms, LabelDev** out) {
    auto it = g->merged.find(syms);
    if (it != g->merged.end()) {
        *out = &it->second;
        return RPQ_OK;
    }
    LabelDev M;
    const long long nv = g->nv;
    const int k = (int)syms.size();
    const uint32_t** d_rp = nullptr;
    const int32_t** d_cl = nullptr;
    void* temp = nullptr;
    auto cleanup = [&]() {
        if (d_rp) cudaFree(d_rp);
        if (d_cl) cudaFree(d_cl);
        if (temp) cudaFree(temp);
    };
#define GTRY(expr)                         \
    do {                                   \
        cudaError_t e_ = (expr);           \
        if (e_ != cudaSuccess) {           \
            cleanup();                     \
            free_label(M);                 \
            return cuda_fail(e_, #expr);   \
        }                                  \
    } while (0)
    GTRY(cudaMalloc(&d_rp, sizeof(uint32_t*) * k));
    GTRY(cudaMalloc(&d_cl, sizeof(int32_t*) * k));
    for (int dir = 0; dir < 2; ++dir) {
        std::vector<const uint32_t*> rp(k);
        std::vector<const int32_t*> cl(k);
        unsigned long long nnz = 0;
        for (int i = 0; i < k; ++i) {
            const LabelDev& L = g->labels[syms[i].first];
            const int d = dir == 0 ? syms[i].second : 1 - syms[i].second;
            rp[i] = L.rowptr[d];
            cl[i] = L.col[d];
            nnz += (unsigned long long)L.nnz[d];
        }
        if (nnz > 0xFFFFFFFFull) {
            cleanup();
            free_label(M);
            return fail(RPQ_EINVAL, "merged adjacency would exceed 2^32 edges");
        }
        GTRY(cudaMemcpy(d_rp, rp.data(), sizeof(uint32_t*) * k, cudaMemcpyHostToDevice));
        GTRY(cudaMemcpy(d_cl, cl.data(), sizeof(int32_t*) * k, cudaMemcpyHostToDevice));
        GTRY(cudaMalloc(&M.rowptr[dir], (size_t)(nv + 1) * 4));
        GTRY(cudaMalloc(&M.col[dir], (size_t)std::max<unsigned long long>(nnz, 1) * 4));
        GTRY(cudaMemset(M.rowptr[dir], 0, (size_t)(nv + 1) * 4));
        if (nv > 0) {
            merge_degree_kernel<<<1184, 256>>>(d_rp, k, nv, M.rowptr[dir]);
            GTRY(cudaGetLastError());
            size_t tb = 0;
            GTRY(cub::DeviceScan::InclusiveSum(nullptr, tb, M.rowptr[dir], M.rowptr[dir], (int)(nv + 1)));
            GTRY(cudaMalloc(&temp, std::max<size_t>(tb, 16)));
            GTRY(cub::DeviceScan::InclusiveSum(temp, tb, M.rowptr[dir], M.rowptr[dir], (int)(nv + 1)));
            cudaFree(temp);
            temp = nullptr;
            merge_copy_kernel<<<1184, 256>>>(d_rp, d_cl, k, nv, M.rowptr[dir], M.col[dir]);
            GTRY(cudaGetLastError());
        }
        M.nnz[dir] = (int64_t)nnz;
        g->bytes += (nv + 1) * 4 + (int64_t)std::max<unsigned long long>(nnz, 1) * 4;
    }
    GTRY(cudaDeviceSynchronize());
#undef GTRY
    cleanup();
    M.resident = true;
    auto res = g->merged.emplace(syms, M);
    *out = &res.first->second;
    return RPQ_OK;
}

void free_query_buffers(rpq_query* q) {
    if (q->d_in) cudaFree(q->d_in);
    if (q->h_in) cudaFreeHost(q->h_in);
    if (q->d_slot_nnz) cudaFree(q->d_slot_nnz);
    if (q->d_ne_tab) cudaFree(q->d_ne_tab);
    if (q->d_visited) cudaFree(q->d_visited);
    for (int f = 0; f < 3; ++f)
        if (q->d_fb[f]) cudaFree(q->d_fb[f]);
    for (int b = 0; b < 2; ++b) {
        if (q->d_seg[b]) cudaFree(q->d_seg[b]);
        if (q->d_bun[b]) cudaFree(q->d_bun[b]);
    }

    if (q->d_ctl) cudaFree(q->d_ctl);
    if (q->d_step_acc) cudaFree(q->d_step_acc);
    if (q->h_ctl) cudaFreeHost(q->h_ctl);
    if (q->d_reach) cudaFree(q->d_reach);
    if (q->d_reach_bits) cudaFree(q->d_reach_bits);
    if (q->h_reach_bits) cudaFreeHost(q->h_reach_bits);

    if (q->d_trace) cudaFree(q->d_trace);
    if (q->d_bvis) cudaFree(q->d_bvis);
    for (int b = 0; b < 2; ++b) {
        if (q->d_bfw[b]) cudaFree(q->d_bfw[b]);
        if (q->d_bact[b]) cudaFree(q->d_bact[b]);
    }
    if (q->d_bheavy) cudaFree(q->d_bheavy);
    if (q->d_blist) cudaFree(q->d_blist);
    if (q->d_bctl) cudaFree(q->d_bctl);
    if (q->h_bctl) cudaFreeHost(q->h_bctl);
    if (q->d_bargs) cudaFree(q->d_bargs);
    if (q->h_bargs) cudaFreeHost(q->h_bargs);
    if (q->d_bout) cudaFree(q->d_bout);

    for (auto& gx : q->graphs)
        if (gx) cudaGraphExecDestroy(gx);
    if (q->ev0) cudaEventDestroy(q->ev0);
    if (q->ev1) cudaEventDestroy(q->ev1);
    if (q->own_stream) cudaStreamDestroy(q->own_stream);
}

// A kernel's dynamic shared memory limit belongs to the function, shared by
// every query and graph: raise it once to the device's opt-in maximum (each
// launch still passes its own size).  Setting it to one query's size would
// make an earlier, larger query's launches fail.
cudaError_t allow_dyn_smem(const void* fn) {
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return e;
    const int cap = optin - (int)fa.sharedSizeBytes;
    if (fa.maxDynamicSharedSizeBytes >= cap) return cudaSuccess;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
}

}  // namespace

extern "C" {

int rpq_abi_version(void) { return RPQ_ABI_VERSION; }

int rpq_checked_build(void) {
#ifdef RPQ_CHECKED
    return 1;
#else
    return 0;
#endif
}

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

int rpq_graph_create_coo(int32_t num_vertices, int32_t num_labels, int64_t nnz, const int32_t* src,
                         const int32_t* dst, const int32_t* label, int32_t device, rpq_graph** out) {
    if (!out) return fail(RPQ_EINVAL, "null output handle");
    *out = nullptr;
    if (nnz < 0 || (nnz > 0 && (!src || !dst || !label))) return fail(RPQ_EINVAL, "null edge array");
    rpq_graph* g = nullptr;
    int rc = rpq_graph_create(num_vertices, num_labels, device, &g);
    if (rc != RPQ_OK) return rc;
    for (int64_t i = 0; i < nnz; i += 1 << 20) {  // validate on the host (cheap next to the upload)
        const int64_t hi = std::min<int64_t>(nnz, i + (1 << 20));
        for (int64_t j = i; j < hi; ++j)
            if (src[j] < 0 || src[j] >= num_vertices || dst[j] < 0 || dst[j] >= num_vertices || label[j] < 0 ||
                label[j] >= num_labels) {
                rpq_graph_destroy(g);
                return fail(RPQ_EINVAL, "edge " + std::to_string(j) + " out of range");
            }
    }
    int32_t *d_src = nullptr, *d_dst = nullptr, *d_lab = nullptr;
    unsigned long long *hist = nullptr, *cursor = nullptr;
    auto cleanup = [&]() {
        if (d_src) cudaFree(d_src);
        if (d_dst) cudaFree(d_dst);
        if (d_lab) cudaFree(d_lab);
        if (hist) cudaFree(hist);
        if (cursor) cudaFree(cursor);
    };
#define GTRY(expr)                                \
    do {                                          \
        cudaError_t e_ = (expr);                  \
        if (e_ != cudaSuccess) {                  \
            cleanup();                            \
            rpq_graph_destroy(g);                 \
            return cuda_fail(e_, #expr);          \
        }                                         \
    } while (0)
    const size_t nn = (size_t)std::max<int64_t>(nnz, 1);
    GTRY(cudaMalloc(&d_src, nn * 4));
    GTRY(cudaMalloc(&d_dst, nn * 4));
    GTRY(cudaMalloc(&d_lab, nn * 4));
    GTRY(cudaMalloc(&g->d_coo, nn * 8));
    GTRY(cudaMalloc(&hist, (size_t)(num_labels + 1) * 8));
    GTRY(cudaMalloc(&cursor, (size_t)(num_labels + 1) * 8));
    if (nnz > 0) {
        GTRY(cudaMemcpy(d_src, src, nnz * 4, cudaMemcpyHostToDevice));
        GTRY(cudaMemcpy(d_dst, dst, nnz * 4, cudaMemcpyHostToDevice));
        GTRY(cudaMemcpy(d_lab, label, nnz * 4, cudaMemcpyHostToDevice));
    }
    GTRY(cudaMemset(hist, 0, (size_t)(num_labels + 1) * 8));
    const int nl = num_labels;
    if (nnz > 0 && nl > 0) {
        const size_t sh = nl <= 8192 ? (size_t)nl * 4 : 0;
        label_histogram_kernel<<<1184, 256, sh>>>(d_lab, nnz, nl, hist);
        GTRY(cudaGetLastError());
    }
    std::vector<unsigned long long> h(nl + 1, 0);
    if (nl > 0) GTRY(cudaMemcpy(h.data(), hist, (size_t)nl * 8, cudaMemcpyDeviceToHost));
    g->coo_off.assign(nl + 1, 0);
    for (int l = 0; l < nl; ++l) g->coo_off[l + 1] = g->coo_off[l] + h[l];
    if (nl > 0) GTRY(cudaMemcpy(cursor, g->coo_off.data(), (size_t)nl * 8, cudaMemcpyHostToDevice));
    if (nnz > 0 && nl > 0) {
        // shared memory: nl counters (padded to even) + nl 64-bit range bases
        const size_t sm = nl <= 8192 ? (size_t)((nl + 1) & ~1) * 4 + (size_t)nl * 8 : 0;
        if (sm > 48 * 1024) GTRY(allow_dyn_smem((const void*)label_scatter_kernel));
        label_scatter_kernel<<<1184, 256, sm>>>(d_src, d_dst, d_lab, nnz, nl, cursor, g->d_coo);
        GTRY(cudaGetLastError());
    }
    GTRY(cudaDeviceSynchronize());
#undef GTRY
    cleanup();
    g->bytes += (int64_t)nn * 8;
    *out = g;
    return RPQ_OK;
}

int rpq_graph_materialize_label(rpq_graph* g, int32_t label) {
    if (!g) return fail(RPQ_EINVAL, "null graph");
    if (label < 0 || label >= g->nl) return fail(RPQ_EINVAL, "label index out of range");
    std::lock_guard<std::mutex> lk(g->mu);
    if (cudaSetDevice(g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    return materialize_label(g, label);
}

int rpq_graph_copy_label(const rpq_graph* g, int32_t label, int32_t transpose, uint32_t* rowptr, int32_t* col,
                         int64_t col_capacity, int64_t* nnz) {
    if (!g || label < 0 || label >= g->nl) return fail(RPQ_EINVAL, "bad graph or label");
    const LabelDev& L = g->labels[label];
    if (!L.resident) return fail(RPQ_ENOLABEL, "label " + std::to_string(label) + " is not resident");
    const int d = transpose ? 1 : 0;
    if (nnz) *nnz = L.nnz[d];
    if (cudaSetDevice(g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    if (rowptr)
        CUDA_TRY(cudaMemcpy(rowptr, L.rowptr[d], ((size_t)g->nv + 1) * 4, cudaMemcpyDeviceToHost));
    if (col) {
        if (col_capacity < L.nnz[d]) return fail(RPQ_EINVAL, "column buffer too small");
        if (L.nnz[d] > 0) CUDA_TRY(cudaMemcpy(col, L.col[d], (size_t)L.nnz[d] * 4, cudaMemcpyDeviceToHost));
    }
    return RPQ_OK;
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
    for (auto& kv : g->merged) free_label(kv.second);
    if (g->d_coo) cudaFree(g->d_coo);
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

    // usable transitions -> slots (label, inv), push groups (state, slot) ->
    // targets, pull in-transitions target -> (source state, slot)
    std::map<std::pair<int, int>, int> slot_of;
    std::vector<std::pair<int, int>> slot_keys;
    std::map<std::pair<int, int>, std::set<int>> group_targets;
    std::map<int, std::set<std::pair<int, int>>> in_trans;
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
            const int sl = slot_of[{t_label[i], t_inv[i] ? 1 : 0}];
            group_targets[{t_src[i], sl}].insert(t_dst[i]);
            in_trans[t_dst[i]].insert({t_src[i], sl});
        }
    }
    if ((int)slot_keys.size() > kMaxSlots) return fail(RPQ_EINVAL, "too many distinct symbols");
    if ((int)group_targets.size() > kMaxGroups)
        return fail(RPQ_EINVAL, "automaton has more than 256 (state, symbol) groups");
    // slot entries: direction 0 = the push matrix A_s, 1 = its transpose
    struct SlotEnt {
        const uint32_t* rowptr[2];
        const int32_t* col[2];
        int64_t nnz[2];
        LabelDev* ne_of;     // the label whose direction ne_dir is the transpose (its non-empty-row
        int ne_dir;          // bitmap is built after the query's own buffers are allocated)
        int push_dir;        // ... and whose direction push_dir is the push matrix A_s
    };
    // words per bitmap row, as the query's bitmaps are laid out (a multiple of 4)
    const long long ne_words = (((long long)g->nv + 31) / 32 + 3) / 4 * 4;
    auto ensure_ne = [&](LabelDev& L, int d) -> const uint32_t* {
        if (L.ne[d] || !L.rowptr[d]) return L.ne[d];
        if (cudaMalloc(&L.ne[d], (size_t)ne_words * sizeof(uint32_t)) != cudaSuccess) {
            L.ne[d] = nullptr;  // (the kernel falls back to reading row pointers)
            cudaGetLastError();
            return nullptr;
        }
        nonempty_bitmap_kernel<<<4 * g->sm_count, 256>>>(L.rowptr[d], g->nv, L.ne[d], ne_words);
        // (query streams do not synchronize with the default stream: finish it here, once per label)
        if (cudaStreamSynchronize(0) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(L.ne[d]);
            L.ne[d] = nullptr;
            return nullptr;
        }
        g->bytes += ne_words * (long long)sizeof(uint32_t);
        return L.ne[d];
    };
    std::vector<SlotEnt> ents;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (cudaSetDevice(g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
        for (auto& k : slot_keys) {
            const int rc = materialize_label(g, k.first);  // device edge list, if any
            if (rc != RPQ_OK) return rc;
            LabelDev& L = g->labels[k.first];
            ents.push_back(SlotEnt{{L.rowptr[k.second], L.rowptr[1 - k.second]},
                                   {L.col[k.second], L.col[1 - k.second]},
                                   {L.nnz[k.second], L.nnz[1 - k.second]},
                                   &L, 1 - k.second, k.second});
        }
        // A state that reads several symbols into the same targets (e.g. the
        // one state of (a|b|c|d)*) gets one merged slot: its rows are the
        // symbols' rows concatenated, so a pair costs one row-pointer read and
        // one column run instead of one per symbol; pull in-rows likewise.
        // RPQ_MERGE=0 in the environment turns this off (A/B measurements).
        const char* env = std::getenv("RPQ_MERGE");
        if (!(env && env[0] == '0')) {
            std::map<std::pair<int, std::set<int>>, std::vector<int>> buckets;
            for (auto& kv : group_targets) buckets[{kv.first.first, kv.second}].push_back(kv.first.second);
            std::map<std::vector<std::pair<int, int>>, int> merged_slot;
            std::map<std::pair<int, int>, std::set<int>> ng;
            std::map<int, std::set<std::pair<int, int>>> nin;
            for (auto& b : buckets) {
                const int st = b.first.first;
                int sl = b.second[0];
                if (b.second.size() >= 2) {
                    std::vector<std::pair<int, int>> syms;
                    for (int x : b.second) syms.push_back(slot_keys[x]);
                    std::sort(syms.begin(), syms.end());
                    auto f = merged_slot.find(syms);
                    if (f != merged_slot.end()) {
                        sl = f->second;
                    } else {
                        LabelDev* M = nullptr;
                        const int rc = build_merged(g, syms, &M);
                        if (rc != RPQ_OK) return rc;
                        sl = (int)ents.size();
                        ents.push_back(SlotEnt{{M->rowptr[0], M->rowptr[1]}, {M->col[0], M->col[1]},
                                               {M->nnz[0], M->nnz[1]}, M, 1, 0});
                        merged_slot[syms] = sl;
                    }
                }
                ng[{st, sl}] = b.first.second;
                for (int t : b.first.second) nin[t].insert({st, sl});
            }
            // in-transitions are the same relation read by target: rebuilt from the groups
            group_targets.swap(ng);
            in_trans.swap(nin);
        }
    }
    if ((int)ents.size() > kMaxSlots) return fail(RPQ_EINVAL, "too many distinct symbols");

    rpq_query* q = new rpq_query();
    q->g = g;
    q->nstates = nstates;
    std::vector<int32_t> gbeg(nstates + 1, 0), gslot, toff, targets, ibeg(nstates + 1, 0), isrc,
        islot;
    std::vector<int> gcount(nstates, 0);
    for (auto& kv : group_targets) gcount[kv.first.first]++;
    for (int st = 0; st < nstates; ++st) gbeg[st + 1] = gbeg[st] + gcount[st];
    // std::map iterates (state, slot) in order, so a state's groups are contiguous
    int maxT = 0;
    toff.push_back(0);
    uint64_t groups_total = 0, edge_bound = 0;
    for (auto& kv : group_targets) {
        gslot.push_back(kv.first.second);
        for (int t : kv.second) targets.push_back(t);
        toff.push_back((int32_t)targets.size());
        maxT = std::max<int>(maxT, (int)kv.second.size());
        groups_total += 1;
        edge_bound += (uint64_t)ents[kv.first.second].nnz[0];
    }
    for (int st = 0; st < nstates; ++st) {
        auto it = in_trans.find(st);
        if (it != in_trans.end())
            for (auto& e : it->second) {
                isrc.push_back(e.first);
                islot.push_back(e.second);
            }
        ibeg[st + 1] = (int32_t)isrc.size();
    }
    std::set<int> sset, fset;
    for (int i = 0; i < nstarts; ++i)
        if (starts[i] >= 0 && starts[i] < nstates) sset.insert(starts[i]);
    for (int i = 0; i < nfinals; ++i)
        if (finals[i] >= 0 && finals[i] < nstates) fset.insert(finals[i]);
    q->edge_bound = edge_bound;
    q->ngroups = (int)gslot.size();
    q->nslots = (int)ents.size();
    q->ntargets = (int)targets.size();
    q->nstarts = (int)sset.size();
    q->nfinals = (int)fset.size();
    q->nin = (int)isrc.size();
    q->maxT = maxT;
    auto& T = q->tables;
    T.insert(T.end(), gbeg.begin(), gbeg.end());
    T.insert(T.end(), gslot.begin(), gslot.end());
    T.insert(T.end(), toff.begin(), toff.end());
    T.insert(T.end(), targets.begin(), targets.end());
    T.insert(T.end(), sset.begin(), sset.end());
    T.insert(T.end(), fset.begin(), fset.end());
    T.insert(T.end(), ibeg.begin(), ibeg.end());
    T.insert(T.end(), isrc.begin(), isrc.end());
    T.insert(T.end(), islot.begin(), islot.end());
    for (int pass = 0; pass < 2; ++pass)  // pass 1: the transposes
        for (auto& en : ents) q->slots.push_back(Slot{en.rowptr[pass], en.col[pass]});

    for (auto& en : ents) q->slot_nnz.push_back((unsigned long long)en.nnz[0]);

    // queue capacities: every (state, vertex) pair is discovered at most once,
    // so one level holds at most |V| segments per group (+ splits of huge
    // rows); bundles are at most one partial per emission plus edges/kBundle.
    const unsigned long long nv = (unsigned long long)g->nv;
    const unsigned long long segbound = nv * groups_total + edge_bound / kSegLenMax + 64;
    const unsigned long long bunbound = segbound + edge_bound / kBundle + 64;
    q->shard_segcap = segbound / kShards + segbound / (4 * kShards) + 1024;
    q->shard_buncap = bunbound / kShards + bunbound / (4 * kShards) + 1024;
    q->ovf_segcap = segbound;
    q->ovf_buncap = bunbound;
    q->seg_alloc = q->shard_segcap * kShards + q->ovf_segcap + 32;
    q->bun_alloc = q->shard_buncap * kShards + q->ovf_buncap;
    if (q->seg_alloc >= 0xFFFFFFFFull || q->shard_buncap >= 0xFFFFFFFFull ||
        q->ovf_buncap >= 0xFFFFFFFFull) {
        delete q;
        return fail(RPQ_EINVAL, "frontier queue would exceed 2^32 entries");
    }
    q->W = (((long long)g->nv + 31) / 32 + 3) / 4 * 4;

    auto bail = [&](int rc) {
        free_query_buffers(q);
        delete q;
        return rc;
    };
    if (cudaSetDevice(g->device) != cudaSuccess) return bail(fail(RPQ_ECUDA, "cudaSetDevice"));
#define QTRY(expr)                                                \
    do {                                                          \
        cudaError_t e_ = (expr);                                  \
        if (e_ != cudaSuccess) return bail(cuda_fail(e_, #expr)); \
    } while (0)
    const size_t bitmap_bytes = (size_t)q->W * nstates * sizeof(uint32_t);
    q->off_slots = (sizeof(RunArgs) + 15) / 16 * 16;
    q->off_tables = q->off_slots + q->slots.size() * sizeof(Slot);
    q->in_bytes = q->off_tables + std::max<size_t>(T.size(), 1) * sizeof(int32_t);
    QTRY(cudaMalloc(&q->d_in, q->in_bytes));
    QTRY(cudaMallocHost(&q->h_in, q->in_bytes));
    QTRY(cudaMalloc(&q->d_slot_nnz, std::max<size_t>(q->slot_nnz.size(), 1) * sizeof(unsigned long long)));
    QTRY(cudaMalloc(&q->d_visited, bitmap_bytes));
    for (int f = 0; f < 3; ++f) QTRY(cudaMalloc(&q->d_fb[f], bitmap_bytes));
    for (int b = 0; b < 2; ++b) {
        QTRY(cudaMalloc(&q->d_seg[b], (size_t)q->seg_alloc * sizeof(uint2)));
        QTRY(cudaMalloc(&q->d_bun[b], (size_t)q->bun_alloc * sizeof(uint2)));
        // a consumer reads up to 32 segments past a bundle's own; keep them
        // finite so its scan cannot wrap
        QTRY(cudaMemset(q->d_seg[b], 0, (size_t)q->seg_alloc * sizeof(uint2)));
    }
    QTRY(cudaMalloc(&q->d_ctl, sizeof(Ctl)));
    QTRY(cudaMalloc(&q->d_step_acc, 2 * sizeof(unsigned int)));
    QTRY(cudaMemset(q->d_step_acc, 0, 2 * sizeof(unsigned int)));
    QTRY(cudaMallocHost(&q->h_ctl, sizeof(Ctl)));
    QTRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&q->h_ctl_dev), q->h_ctl, 0));
    QTRY(cudaMalloc(&q->d_reach, (size_t)(q->W * 32 + 32)));
    QTRY(cudaMalloc(&q->d_reach_bits, (size_t)q->W * sizeof(uint32_t)));
    QTRY(cudaMallocHost(&q->h_reach_bits, (size_t)q->W * sizeof(uint32_t)));
    QTRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&q->h_reach_bits_dev), q->h_reach_bits, 0));

    QTRY(cudaStreamCreateWithFlags(&q->own_stream, cudaStreamNonBlocking));
    QTRY(cudaEventCreate(&q->ev0));
    QTRY(cudaEventCreate(&q->ev1));
    std::memset(q->h_in, 0, q->in_bytes);
    if (!q->slots.empty()) std::memcpy(q->h_in + q->off_slots, q->slots.data(), q->slots.size() * sizeof(Slot));
    if (!T.empty()) std::memcpy(q->h_in + q->off_tables, T.data(), T.size() * sizeof(int32_t));
    QTRY(cudaMemset(q->d_ctl, 0, sizeof(Ctl)));
    {   // mean degree over non-empty rows, per push slot (the defer predictor)
        unsigned long long* d_cnt = nullptr;
        QTRY(cudaMalloc(&d_cnt, sizeof(unsigned long long)));
        for (size_t i = 0; i < ents.size(); ++i) {
            if (!ents[i].rowptr[0] || q->slot_nnz[i] == 0) continue;
            unsigned long long rows = 0;
            QTRY(cudaMemset(d_cnt, 0, sizeof(unsigned long long)));
            count_nonempty_kernel<<<4 * g->sm_count, 256>>>(ents[i].rowptr[0], g->nv, d_cnt);
            QTRY(cudaMemcpy(&rows, d_cnt, sizeof(rows), cudaMemcpyDeviceToHost));
            if (rows) q->dmax_ne = std::max(q->dmax_ne, (float)((double)q->slot_nnz[i] / (double)rows));
        }
        cudaFree(d_cnt);
    }
    if (!q->slot_nnz.empty())
        QTRY(cudaMemcpy(q->d_slot_nnz, q->slot_nnz.data(), q->slot_nnz.size() * sizeof(unsigned long long),
                        cudaMemcpyHostToDevice));
    {   // non-empty-row bitmaps of the pulled (transposed) slots, cached per label
        std::lock_guard<std::mutex> lk(g->mu);
        for (auto& en : ents) {
            q->ne_tab.push_back(ensure_ne(*en.ne_of, en.ne_dir));
            if (!q->ne_tab.back() && en.rowptr[1]) return bail(fail(RPQ_ECUDA, "out of device memory (row bitmaps)"));
        }
        // the start states' push rows, on the host: which sources have any seed edge at all
        q->seed_ne_ok = true;
        std::set<int> seen_start;
        for (int i = 0; i < nstarts && q->seed_ne_ok; ++i) {
            if (!seen_start.insert(starts[i]).second) continue;
            for (int gi = gbeg[starts[i]]; gi < gbeg[starts[i] + 1] && q->seed_ne_ok; ++gi) {
                SlotEnt& en = ents[gslot[gi]];
                if (en.nnz[0] == 0) continue;  // (no edges: no seed edge)
                LabelDev& L = *en.ne_of;
                const int d = en.push_dir;
                if (L.h_ne[d].empty()) {
                    const uint32_t* dev = ensure_ne(L, d);
                    if (!dev) {
                        q->seed_ne_ok = false;
                        break;
                    }
                    L.h_ne[d].resize((size_t)ne_words);
                    if (cudaMemcpy(L.h_ne[d].data(), dev, (size_t)ne_words * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost) != cudaSuccess) {
                        cudaGetLastError();
                        L.h_ne[d].clear();
                        q->seed_ne_ok = false;
                        break;
                    }
                }
                q->seed_ne.push_back(L.h_ne[d].data());
            }
        }
        q->distinct_starts = (int)seen_start.size();
        for (int i = 0; i < nfinals; ++i) q->start_is_final |= seen_start.count(finals[i]) != 0;
    }
    if (!q->ne_tab.empty()) {
        QTRY(cudaMalloc(&q->d_ne_tab, q->ne_tab.size() * sizeof(const uint32_t*)));
        QTRY(cudaMemcpy(q->d_ne_tab, q->ne_tab.data(), q->ne_tab.size() * sizeof(const uint32_t*),
                        cudaMemcpyHostToDevice));
    }
    // large state spaces: the 32-warp variant (more loads in flight); small: 24 warps
    bool large = (long long)nstates * (long long)g->nv >= kLargePairs;
    if (const char* ev = std::getenv("RPQ_KERNEL_THREADS")) {  // experiments: force a variant
        if (std::atoi(ev) == kThreads) large = false;
        if (std::atoi(ev) == kThreadsLarge) large = true;
    }
    q->nthreads = large ? kThreadsLarge : kThreads;
    q->smem = kStageBytes(q->nthreads) + q->slots.size() * sizeof(Slot) + T.size() * sizeof(int32_t) + 16;
    const void* kfn = large ? (const void*)ssr_kernel<kThreadsLarge> : (const void*)ssr_kernel<kThreads>;
    QTRY(allow_dyn_smem(kfn));
    int per_sm = 0;
    QTRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, q->nthreads, q->smem));
    if (per_sm < 1) return bail(fail(RPQ_ECUDA, "step kernel cannot be resident"));
    q->grid = std::min(g->sm_count * per_sm, kShards);  // one queue shard per CTA
    if ((long long)nstates * q->W <= kSmallMaxWords) {
        q->small_smem = q->slots.size() * sizeof(Slot) + (T.size() * sizeof(int32_t) + 15) / 16 * 16 +
                        3 * (size_t)nstates * (size_t)q->W * sizeof(uint32_t);
        if (q->small_smem <= 200 * 1024) {
            QTRY(allow_dyn_smem((const void*)small_kernel));
            q->small_ok = true;
        }
    }
#undef QTRY
    *out = q;
    return RPQ_OK;
}

int rpq_query_set_options(rpq_query* q, int32_t direction, int32_t count_te, double alpha) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (direction < RPQ_DIR_AUTO || direction > RPQ_DIR_PULL) return fail(RPQ_EINVAL, "bad direction");
    if (!(alpha > 0)) return fail(RPQ_EINVAL, "alpha must be > 0");
    q->dir_mode = direction;
    q->count_te = count_te ? 1 : 0;
    q->alpha = (float)alpha;
    return RPQ_OK;
}

namespace {

Params make_params(const rpq_query* q) {
    Params p{};
    p.run = reinterpret_cast<const RunArgs*>(q->d_in);
    p.tables = reinterpret_cast<const int32_t*>(q->d_in + q->off_tables);
    p.slots = reinterpret_cast<const Slot*>(q->d_in + q->off_slots);
    p.slot_nnz = q->d_slot_nnz;
    p.ne_tab = q->d_ne_tab;
    p.visited = q->d_visited;
    for (int f = 0; f < 3; ++f) p.fb[f] = q->d_fb[f];
    for (int b = 0; b < 2; ++b) {
        p.seg[b] = q->d_seg[b];
        p.bun[b] = q->d_bun[b];
    }
    p.ctl = q->d_ctl;
    p.host_ctl = q->zero_copy ? q->h_ctl_dev : nullptr;
    p.host_bits = q->zero_copy && q->output_mode == 1 ? q->h_reach_bits_dev : nullptr;
    p.reach = q->d_reach;
    p.reach_bits = q->d_reach_bits;
    p.shard_segcap = q->shard_segcap;
    p.shard_buncap = q->shard_buncap;
    p.ovf_segcap = q->ovf_segcap;
    p.ovf_buncap = q->ovf_buncap;
    p.seg_alloc = q->seg_alloc;
    p.bun_alloc = q->bun_alloc;
    p.W = q->W;
    p.nv = q->g->nv;
    p.nstates = q->nstates;
    p.ngroups = q->ngroups;
    p.nslots = q->nslots;
    p.ntargets = q->ntargets;
    p.nstarts = q->nstarts;
    p.nfinals = q->nfinals;
    p.nin = q->nin;
    p.maxT = q->maxT;
    p.table_ints = (int)q->tables.size();
    p.trace = q->d_trace;
    p.trace_levels = q->d_trace ? q->trace_levels : 0;
    p.step_acc = q->d_step_acc;
    p.dmax_ne = q->use_dmax_ne ? q->dmax_ne : 0.0f;
    return p;
}

// The run sequence: inputs H2D (run block + automaton tables, pinned), control
// block reset, the cooperative kernel, statistics (and answer bitmap) D2H.
// The single-CTA kernel runs a full evaluation when the state space fits its
// shared memory (and no pull levels were asked for).
bool use_small(const rpq_query* q) { return q->small_ok && q->allow_small && q->dir_mode != RPQ_DIR_PULL; }

cudaError_t enqueue_run(rpq_query* q, cudaStream_t st, const Params* override = nullptr, bool small = false) {
    cudaError_t e;
    // inputs: run arguments + automaton tables in one pinned block (a copy
    // node: the kernel prologue reading them from host memory instead was
    // 65 us slower on cfg2 -- 148 CTAs of small uncached PCIe reads)
    if ((e = cudaMemcpyAsync(q->d_in, q->h_in, q->in_bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return e;
    Params p = override ? *override : make_params(q);
    if (small) {  // (the single-CTA kernel's block and answer are copied below)
        p.host_ctl = nullptr;
        p.host_bits = nullptr;
    }
    if (override) p.host_bits = nullptr;  // a step projects no answer
    void* args[] = {&p};
    if (small) {
        small_kernel<<<1, kSmallThreads, q->small_smem, st>>>(p);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else if ((e = cudaLaunchCooperativeKernel(q->nthreads == kThreadsLarge ? (const void*)ssr_kernel<kThreadsLarge>
                                                                             : (const void*)ssr_kernel<kThreads>,
                                                dim3(q->grid), dim3(q->nthreads), args, q->smem, st)) != cudaSuccess) {
        return e;
    }
    // outputs: the control block's results prefix (and the answer bitmap)
    if (!p.host_ctl &&
        (e = cudaMemcpyAsync(q->h_ctl, q->d_ctl, offsetof(Ctl, qc), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return e;
    // (a step-mode run, `override`, projects no answer: nothing to copy)
    if (q->output_mode == 1 && !override && !p.host_bits && q->g->nv > 0 &&
        (e = cudaMemcpyAsync(q->h_reach_bits, q->d_reach_bits, (size_t)((q->g->nv + 31) / 32) * 4,
                             cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return e;
    return cudaSuccess;
}

// Capture enqueue_run into a graph once per output mode: one cudaGraphLaunch
// per run.  Falls back to direct launches if capture is not possible.
void build_graph(rpq_query* q) {
    const int variant = q->output_mode | (use_small(q) ? 2 : 0);
    q->graph = q->graphs[variant];
    if (q->graph) return;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(q->own_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        q->graph_failed = true;
        return;
    }
    cudaError_t e = enqueue_run(q, q->own_stream, nullptr, use_small(q));
    cudaError_t e2 = cudaStreamEndCapture(q->own_stream, &g);
    if (e != cudaSuccess || e2 != cudaSuccess || !g ||
        cudaGraphInstantiate(&q->graphs[variant], g, 0) != cudaSuccess) {
        cudaGetLastError();
        q->graphs[variant] = nullptr;
        q->graph_failed = true;
    }
    q->graph = q->graphs[variant];
    if (g) cudaGraphDestroy(g);
}

// Captured runs hold the parameters of their capture: drop them all.
void drop_graphs(rpq_query* q) {
    for (auto& gx : q->graphs)
        if (gx) {
            cudaGraphExecDestroy(gx);
            gx = nullptr;
        }
    q->graph = nullptr;
}

}  // namespace

int rpq_query_set_tuning(rpq_query* q, int32_t key, double value) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    switch (key) {
        case RPQ_TUNE_EMIT_MODE:
            if (value < 0 || value > 2) return fail(RPQ_EINVAL, "emit mode must be 0, 1 or 2");
            q->emit_mode = (int)value;
            return RPQ_OK;
        case RPQ_TUNE_EMIT_INLINE_MAX:
            if (value < 0 || value > 4.0e9) return fail(RPQ_EINVAL, "bad inline threshold");
            q->emit_inline_max = (unsigned int)value;
            return RPQ_OK;
        case RPQ_TUNE_ZERO_COPY:
            if (value != 0 && value != 1) return fail(RPQ_EINVAL, "zero-copy switch must be 0 or 1");
            q->zero_copy = (int)value;
            if (q->inflight) {  // let a run in flight finish with the old graph
                CUDA_TRY(cudaStreamSynchronize(q->last_stream));
                q->bar_next = q->h_ctl->bar;
                q->inflight = false;
            }
            drop_graphs(q);  // the captured runs hold the old parameters and nodes
            return RPQ_OK;
        case RPQ_TUNE_DEFER:
            if (!(value >= 0) || value > 1e6) return fail(RPQ_EINVAL, "defer factor must be >= 0");
            q->defer_alpha = (float)value;
            return RPQ_OK;
        case RPQ_TUNE_SMALL:
            if (value != 0 && value != 1) return fail(RPQ_EINVAL, "small-kernel switch must be 0 or 1");
            q->allow_small = (int)value;
            return RPQ_OK;
        case RPQ_TUNE_FLAGS:
            if (value < 0 || value > 31) return fail(RPQ_EINVAL, "flags must be in [0, 31]");
            q->run_flags = (unsigned)value & 23u;  // (bit 3 is host-side: use_dmax_ne)
            if (q->use_dmax_ne != !((unsigned)value & 8u)) {
                if (q->inflight) {  // let a run in flight finish with the old graph
                    CUDA_TRY(cudaStreamSynchronize(q->last_stream));
                    q->bar_next = q->h_ctl->bar;
                    q->inflight = false;
                }
                q->use_dmax_ne = !((unsigned)value & 8u);
                drop_graphs(q);  // the captured runs carry the predictor's degree
            }
            return RPQ_OK;
        case RPQ_TUNE_TRACE: {
            if (value < 0 || value > 4096) return fail(RPQ_EINVAL, "trace levels must be in [0, 4096]");
            if (q->inflight) {  // a run in flight may still write the old buffer
                CUDA_TRY(cudaStreamSynchronize(q->last_stream));
                q->bar_next = q->h_ctl->bar;
                q->inflight = false;
            }
            if (q->d_trace) cudaFree(q->d_trace);
            q->d_trace = nullptr;
            q->trace_levels = (int)value;
            if (q->trace_levels > 0) {
                const size_t bytes = (size_t)q->trace_levels * q->grid * 8 * sizeof(unsigned long long);
                CUDA_TRY(cudaMalloc(&q->d_trace, bytes));
                CUDA_TRY(cudaMemset(q->d_trace, 0, bytes));
            }
            drop_graphs(q);  // the captured runs hold the old parameters
            return RPQ_OK;
        }
        default:
            return fail(RPQ_EINVAL, "unknown tuning key");
    }
}

int rpq_query_run(rpq_query* q, int32_t source, double timeout_s, void* stream) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    q->host_answered = false;
    if (source < 0 || source >= q->g->nv)
        return fail(RPQ_ERANGE, "vertex index " + std::to_string(source) + " out of range");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    cudaStream_t st = stream ? (cudaStream_t)stream : q->own_stream;
    // the pinned input block is read by the previous run's H2D copy: let it finish
    if (q->inflight) {
        CUDA_TRY(cudaStreamSynchronize(q->last_stream));
        q->bar_next = q->h_ctl->bar;
        q->inflight = false;
    }
    RunArgs ra{};
    ra.mode = 0;
    ra.bar_base = q->bar_next;
    ra.emit_mode = q->emit_mode;
    ra.emit_inline_max = q->emit_inline_max;
    ra.defer_alpha = q->defer_alpha;
    ra.flags = q->run_flags;
    ra.source = source;
    ra.dir_mode = q->dir_mode;
    ra.count_te = q->count_te;
    ra.alpha = q->alpha;
    // the caller's pinned answer buffer (grid kernel only; the single-CTA
    // kernel's answer goes through h_reach_bits)
    ra.out_bits = use_small(q) ? nullptr : q->run_out_bits;
    ra.run_seq = ++q->run_seq;
    q->last_zc = q->zero_copy && !use_small(q);
    ra.out_list = ra.out_bits && q->run_out_list ? 1 : 0;
    q->out_direct = ra.out_bits != nullptr;
    q->reach_stale = true;
    if (!(timeout_s >= 0) || std::isinf(timeout_s) || timeout_s > 1.0e9)
        ra.budget_ns = ~0ull;
    else
        ra.budget_ns = (unsigned long long)(timeout_s * 1e9);
    *reinterpret_cast<RunArgs*>(q->h_in) = ra;
    q->step_ra_valid = false;
    if (!q->graph_failed) build_graph(q);
    // timing events bracket the whole run (graph event nodes cannot be timed)
    CUDA_TRY(cudaEventRecord(q->ev0, st));
    if (q->graph)
        CUDA_TRY(cudaGraphLaunch(q->graph, st));
    else
        CUDA_TRY(enqueue_run(q, st, nullptr, use_small(q)));
    CUDA_TRY(cudaEventRecord(q->ev1, st));
    q->last_stream = st;
    q->ran = true;
    q->inflight = true;
    return RPQ_OK;
}

namespace {
// Wait for the last run.  poll: the grid kernel's last CTA writes the results
// prefix to pinned host memory and then the run's number; spinning on that
// flag returns as soon as it lands (a stream synchronize wakes up several us
// later).  device_ms is then the kernel's own time (globaltimer), without the
// launch.  Anything unusual (no flag, an error) falls back to the stream.
int wait_impl(rpq_query* q, rpq_stats* stats, bool poll) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (!q->ran) return fail(RPQ_EINVAL, "query has not been run");
    bool polled = false;
#ifndef RPQ_CHECKED
    if (poll && q->last_zc) {
        volatile const unsigned* flag = &q->h_ctl->done_seq;
        for (unsigned long long i = 1;; ++i) {
            if (*flag == q->run_seq) {
                polled = true;
                break;
            }
            if ((i & 255) == 0 && cudaStreamQuery(q->last_stream) != cudaErrorNotReady) break;
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    }
#endif
    if (!polled) CUDA_TRY(cudaStreamSynchronize(q->last_stream));
    q->inflight = false;
    q->bar_next = polled ? 0u : q->h_ctl->bar;
    if (const int crc = check_sites()) return crc;
    const Ctl& c = *q->h_ctl;
    float ms = 0.f;
    if (polled)
        ms = (float)((double)(c.t_end - c.t0) * 1e-6);
    else
        CUDA_TRY(cudaEventElapsedTime(&ms, q->ev0, q->ev1));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->status = c.status;
        stats->iterations = c.iterations;
        stats->levels = c.levels;
        stats->grid = q->grid;
        stats->te = q->count_te ? (int64_t)c.te_exact : (int64_t)c.te_push;
        stats->segments = (int64_t)c.segments;
        stats->visited_pairs = (int64_t)c.pairs;
        stats->reach_count = (int64_t)c.reach_count;
        stats->answer_list = q->out_direct ? c.ans_list : 0;
        stats->answer_words = (int64_t)c.ans_words;
        stats->device_ms = ms;
        stats->pull_levels = c.pull_levels;
        for (int i = 0; i < RPQ_STATS_LEVELS; ++i) {
            const bool ran_level = i <= c.iterations;
            stats->level_new[i] = ran_level ? c.level_new[i] : 0;
            stats->level_edges[i] = ran_level ? c.level_edges[i] : 0;
            stats->level_ns[i] = ran_level ? (int64_t)c.level_ns[i] : 0;
            stats->work_ns[i] = ran_level ? (int64_t)c.work_ns[i] : 0;
            stats->bar_ns[i] = ran_level ? (int64_t)c.bar_ns[i] : 0;
            stats->level_dir[i] = ran_level && i < c.iterations ? (int8_t)c.level_dir[i] : 0;
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
}  // namespace

int rpq_query_wait(rpq_query* q, rpq_stats* stats) { return wait_impl(q, stats, false); }

namespace {
int query_eval(rpq_query* q, int32_t source, double timeout_s, int32_t direction, int32_t count_te, double alpha,
               int32_t allow_small, rpq_stats* stats, uint32_t* reach_words, int64_t nwords, bool allow_list) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    const int64_t words = ((int64_t)q->g->nv + 31) / 32;
    if (reach_words == nullptr ? nwords != 0 : nwords < words) return fail(RPQ_EINVAL, "answer buffer too small");
    int rc = rpq_query_set_options(q, direction, count_te, alpha);
    if (rc == RPQ_OK) rc = rpq_query_set_tuning(q, RPQ_TUNE_SMALL, allow_small ? 1.0 : 0.0);
    // a buffer from rpq_host_alloc is written by the kernel itself (mapped
    // pinned memory, unified addressing): no copy node and no host memcpy
    const bool direct = reach_words && words && q->zero_copy && !use_small(q) &&
                        host_block_covers(reach_words, (size_t)words * 4);
    if (rc == RPQ_OK) rc = rpq_query_set_output(q, reach_words && !direct ? 1 : 0);
    // A source none of whose seed rows has an edge: P is the seed, the first
    // step finds nothing (engine.py:156-160: one iteration; none without a
    // start state), the answer is the source itself when a start state is
    // final.  Known on the host from the row bitmaps: no launch.  (Not when
    // the caller wants the device-side counts: count_te / debug runs.)
    if (rc == RPQ_OK && q->seed_ne_ok && !count_te && stats && source >= 0 && source < q->g->nv &&
        !(timeout_s >= 0 && timeout_s == 0.0)) {
        bool any_edge = false;
        for (const uint32_t* bm : q->seed_ne) any_edge |= ((bm[source >> 5] >> (source & 31)) & 1u) != 0;
        if (!any_edge) {
            rpq_stats st{};
            st.iterations = q->distinct_starts ? 1 : 0;
            st.visited_pairs = q->distinct_starts;
            st.level_new[0] = q->distinct_starts;
            const bool hit = q->distinct_starts && q->start_is_final;
            st.reach_count = hit ? 1 : 0;
            if (reach_words && words > 0) {
                if (allow_list && 2 * (int64_t)(hit ? 1 : 0) < words) {
                    st.answer_list = 1;
                    st.answer_words = hit ? 1 : 0;
                    if (hit) {
                        reach_words[0] = (uint32_t)(source >> 5);
                        reach_words[1] = 1u << (source & 31);
                    }
                } else {
                    std::memset(reach_words, 0, (size_t)words * 4);
                    if (hit) reach_words[source >> 5] = 1u << (source & 31);
                }
            }
            *stats = st;
            q->host_answered = true;
            q->host_answered_source = source;
            return RPQ_OK;
        }
    }
    q->run_out_bits = direct ? reach_words : nullptr;
    q->run_out_list = direct && allow_list && stats;
    if (rc == RPQ_OK) rc = rpq_query_run(q, source, timeout_s, nullptr);
    q->run_out_bits = nullptr;
    q->run_out_list = false;
    if (rc != RPQ_OK) return rc;
    rc = wait_impl(q, stats, true);
    if (rc != RPQ_OK) return rc;
    if (reach_words && words && !direct) std::memcpy(reach_words, q->h_reach_bits, (size_t)words * 4);
    return RPQ_OK;
}
}  // namespace

int rpq_query_eval(rpq_query* q, int32_t source, double timeout_s, int32_t direction, int32_t count_te,
                   double alpha, int32_t allow_small, rpq_stats* stats, uint32_t* reach_words, int64_t nwords) {
    return query_eval(q, source, timeout_s, direction, count_te, alpha, allow_small, stats, reach_words, nwords,
                      false);
}

int rpq_query_eval_list(rpq_query* q, int32_t source, double timeout_s, int32_t direction, int32_t count_te,
                        double alpha, int32_t allow_small, rpq_stats* stats, uint32_t* reach_words,
                        int64_t nwords) {
    return query_eval(q, source, timeout_s, direction, count_te, alpha, allow_small, stats, reach_words, nwords,
                      true);
}

namespace {
// The last query_eval was answered on the host (no seed edge): the accessors
// of device-side results run it on the device first.
int rerun_if_host_answered(rpq_query* q) {
    if (!q->host_answered) return RPQ_OK;
    q->host_answered = false;
    int rc = rpq_query_set_output(q, 1);
    if (rc == RPQ_OK) rc = rpq_query_run(q, q->host_answered_source, -1.0, nullptr);
    if (rc == RPQ_OK) rc = wait_impl(q, nullptr, false);
    return rc;
}
// The uint8[nv] answer vector of the last run, expanded from its bitmap on
// the run's stream the first time it is asked for.
int materialize_reach(rpq_query* q) {
    if (!q->reach_stale || q->g->nv == 0) return RPQ_OK;
    cudaStream_t st = q->last_stream ? q->last_stream : q->own_stream;
    const long long words = ((long long)q->g->nv + 31) / 32;
    reach_bytes_kernel<<<(unsigned)std::min<long long>((words + 255) / 256, 4L * q->g->sm_count), 256, 0, st>>>(
        q->d_reach_bits, q->d_reach, words);
    CUDA_TRY(cudaGetLastError());
    q->reach_stale = false;
    return RPQ_OK;
}
}  // namespace

int rpq_query_reach_device(rpq_query* q, uint8_t** d_reach) {
    if (!q || !d_reach) return fail(RPQ_EINVAL, "null argument");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    if (const int hrc = rerun_if_host_answered(q)) return hrc;
    if (q->ran) {
        const int rc = materialize_reach(q);
        if (rc != RPQ_OK) return rc;
    }
    *d_reach = q->d_reach;
    return RPQ_OK;
}

int rpq_query_copy_reach(rpq_query* q, uint8_t* host_reach) {
    if (!q || !host_reach) return fail(RPQ_EINVAL, "null argument");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    if (q->g->nv == 0) return RPQ_OK;
    if (const int hrc = rerun_if_host_answered(q)) return hrc;
    const int rc = materialize_reach(q);
    if (rc != RPQ_OK) return rc;
    CUDA_TRY(cudaMemcpyAsync(host_reach, q->d_reach, (size_t)q->g->nv, cudaMemcpyDeviceToHost,
                             q->last_stream ? q->last_stream : q->own_stream));
    CUDA_TRY(cudaStreamSynchronize(q->last_stream ? q->last_stream : q->own_stream));
    return RPQ_OK;
}

int rpq_query_copy_visited(rpq_query* q, uint32_t* host_words, int64_t nwords) {
    if (!q || !host_words) return fail(RPQ_EINVAL, "null argument");
    const int64_t words = ((int64_t)q->g->nv + 31) / 32;
    if (q->g->nv == 0) return RPQ_OK;
    if (nwords < words * q->nstates) return fail(RPQ_EINVAL, "output buffer too small");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    if (const int hrc = rerun_if_host_answered(q)) return hrc;
    cudaStream_t st = q->last_stream ? q->last_stream : q->own_stream;
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaMemcpy2D(host_words, (size_t)words * 4, q->d_visited, (size_t)q->W * 4,
                          (size_t)words * 4, (size_t)q->nstates, cudaMemcpyDeviceToHost));
    return RPQ_OK;
}

int rpq_query_step(rpq_query* q, const uint32_t* m_words, const uint32_t* p_words, int64_t row_words,
                   uint32_t* out_words) {
    if (!q || !m_words || !p_words || !out_words) return fail(RPQ_EINVAL, "null argument");
    const int64_t words = ((int64_t)q->g->nv + 31) / 32;
    if (row_words < words) return fail(RPQ_EINVAL, "row_words < ceil(num_vertices / 32)");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    cudaStream_t st = q->own_stream;
    if (q->inflight) {
        CUDA_TRY(cudaStreamSynchronize(q->last_stream));
        q->bar_next = q->h_ctl->bar;
        q->inflight = false;
    }
    const size_t dpitch = (size_t)q->W * 4, spitch = (size_t)row_words * 4, width = (size_t)words * 4;
    if (words > 0) {
        CUDA_TRY(cudaMemset2DAsync(q->d_visited, dpitch, 0, dpitch, (size_t)q->nstates, st));
        CUDA_TRY(cudaMemset2DAsync(q->d_fb[0], dpitch, 0, dpitch, (size_t)q->nstates, st));
        CUDA_TRY(cudaMemcpy2DAsync(q->d_visited, dpitch, p_words, spitch, width, (size_t)q->nstates,
                                   cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpy2DAsync(q->d_fb[0], dpitch, m_words, spitch, width, (size_t)q->nstates,
                                   cudaMemcpyHostToDevice, st));
    }
    RunArgs ra{};
    ra.mode = 1;
    ra.dir_mode = 1;
    ra.alpha = q->alpha;
    ra.budget_ns = ~0ull;
    ra.bar_base = q->bar_next;
    *reinterpret_cast<RunArgs*>(q->h_in) = ra;
    q->step_ra_valid = false;
    CUDA_TRY(cudaEventRecord(q->ev0, st));
    CUDA_TRY(enqueue_run(q, st));
    CUDA_TRY(cudaEventRecord(q->ev1, st));
    q->last_stream = st;
    q->ran = true;
    q->inflight = true;
    rpq_stats stats;
    const int rc = rpq_query_wait(q, &stats);
    if (rc != RPQ_OK) return rc;
    if (words > 0)
        CUDA_TRY(cudaMemcpy2D(out_words, spitch, q->d_fb[1], dpitch, width, (size_t)q->nstates,
                              cudaMemcpyDeviceToHost));
    return RPQ_OK;
}

int rpq_query_copy_trace(rpq_query* q, uint64_t* host, int64_t n, int32_t* grid) {
    if (!q || !grid) return fail(RPQ_EINVAL, "null argument");
    *grid = q->grid;
    const int64_t need = (int64_t)q->trace_levels * q->grid * 8;
    if (!q->d_trace) return fail(RPQ_EINVAL, "tracing is off (RPQ_TUNE_TRACE)");
    if (!host || n < need) return fail(RPQ_EINVAL, "trace buffer too small");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    CUDA_TRY(cudaStreamSynchronize(q->last_stream ? q->last_stream : q->own_stream));
    CUDA_TRY(cudaMemcpy(host, q->d_trace, (size_t)need * 8, cudaMemcpyDeviceToHost));
    return RPQ_OK;
}

int rpq_query_set_owned(rpq_query* q, int64_t word_lo, int64_t word_hi) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (word_lo < 0 || word_hi < word_lo || word_hi > q->W) return fail(RPQ_EINVAL, "bad owned word range");
    q->own_w0 = word_lo;
    q->own_w1 = word_hi;
    return RPQ_OK;
}

int rpq_query_row_words(const rpq_query* q, int64_t* row_words) {
    if (!q || !row_words) return fail(RPQ_EINVAL, "null argument");
    *row_words = q->W;
    return RPQ_OK;
}

int rpq_query_step_device(rpq_query* q, const uint32_t* d_m, uint32_t* d_p, uint32_t* d_out, void* stream) {
    if (!q || !d_m || !d_p || !d_out) return fail(RPQ_EINVAL, "null argument");
    if (d_out == d_m || d_out == d_p || d_m == d_p) return fail(RPQ_EINVAL, "M, P and the output must be distinct");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    cudaStream_t st = stream ? (cudaStream_t)stream : q->own_stream;
    RunArgs ra{};
    ra.mode = 1;
    ra.dir_mode = q->dir_mode;  // auto: pull when M is dense against the owned targets
    ra.alpha = q->alpha;
    ra.budget_ns = ~0ull;
    ra.bar_base = 0;  // the last CTA of every run resets the barrier counter
    ra.flags = q->run_flags;
    ra.defer_alpha = q->defer_alpha;
    ra.own_w0 = q->own_w0;
    ra.own_w1 = q->own_w1;
    // consecutive steps with the same arguments on the same stream reuse the
    // pinned input block as it is: no host round trip between levels (a
    // failed step latches its status in step_acc, read by rpq_query_step_end)
    const bool same = q->step_ra_valid && q->inflight && q->last_stream == st &&
                      std::memcmp(&q->step_ra, &ra, sizeof(RunArgs)) == 0;
    if (q->inflight && !same) {  // the pinned input block is read by the previous run's copy
        CUDA_TRY(cudaStreamSynchronize(q->last_stream));
        q->bar_next = q->h_ctl->bar;
        q->inflight = false;
        // the previous step's status would be overwritten by this run: a
        // failed step (queue overflow, barrier abort) fails the chain here
        const int prev = q->h_ctl->status;
        if (prev == ST_OVERFLOW) return fail(RPQ_ECUDA, "internal: frontier queue capacity exceeded (previous step)");
        if (prev == ST_DEADLOCK) return fail(RPQ_ECUDA, "internal: grid barrier spin limit exceeded (previous step)");
        if (prev != 0) return fail(RPQ_ECUDA, "previous step failed with kernel status " + std::to_string(prev));
    }
    if (!same) {
        *reinterpret_cast<RunArgs*>(q->h_in) = ra;
        q->step_ra = ra;
    }
    q->step_ra_valid = true;
    // the caller's buffers stand in for P and F_0 / F_1; F_2 is the query's
    // (step mode reads F_0, writes F_1, zeroes F_1 and F_2 first, keeps P)
    Params p = make_params(q);
    p.visited = d_p;
    p.fb[0] = const_cast<uint32_t*>(d_m);
    p.fb[1] = d_out;
    p.fb[2] = q->d_fb[2];
    CUDA_TRY(cudaEventRecord(q->ev0, st));
    CUDA_TRY(enqueue_run(q, st, &p));
    CUDA_TRY(cudaEventRecord(q->ev1, st));
    q->last_stream = st;
    q->ran = true;
    q->inflight = true;
    return RPQ_OK;
}

int rpq_query_step_begin(rpq_query* q, void* stream) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    cudaStream_t st = stream ? (cudaStream_t)stream : q->own_stream;
    CUDA_TRY(cudaMemsetAsync(q->d_step_acc, 0, 2 * sizeof(unsigned int), st));
    return RPQ_OK;
}

int rpq_query_step_end(rpq_query* q, int64_t* steps) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    if (q->inflight) {
        CUDA_TRY(cudaStreamSynchronize(q->last_stream));
        q->bar_next = q->h_ctl->bar;
        q->inflight = false;
    }
    if (const int crc = check_sites()) return crc;
    unsigned acc[2] = {0, 0};
    CUDA_TRY(cudaMemcpy(acc, q->d_step_acc, sizeof(acc), cudaMemcpyDeviceToHost));
    if (steps) *steps = (int64_t)acc[0];
    if (acc[1] == (unsigned)ST_OVERFLOW) return fail(RPQ_ECUDA, "internal: frontier queue capacity exceeded (a step)");
    if (acc[1] == (unsigned)ST_DEADLOCK) return fail(RPQ_ECUDA, "internal: grid barrier spin limit exceeded (a step)");
    if (acc[1] != 0) return fail(RPQ_ECUDA, "a step failed with kernel status " + std::to_string(acc[1]));
    return RPQ_OK;
}

int rpq_query_set_output(rpq_query* q, int32_t mode) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (mode < 0 || mode > 1) return fail(RPQ_EINVAL, "output mode must be 0 or 1");
    q->output_mode = mode;
    return RPQ_OK;
}

int rpq_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes <= 0) return fail(RPQ_EINVAL, "rpq_host_alloc: bad argument");
    void* p = nullptr;
    CUDA_TRY(cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    {
        std::lock_guard<std::mutex> lk(g_host_mu);
        g_host_blocks[reinterpret_cast<uintptr_t>(p)] = (size_t)bytes;
    }
    *out = p;
    return RPQ_OK;
}

int rpq_host_free(void* p) {
    if (!p) return RPQ_OK;
    {
        std::lock_guard<std::mutex> lk(g_host_mu);
        auto it = g_host_blocks.find(reinterpret_cast<uintptr_t>(p));
        if (it == g_host_blocks.end()) return fail(RPQ_EINVAL, "rpq_host_free: not an rpq_host_alloc block");
        g_host_blocks.erase(it);
    }
    CUDA_TRY(cudaFreeHost(p));
    return RPQ_OK;
}

int rpq_query_copy_reach_bits(rpq_query* q, uint32_t* host_words, int64_t nwords) {
    if (!q || (!host_words && nwords)) return fail(RPQ_EINVAL, "null argument");
    const int64_t words = ((int64_t)q->g->nv + 31) / 32;
    if (nwords < words) return fail(RPQ_EINVAL, "output buffer too small");
    if (q->host_answered) {
        if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
        if (const int hrc = rerun_if_host_answered(q)) return hrc;
    }
    if (!q->ran) return fail(RPQ_EINVAL, "query has not been run");
    if (q->output_mode == 1 && !q->out_direct) {  // already on the host (pinned), after rpq_query_wait
        std::memcpy(host_words, q->h_reach_bits, (size_t)words * 4);
        return RPQ_OK;
    }
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    cudaStream_t st = q->last_stream ? q->last_stream : q->own_stream;
    CUDA_TRY(cudaMemcpyAsync(host_words, q->d_reach_bits, (size_t)words * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return RPQ_OK;
}

int rpq_query_io_bytes(const rpq_query* q, int64_t* h2d_per_run, int64_t* d2h_per_run) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (h2d_per_run)
        *h2d_per_run = (int64_t)q->in_bytes;
    if (d2h_per_run)
        *d2h_per_run = (int64_t)offsetof(Ctl, qc) + (q->output_mode == 1 ? ((int64_t)q->g->nv + 31) / 32 * 4 : 0);
    return RPQ_OK;
}

namespace {

int batch_alloc(rpq_query* q) {
    if (q->d_bvis) return RPQ_OK;
#define BTRY(expr)                                                    \
    do {                                                              \
        cudaError_t e_ = (expr);                                      \
        if (e_ != cudaSuccess) {                                      \
            const int rc_ = cuda_fail(e_, #expr);                     \
            for (int b = 0; b < 2; ++b) {                             \
                if (q->d_bfw[b]) cudaFree(q->d_bfw[b]);               \
                if (q->d_bact[b]) cudaFree(q->d_bact[b]);             \
                q->d_bfw[b] = nullptr;                                \
                q->d_bact[b] = nullptr;                               \
            }                                                         \
            if (q->d_bheavy) cudaFree(q->d_bheavy);                   \
            if (q->d_blist) cudaFree(q->d_blist);                     \
            q->d_blist = nullptr;                                     \
            if (q->d_bctl) cudaFree(q->d_bctl);                       \
            if (q->h_bctl) cudaFreeHost(q->h_bctl);                   \
            if (q->d_bargs) cudaFree(q->d_bargs);                     \
            if (q->h_bargs) cudaFreeHost(q->h_bargs);                 \
            if (q->d_bout) cudaFree(q->d_bout);                       \
            if (q->d_bvis) cudaFree(q->d_bvis);                       \
            q->d_bheavy = nullptr;                                    \
            q->d_bctl = nullptr;                                      \
            q->h_bctl = nullptr;                                      \
            q->d_bargs = nullptr;                                     \
            q->h_bargs = nullptr;                                     \
            q->d_bout = nullptr;                                      \
            q->d_bvis = nullptr;                                      \
            return rc_;                                               \
        }                                                             \
    } while (0)
    const long long nv = q->g->nv;
    q->bnvp = std::max<long long>((nv + kBlockWords - 1) / kBlockWords, 1) * kBlockWords;
    q->bnblk = q->bnvp / kBlockWords;
    // rows longer than kLightDeg: at most nnz / kLightDeg of them per group and
    // level, each cut into ceil(deg / kChunk) chunks
    q->bheavy_cap = q->edge_bound / kLightDeg + q->edge_bound / kChunk + 1024;
    if (q->bheavy_cap >= 0xFFFFFFFFull) return fail(RPQ_EINVAL, "batch chunk list would exceed 2^32 entries");
    const size_t words = (size_t)q->nstates * (size_t)q->bnvp;
    BTRY(cudaMalloc(&q->d_bvis, words * sizeof(SW)));
    for (int b = 0; b < 2; ++b) {
        BTRY(cudaMalloc(&q->d_bfw[b], words * sizeof(SW)));
        BTRY(cudaMalloc(&q->d_bact[b], (size_t)q->nstates * (size_t)q->bnblk * 4));
    }
    BTRY(cudaMalloc(&q->d_blist, (size_t)q->nstates * (size_t)q->bnblk * sizeof(uint32_t)));
    BTRY(cudaMalloc(&q->d_bheavy, (size_t)q->bheavy_cap * sizeof(BHeavy)));
    BTRY(cudaMalloc(&q->d_bctl, sizeof(BCtl)));
    BTRY(cudaMemset(q->d_bctl, 0, sizeof(BCtl)));
    BTRY(cudaMallocHost(&q->h_bctl, sizeof(BCtl)));
    BTRY(cudaMalloc(&q->d_bargs, sizeof(BatchArgs)));
    BTRY(cudaMallocHost(&q->h_bargs, sizeof(BatchArgs)));
    BTRY(cudaMalloc(&q->d_bout, (size_t)kBatch * (size_t)q->W * 4));
    BTRY(allow_dyn_smem((const void*)batch_kernel));
    int per_sm = 0;
    q->bsmem = kBWordsBytes + q->slots.size() * sizeof(Slot) + q->tables.size() * sizeof(int32_t) + 16;
    BTRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batch_kernel, kBThreads, q->bsmem));
    if (per_sm < 1) BTRY(cudaErrorInvalidConfiguration);
    q->bgrid = q->g->sm_count * per_sm;
    q->bbar_next = 0;
#undef BTRY
    return RPQ_OK;
}

}  // namespace

int rpq_query_run_batch(rpq_query* q, int32_t nsrc, const int32_t* sources, double timeout_s, void* stream) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (nsrc < 1 || nsrc > kBatch) return fail(RPQ_EINVAL, "nsrc must be in [1, " + std::to_string(kBatch) + "]");
    if (!sources) return fail(RPQ_EINVAL, "null sources");
    for (int i = 0; i < nsrc; ++i)
        if (sources[i] < 0 || sources[i] >= q->g->nv)
            return fail(RPQ_ERANGE, "vertex index " + std::to_string(sources[i]) + " out of range");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    const int rc = batch_alloc(q);
    if (rc != RPQ_OK) return rc;
    cudaStream_t st = stream ? (cudaStream_t)stream : q->own_stream;
    if (q->binflight) {  // the pinned argument block is read by the previous run's copy
        CUDA_TRY(cudaStreamSynchronize(q->blast_stream));
        q->bbar_next = q->h_bctl->bar;
        q->binflight = false;
    }
    BatchArgs a{};
    a.nsrc = nsrc;
    a.bar_base = q->bbar_next;
    if (!(timeout_s >= 0) || std::isinf(timeout_s) || timeout_s > 1.0e9)
        a.budget_ns = ~0ull;
    else
        a.budget_ns = (unsigned long long)(timeout_s * 1e9);
    for (int i = 0; i < nsrc; ++i) a.sources[i] = sources[i];
    *q->h_bargs = a;
    BParams p{};
    p.run = q->d_bargs;
    p.tables = reinterpret_cast<const int32_t*>(q->d_in + q->off_tables);
    p.slots = reinterpret_cast<const Slot*>(q->d_in + q->off_slots);
    p.vis = q->d_bvis;
    for (int b = 0; b < 2; ++b) {
        p.fw[b] = q->d_bfw[b];
        p.act[b] = q->d_bact[b];
    }
    p.heavy = q->d_bheavy;
    p.blist = q->d_blist;
    p.ctl = q->d_bctl;
    p.out = q->d_bout;
    p.nvp = q->bnvp;
    p.nblk = q->bnblk;
    p.W = q->W;
    p.heavy_cap = q->bheavy_cap;
    p.nv = q->g->nv;
    p.nstates = q->nstates;
    p.ngroups = q->ngroups;
    p.nslots = q->nslots;
    p.ntargets = q->ntargets;
    p.nstarts = q->nstarts;
    p.nfinals = q->nfinals;
    p.nin = q->nin;
    p.table_ints = (int)q->tables.size();
    void* args[] = {&p};
    CUDA_TRY(cudaEventRecord(q->ev0, st));
    // the automaton tables live in the single-source input block: send it too
    CUDA_TRY(cudaMemcpyAsync(q->d_in, q->h_in, q->in_bytes, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(q->d_bargs, q->h_bargs, sizeof(BatchArgs), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)batch_kernel, dim3(q->bgrid), dim3(kBThreads), args, q->bsmem,
                                         st));
    CUDA_TRY(cudaMemcpyAsync(q->h_bctl, q->d_bctl, offsetof(BCtl, bc), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(q->ev1, st));
    q->blast_stream = st;
    q->bnsrc = nsrc;
    q->bran = true;
    q->binflight = true;
    return RPQ_OK;
}

int rpq_query_wait_batch(rpq_query* q, rpq_batch_stats* stats) {
    if (!q) return fail(RPQ_EINVAL, "null query");
    if (!q->bran) return fail(RPQ_EINVAL, "no batch has been run");
    CUDA_TRY(cudaStreamSynchronize(q->blast_stream));
    q->binflight = false;
    if (const int crc = check_sites()) return crc;
    const BCtl& c = *q->h_bctl;
    q->bbar_next = c.bar;
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, q->ev0, q->ev1));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->status = c.status;
        stats->nsrc = q->bnsrc;
        stats->levels = c.levels;
        stats->grid = q->bgrid;
        stats->te = (int64_t)c.te;
        stats->rows = (int64_t)c.rows;
        stats->visited_pairs = (int64_t)c.pairs;
        stats->device_ms = ms;
        for (int s = 0; s < q->bnsrc; ++s) {
            stats->iterations[s] = c.last_level[s] + 1;
            stats->reach_count[s] = (int64_t)c.reach_count[s];
        }
        for (int i = 0; i < RPQ_STATS_LEVELS && i < c.levels; ++i) {
            stats->level_items[i] = (int64_t)c.level_items[i];
            stats->level_new[i] = (int64_t)c.level_new[i];
            stats->level_ns[i] = (int64_t)c.level_ns[i];
            stats->level_rows[i] = (int64_t)c.level_rows[i];
        }
    }
    if (c.status == ST_OVERFLOW) {
        if (stats) stats->status = RPQ_ECUDA;
        return fail(RPQ_ECUDA, "internal: batch frontier capacity exceeded");
    }
    if (c.status == ST_DEADLOCK) {
        if (stats) stats->status = RPQ_ECUDA;
        return fail(RPQ_ECUDA, "internal: grid barrier spin limit exceeded");
    }
    if (c.status == RPQ_ETIMEOUT) return fail(RPQ_ETIMEOUT, "query timed out");
    if (c.status != 0) return fail(RPQ_ECUDA, "kernel status " + std::to_string(c.status));
    return RPQ_OK;
}

int rpq_query_copy_batch_bits(rpq_query* q, uint32_t* host_words, int64_t row_words) {
    if (!q || !host_words) return fail(RPQ_EINVAL, "null argument");
    if (!q->bran) return fail(RPQ_EINVAL, "no batch has been run");
    const int64_t words = ((int64_t)q->g->nv + 31) / 32;
    if (row_words < words) return fail(RPQ_EINVAL, "row_words < ceil(num_vertices / 32)");
    if (cudaSetDevice(q->g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
    CUDA_TRY(cudaStreamSynchronize(q->blast_stream));
    if (words == 0) return RPQ_OK;
    CUDA_TRY(cudaMemcpy2D(host_words, (size_t)row_words * 4, q->d_bout, (size_t)q->W * 4, (size_t)words * 4,
                          (size_t)q->bnsrc, cudaMemcpyDeviceToHost));
    return RPQ_OK;
}

int rpq_query_batch_bits_device(rpq_query* q, uint32_t** d_bits, int64_t* row_words) {
    if (!q || !d_bits || !row_words) return fail(RPQ_EINVAL, "null argument");
    *d_bits = q->d_bout;
    *row_words = q->W;
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

int rpq_ssr_wide(rpq_graph* g, int32_t nstates, int32_t ntrans, const int32_t* t_src,
                 const int32_t* t_label, const uint8_t* t_inv, const int32_t* t_dst, int32_t nstarts,
                 const int32_t* starts, int32_t nfinals, const int32_t* finals, int32_t source,
                 double timeout_s, uint32_t* out_bits, int64_t nwords, rpq_stats* stats) {
    if (!g) return fail(RPQ_EINVAL, "null graph");
    if (nstates < 1) return fail(RPQ_EINVAL, "nstates must be >= 1");
    if (ntrans < 0 || nstarts < 0 || nfinals < 0) return fail(RPQ_EINVAL, "negative count");
    if ((ntrans && (!t_src || !t_label || !t_inv || !t_dst)) || (nstarts && !starts) || (nfinals && !finals))
        return fail(RPQ_EINVAL, "null automaton array");
    if (source < 0 || source >= g->nv)
        return fail(RPQ_ERANGE, "vertex index " + std::to_string(source) + " out of range");
    const long long Wn = ((long long)g->nv + 31) / 32;
    if (out_bits && nwords < Wn) return fail(RPQ_EINVAL, "answer buffer too small");
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    std::vector<WideTrans> tr;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (cudaSetDevice(g->device) != cudaSuccess) return fail(RPQ_ECUDA, "cudaSetDevice");
        for (int i = 0; i < ntrans; ++i) {
            if (t_src[i] < 0 || t_src[i] >= nstates || t_dst[i] < 0 || t_dst[i] >= nstates)
                return fail(RPQ_EINVAL, "transition state out of range");
            if (t_label[i] < 0) return fail(RPQ_EINVAL, "negative label index");
            if (t_label[i] >= g->nl) continue;  // engine.py:100-101
            const int rc = materialize_label(g, t_label[i]);
            if (rc != RPQ_OK) return rc;
            const LabelDev& L = g->labels[t_label[i]];
            const int d = t_inv[i] ? 1 : 0;
            if (L.nnz[d] == 0) continue;
            tr.push_back(WideTrans{L.rowptr[d], L.col[d], t_src[i], t_dst[i]});
        }
    }
    for (int i = 0; i < nstarts; ++i)
        if (starts[i] < 0 || starts[i] >= nstates) return fail(RPQ_EINVAL, "start state out of range");
    for (int i = 0; i < nfinals; ++i)
        if (finals[i] < 0 || finals[i] >= nstates) return fail(RPQ_EINVAL, "final state out of range");
    const long long W = (Wn + 3) / 4 * 4;
    const size_t bitmap_bytes = (size_t)W * nstates * sizeof(uint32_t);
    WideTrans* d_tr = nullptr;
    uint32_t *d_p = nullptr, *d_f[2] = {nullptr, nullptr}, *d_out = nullptr;
    unsigned int* d_cnt[2] = {nullptr, nullptr};
    unsigned long long* d_tot = nullptr;
    int32_t *d_starts = nullptr, *d_finals = nullptr;
    auto cleanup = [&]() {
        cudaFree(d_tr); cudaFree(d_p); cudaFree(d_f[0]); cudaFree(d_f[1]); cudaFree(d_out);
        cudaFree(d_cnt[0]); cudaFree(d_cnt[1]); cudaFree(d_tot); cudaFree(d_starts); cudaFree(d_finals);
    };
#define WTRY(expr)                                   \
    do {                                             \
        cudaError_t e_ = (expr);                     \
        if (e_ != cudaSuccess) {                     \
            cleanup();                               \
            return cuda_fail(e_, #expr);             \
        }                                            \
    } while (0)
    WTRY(cudaMalloc(&d_tr, std::max<size_t>(tr.size(), 1) * sizeof(WideTrans)));
    WTRY(cudaMalloc(&d_p, bitmap_bytes));
    for (int f = 0; f < 2; ++f) {
        WTRY(cudaMalloc(&d_f[f], bitmap_bytes));
        WTRY(cudaMalloc(&d_cnt[f], (size_t)nstates * sizeof(unsigned int)));
    }
    WTRY(cudaMalloc(&d_out, (size_t)W * sizeof(uint32_t)));
    WTRY(cudaMalloc(&d_tot, 3 * sizeof(unsigned long long)));
    WTRY(cudaMalloc(&d_starts, std::max<size_t>(nstarts, 1) * sizeof(int32_t)));
    WTRY(cudaMalloc(&d_finals, std::max<size_t>(nfinals, 1) * sizeof(int32_t)));
    if (!tr.empty()) WTRY(cudaMemcpy(d_tr, tr.data(), tr.size() * sizeof(WideTrans), cudaMemcpyHostToDevice));
    if (nstarts) WTRY(cudaMemcpy(d_starts, starts, (size_t)nstarts * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (nfinals) WTRY(cudaMemcpy(d_finals, finals, (size_t)nfinals * sizeof(int32_t), cudaMemcpyHostToDevice));
    WTRY(cudaMemset(d_p, 0, bitmap_bytes));
    WTRY(cudaMemset(d_f[0], 0, bitmap_bytes));
    WTRY(cudaMemset(d_cnt[0], 0, (size_t)nstates * sizeof(unsigned int)));
    WTRY(cudaMemset(d_tot, 0, 3 * sizeof(unsigned long long)));
    unsigned long long tot[3] = {0, 0, 0};
    unsigned long long pairs = 0, te = 0;
    int iterations = 0, status = RPQ_OK;
    rpq_stats st{};
    if (nstarts) {
        wide_seed_kernel<<<1, 256>>>(d_starts, nstarts, source, W, d_p, d_f[0], d_cnt[0], d_tot);
        WTRY(cudaMemcpy(tot, d_tot, sizeof(tot), cudaMemcpyDeviceToHost));
    }
    unsigned long long nfront = tot[0];
    pairs = nfront;
    if (stats) st.level_new[0] = (int64_t)nfront;
    // the masked loop (engine.py:156-160): while M: check the clock; step; count
    for (int L = 0; nfront > 0; ++L) {
        if (timeout_s >= 0 && elapsed() > timeout_s) {
            status = RPQ_ETIMEOUT;
            break;
        }
        const int cur = L & 1, nxt = cur ^ 1;
        WTRY(cudaMemsetAsync(d_f[nxt], 0, bitmap_bytes));
        WTRY(cudaMemsetAsync(d_cnt[nxt], 0, (size_t)nstates * sizeof(unsigned int)));
        WTRY(cudaMemsetAsync(d_tot, 0, 2 * sizeof(unsigned long long)));
        wide_step_kernel<<<4 * g->sm_count, 256>>>(d_tr, (int)tr.size(), d_p, d_f[cur], d_f[nxt], W, g->nv,
                                                  d_cnt[cur], d_cnt[nxt], d_tot);
        WTRY(cudaGetLastError());
        WTRY(cudaMemcpy(tot, d_tot, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        ++iterations;
        nfront = tot[0];
        pairs += nfront;
        te += tot[1];
        if (stats && L + 1 < RPQ_STATS_LEVELS) {
            st.level_new[L + 1] = (int64_t)nfront;
            st.level_edges[L] = (int64_t)tot[1];
        }
    }
    if (status == RPQ_OK) {
        WTRY(cudaMemsetAsync(d_tot + 2, 0, sizeof(unsigned long long)));
        wide_project_kernel<<<4 * g->sm_count, 256>>>(d_finals, nfinals, d_p, W, Wn, d_out, d_tot);
        WTRY(cudaGetLastError());
        WTRY(cudaMemcpy(tot + 2, d_tot + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        if (out_bits) WTRY(cudaMemcpy(out_bits, d_out, (size_t)Wn * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    }
#undef WTRY
    cleanup();
    if (stats) {
        st.status = status;
        st.iterations = iterations;
        st.levels = iterations > 0 ? iterations - 1 : 0;
        st.grid = 4 * g->sm_count;
        st.te = (int64_t)te;
        st.visited_pairs = (int64_t)pairs;
        st.reach_count = (int64_t)tot[2];
        st.device_ms = (float)(elapsed() * 1e3);
        *stats = st;
    }
    if (status == RPQ_ETIMEOUT) return fail(RPQ_ETIMEOUT, "query timed out");
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
