// graph.cu -- gm_load_graph: edge list -> label-partitioned CSR in HBM.
//
// PAPER.md §2.1 (lines 143-147): G is an undirected, labelled, simple graph;
// N(v) is the neighbour set.  The device layout stores,
// for row r = v*S + l, the neighbours of v whose label is l, ascending:
//     nbr[offs[r] .. offs[r+1])
// so N(v) restricted to label l -- the only part of N(v) that can hold candidates
// of a query vertex with label l -- is one contiguous, sorted slice.  The build is
// one radix sort of 64-bit keys (row << 32 | neighbour) of both edge directions,
// a dedup, and an offsets pass.
#include <cub/cub.cuh>
#include <stdarg.h>

#include "gm_internal.cuh"

namespace gm {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// Directed keys for both orientations; self loops become the max sentinel.
__global__ void k_make_keys(uint64_t m, const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                            const uint32_t *__restrict__ lab, uint32_t S, uint64_t n,
                            unsigned long long *__restrict__ keys, int *__restrict__ bad) {
    const unsigned long long sentinel = (unsigned long long)(n * S) << 32;  // row past the last
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a = src[i], b = dst[i];
        if (a >= n || b >= n) { *bad = 1; keys[2 * i] = keys[2 * i + 1] = sentinel; continue; }
        if (a == b) { keys[2 * i] = keys[2 * i + 1] = sentinel; continue; }
        uint32_t la = lab ? lab[a] : 0, lb = lab ? lab[b] : 0;
        keys[2 * i] = ((unsigned long long)((uint64_t)a * S + lb) << 32) | b;
        keys[2 * i + 1] = ((unsigned long long)((uint64_t)b * S + la) << 32) | a;
    }
}

__global__ void k_check_labels(uint64_t n, const uint32_t *__restrict__ lab, uint32_t S, int *__restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (lab[i] >= S) *bad = 1;
}

// offs[r] = first position whose row >= r.  Each position that starts a new row
// fills the offsets of the (possibly empty) rows since the previous row.
__global__ void k_offsets(uint64_t nadj, const unsigned long long *__restrict__ keys, uint64_t rows,
                          uint32_t *__restrict__ offs, uint32_t *__restrict__ nbr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nadj;
         i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t r = i < nadj ? (int64_t)(keys[i] >> 32) : (int64_t)rows;
        int64_t rp = i > 0 ? (int64_t)(keys[i - 1] >> 32) : -1;
        for (int64_t rr = rp + 1; rr <= r; ++rr) offs[rr] = (uint32_t)i;
        if (i < nadj) nbr[i] = (uint32_t)(keys[i] & 0xffffffffull);
    }
}

__global__ void k_dmax(uint64_t n, uint32_t S, const uint32_t *__restrict__ offs, unsigned *__restrict__ dmax) {
    uint32_t best = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        best = max(best, offs[(v + 1) * S] - offs[v * S]);
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMax(dmax, best);
}

static int grid_for(uint64_t work, int block = 256) {
    uint64_t g = (work + block - 1) / block;
    if (g > 148ull * 32) g = 148ull * 32;
    return (int)(g ? g : 1);
}

}  // namespace gm

using namespace gm;

extern "C" const char *gm_last_error(void) { return g_err; }
extern "C" const char *gm_version(void) { return "gmatch-b200 0.1 (sm_100a)"; }

extern "C" int gm_load_graph(uint64_t n, uint64_t m, const uint32_t *src, const uint32_t *dst,
                             const uint32_t *labels, uint32_t num_labels, int mem, void *stream_,
                             gm_graph **out) {
    set_error("");
    GM_REQ(out, GM_ERR_ARG, "gm_load_graph: out is NULL");
    *out = nullptr;
    GM_REQ(m == 0 || (src && dst), GM_ERR_ARG, "gm_load_graph: src/dst NULL");
    GM_REQ(num_labels >= 1, GM_ERR_ARG, "gm_load_graph: num_labels must be >= 1");
    GM_REQ(mem == GM_MEM_HOST || mem == GM_MEM_DEVICE, GM_ERR_ARG, "gm_load_graph: bad mem");
    GM_REQ(n < 0xffffffffull, GM_ERR_LIMIT, "gm_load_graph: n=%llu exceeds uint32 ids", (unsigned long long)n);
    GM_REQ(n * (uint64_t)num_labels < 0xffffffffull, GM_ERR_LIMIT,
           "gm_load_graph: n*num_labels=%llu must be < 2^32", (unsigned long long)(n * num_labels));
    GM_REQ(2 * m < 0xffffffffull, GM_ERR_LIMIT, "gm_load_graph: 2m=%llu adjacency entries must be < 2^32",
           (unsigned long long)(2 * m));
    cudaStream_t st = (cudaStream_t)stream_;
    const uint32_t S = num_labels;
    const uint64_t rows = n * S;

    gm_graph *g = new gm_graph();
    GM_CK(cudaGetDevice(&g->device));
    g->n = n; g->S = S;

    uint32_t *d_src = nullptr, *d_dst = nullptr;
    unsigned long long *k0 = nullptr, *k1 = nullptr;
    void *tmp = nullptr;
    int *d_bad = nullptr;
    unsigned long long *d_nsel = nullptr;
    int rc = GM_OK;
    auto fail = [&](int code) { rc = code; };
#define STEP(call)                                                                         \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess) {                                                           \
            set_error("gm_load_graph: %s: %s", #call, cudaGetErrorString(_e));             \
            fail(_e == cudaErrorMemoryAllocation ? GM_ERR_NOMEM : GM_ERR_CUDA);            \
            goto cleanup;                                                                  \
        }                                                                                  \
    } while (0)
    {
        const uint32_t *s = src, *d = dst, *l = labels;
        STEP(cudaMalloc(&g->lab, sizeof(uint32_t) * (n ? n : 1)));
        if (mem == GM_MEM_HOST) {
            if (m) {
                STEP(cudaMalloc(&d_src, sizeof(uint32_t) * m));
                STEP(cudaMalloc(&d_dst, sizeof(uint32_t) * m));
                STEP(cudaMemcpyAsync(d_src, src, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, st));
                STEP(cudaMemcpyAsync(d_dst, dst, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, st));
            }
            s = d_src; d = d_dst;
            if (labels) {
                STEP(cudaMemcpyAsync(g->lab, labels, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
            }
        } else if (labels) {
            STEP(cudaMemcpyAsync(g->lab, labels, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
        }
        if (!labels) STEP(cudaMemsetAsync(g->lab, 0, sizeof(uint32_t) * (n ? n : 1), st));
        l = g->lab;

        STEP(cudaMalloc(&d_bad, 4 * sizeof(int)));
        STEP(cudaMemsetAsync(d_bad, 0, 4 * sizeof(int), st));
        d_nsel = (unsigned long long *)(d_bad + 2);
        if (n) k_check_labels<<<grid_for(n), 256, 0, st>>>(n, l, S, d_bad);

        const uint64_t K = 2 * m;
        STEP(cudaMalloc(&k0, sizeof(unsigned long long) * (K ? K : 1)));
        STEP(cudaMalloc(&k1, sizeof(unsigned long long) * (K ? K : 1)));
        if (m) k_make_keys<<<grid_for(m), 256, 0, st>>>(m, s, d, l, S, n, k0, d_bad);
        STEP(cudaGetLastError());

        int end_bit = 32;  // keys are (row << 32 | nbr) with row <= rows (sentinel = rows)
        while (end_bit < 64 && (rows >> (end_bit - 32)) != 0) ++end_bit;
        size_t tb1 = 0, tb2 = 0;
        if (K) {
            STEP(cub::DeviceRadixSort::SortKeys(nullptr, tb1, k0, k1, (int64_t)K, 0, end_bit, st));
            STEP(cub::DeviceSelect::Unique(nullptr, tb2, k1, k0, d_nsel, (int64_t)K, st));
            size_t tb = tb1 > tb2 ? tb1 : tb2;
            STEP(cudaMalloc(&tmp, tb ? tb : 16));
            STEP(cub::DeviceRadixSort::SortKeys(tmp, tb1, k0, k1, (int64_t)K, 0, end_bit, st));
            STEP(cub::DeviceSelect::Unique(tmp, tb2, k1, k0, d_nsel, (int64_t)K, st));
        }
        int hb[4] = {0, 0, 0, 0};
        STEP(cudaMemcpyAsync(hb, d_bad, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
        STEP(cudaStreamSynchronize(st));
        if (hb[0]) { set_error("gm_load_graph: vertex id >= n or label >= num_labels"); fail(GM_ERR_ARG); goto cleanup; }
        uint64_t nsel = 0;
        memcpy(&nsel, hb + 2, sizeof(nsel));
        if (K == 0) nsel = 0;
        // drop the self-loop/invalid sentinel (row == rows sorts last)
        unsigned long long last = 0;
        if (nsel) {
            STEP(cudaMemcpyAsync(&last, k0 + nsel - 1, sizeof(last), cudaMemcpyDeviceToHost, st));
            STEP(cudaStreamSynchronize(st));
            if ((last >> 32) == rows) --nsel;
        }
        g->nadj = nsel;
        STEP(cudaMalloc(&g->offs, sizeof(uint32_t) * (rows + 1)));
        STEP(cudaMalloc(&g->nbr, sizeof(uint32_t) * (nsel ? nsel : 1)));
        k_offsets<<<grid_for(nsel + 1), 256, 0, st>>>(nsel, k0, rows, g->offs, g->nbr);
        STEP(cudaGetLastError());
        unsigned *d_dmax = (unsigned *)d_bad;
        STEP(cudaMemsetAsync(d_dmax, 0, sizeof(unsigned), st));
        if (n) k_dmax<<<grid_for(n), 256, 0, st>>>(n, S, g->offs, d_dmax);
        STEP(cudaGetLastError());
        STEP(cudaMemcpyAsync(&g->dmax, d_dmax, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        STEP(cudaStreamSynchronize(st));
        cudaFree(k0); cudaFree(k1); cudaFree(tmp);   // release sort scratch before the hub index
        k0 = k1 = nullptr; tmp = nullptr;
        rc = build_hubs(g, kDefaultHubBudget, kDefaultHubMinDegree, st);
        if (rc != GM_OK) goto cleanup;
        g->bytes = sizeof(uint32_t) * (rows + 1 + (nsel ? nsel : 1) + (n ? n : 1)) +
                   (g->nhubs ? 4ull * (n + (uint64_t)g->nhubs * g->hub_words) : 0);
    }
cleanup:
#undef STEP
    cudaFree(d_src); cudaFree(d_dst); cudaFree(k0); cudaFree(k1); cudaFree(tmp); cudaFree(d_bad);
    if (rc != GM_OK) {
        cudaFree(g->offs); cudaFree(g->nbr); cudaFree(g->lab);
        free_hubs(g);
        delete g;
        return rc;
    }
    *out = g;
    return GM_OK;
}

extern "C" int gm_graph_info(const gm_graph *g, gm_graph_info_t *info) {
    GM_REQ(g && info, GM_ERR_ARG, "gm_graph_info: NULL argument");
    info->n = g->n;
    info->num_adj = g->nadj;
    info->num_labels = g->S;
    info->d_max = g->dmax;
    info->device_bytes = g->bytes;
    info->hubs = g->nhubs;
    info->hub_min_degree = g->hub_min_degree;
    return GM_OK;
}

extern "C" int gm_graph_export(const gm_graph *g, uint32_t *offs_host, uint32_t *nbr_host, uint32_t *labels_host) {
    GM_REQ(g, GM_ERR_ARG, "gm_graph_export: NULL graph");
    if (offs_host) GM_CK(cudaMemcpy(offs_host, g->offs, sizeof(uint32_t) * (g->n * g->S + 1), cudaMemcpyDeviceToHost));
    if (nbr_host && g->nadj) GM_CK(cudaMemcpy(nbr_host, g->nbr, sizeof(uint32_t) * g->nadj, cudaMemcpyDeviceToHost));
    if (labels_host && g->n) GM_CK(cudaMemcpy(labels_host, g->lab, sizeof(uint32_t) * g->n, cudaMemcpyDeviceToHost));
    return GM_OK;
}

extern "C" void gm_free_graph(gm_graph *g) {
    if (!g) return;
    cudaFree(g->offs); cudaFree(g->nbr); cudaFree(g->lab);
    free_hubs(g);
    delete g;
}
