// graph.cu -- gm_load_graph: edge list -> degree-ordered, label-partitioned CSR in HBM.
//
// PAPER.md §2.1 (lines 143-147): G is an undirected, labelled, simple graph;
// N(v) is the neighbour set.  The device layout:
//   * vertices are renumbered by decreasing degree (ties by original id), so the
//     highest-degree vertices -- the hubs of a power-law graph -- are ids 0..K-1: "w is a
//     hub" is the compare w < K and a hub's bitmap row is row w (hubs.cu).  The API speaks
//     original ids: old2new / new2old map at the boundary (roots in, embeddings out,
//     exports), never inside the search.
//   * for row r = v*S + l (v a new id), nbr[offs[r] .. offs[r+1]) holds the neighbours of v
//     whose label is l, ascending, so N(v) restricted to label l -- the only part of N(v)
//     that can hold candidates of a query vertex with label l -- is one sorted slice.
// The build: degree histogram + one sort of vertices, then one radix sort of 64-bit keys
// (row << 32 | neighbour) of both edge directions, a dedup, and an offsets pass.
#include <cub/cub.cuh>
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "gm_internal.cuh"

namespace gm {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// Approximate degrees (repeated pairs counted twice; self loops skipped) and id validity.
__global__ void k_degree_count(uint64_t m, const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                               uint64_t n, uint32_t *__restrict__ deg, int *__restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = src[i], b = dst[i];
        if (a >= n || b >= n) { *bad = 1; continue; }
        if (a == b) continue;
        atomicAdd(deg + a, 1u);
        atomicAdd(deg + b, 1u);
    }
}

__global__ void k_iota(uint64_t n, uint32_t *__restrict__ ids) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        ids[v] = (uint32_t)v;
}

// old2new = inverse of new2old; labels permuted into the new id order.
__global__ void k_renumber(uint64_t n, const uint32_t *__restrict__ new2old, const uint32_t *__restrict__ lab_in,
                           uint32_t *__restrict__ old2new, uint32_t *__restrict__ lab_out) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = new2old[v];
        old2new[o] = (uint32_t)v;
        lab_out[v] = lab_in ? lab_in[o] : 0;
    }
}

__global__ void k_check_labels(uint64_t n, const uint32_t *__restrict__ lab, uint32_t S, int *__restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (lab[i] >= S) *bad = 1;
}

// Directed keys (new ids) for both orientations; self loops become a sentinel row.
__global__ void k_make_keys(uint64_t m, const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                            const uint32_t *__restrict__ old2new, const uint32_t *__restrict__ lab, uint32_t S,
                            uint64_t n, unsigned long long *__restrict__ keys) {
    const unsigned long long sentinel = (unsigned long long)(n * S) << 32;  // row past the last
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a0 = src[i], b0 = dst[i];
        if (a0 >= n || b0 >= n || a0 == b0) { keys[2 * i] = keys[2 * i + 1] = sentinel; continue; }
        const uint32_t a = old2new[a0], b = old2new[b0];
        keys[2 * i] = ((unsigned long long)((uint64_t)a * S + lab[b]) << 32) | b;
        keys[2 * i + 1] = ((unsigned long long)((uint64_t)b * S + lab[a]) << 32) | a;
    }
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
extern "C" const char *gm_version(void) { return "gmatch-b200 0.2 (sm_100a)"; }

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
    const uint64_t nn = n ? n : 1;

    gm_graph *g = new gm_graph();
    GM_CK(cudaGetDevice(&g->device));
    g->n = n; g->S = S;

    uint32_t *d_src = nullptr, *d_dst = nullptr, *lab_in = nullptr;
    uint32_t *deg = nullptr, *deg_s = nullptr, *ids = nullptr;
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
        const uint32_t *s = src, *d = dst;
        STEP(cudaMalloc(&g->lab, sizeof(uint32_t) * nn));
        STEP(cudaMalloc(&g->old2new, sizeof(uint32_t) * nn));
        STEP(cudaMalloc(&g->new2old, sizeof(uint32_t) * nn));
        if (labels) STEP(cudaMalloc(&lab_in, sizeof(uint32_t) * nn));
        if (mem == GM_MEM_HOST) {
            if (m) {
                STEP(cudaMalloc(&d_src, sizeof(uint32_t) * m));
                STEP(cudaMalloc(&d_dst, sizeof(uint32_t) * m));
                STEP(cudaMemcpyAsync(d_src, src, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, st));
                STEP(cudaMemcpyAsync(d_dst, dst, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, st));
            }
            s = d_src; d = d_dst;
            if (labels && n) STEP(cudaMemcpyAsync(lab_in, labels, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
        } else if (labels && n) {
            STEP(cudaMemcpyAsync(lab_in, labels, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
        }

        STEP(cudaMalloc(&d_bad, 4 * sizeof(int)));
        STEP(cudaMemsetAsync(d_bad, 0, 4 * sizeof(int), st));
        d_nsel = (unsigned long long *)(d_bad + 2);
        if (labels && n) k_check_labels<<<grid_for(n), 256, 0, st>>>(n, lab_in, S, d_bad);

        // ---- degree order: new id = rank of the vertex by (approximate degree desc, id asc)
        STEP(cudaMalloc(&deg, sizeof(uint32_t) * nn));
        STEP(cudaMalloc(&deg_s, sizeof(uint32_t) * nn));
        STEP(cudaMalloc(&ids, sizeof(uint32_t) * nn));
        STEP(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * nn, st));
        if (m) k_degree_count<<<grid_for(m), 256, 0, st>>>(m, s, d, n, deg, d_bad);
        if (n) k_iota<<<grid_for(n), 256, 0, st>>>(n, ids);
        if (n) {
            size_t tbs = 0;
            STEP(cub::DeviceRadixSort::SortPairsDescending(nullptr, tbs, deg, deg_s, ids, g->new2old, (int64_t)n, 0, 32, st));
            STEP(cudaMalloc(&tmp, tbs ? tbs : 16));
            STEP(cub::DeviceRadixSort::SortPairsDescending(tmp, tbs, deg, deg_s, ids, g->new2old, (int64_t)n, 0, 32, st));
            STEP(cudaFree(tmp));
            tmp = nullptr;
            k_renumber<<<grid_for(n), 256, 0, st>>>(n, g->new2old, lab_in, g->old2new, g->lab);
        }
        STEP(cudaGetLastError());

        // ---- adjacency keys, sort, dedup, offsets
        const uint64_t K = 2 * m;
        STEP(cudaMalloc(&k0, sizeof(unsigned long long) * (K ? K : 1)));
        STEP(cudaMalloc(&k1, sizeof(unsigned long long) * (K ? K : 1)));
        if (m) k_make_keys<<<grid_for(m), 256, 0, st>>>(m, s, d, g->old2new, g->lab, S, n, k0);
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
        // (+4 words: 16-byte vector and bulk copies of a row may round its end up to 16 bytes)
        STEP(cudaMalloc(&g->nbr, sizeof(uint32_t) * (nsel + 4)));
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
        // (no summary level by default: measured slower on rmat24/26)
        rc = build_hubs(g, default_hub_budget(g), kDefaultHubMinDegree, 0, st);
        if (rc != GM_OK) goto cleanup;
        g->bytes = sizeof(uint32_t) * (rows + 1 + (nsel ? nsel : 1) + 3 * nn) +
                   4ull * ((uint64_t)g->nhubs * g->hub_words + (uint64_t)(g->nhubs - g->summ_first) * g->summ_words);
    }
cleanup:
#undef STEP
    cudaFree(d_src); cudaFree(d_dst); cudaFree(lab_in); cudaFree(deg); cudaFree(deg_s); cudaFree(ids);
    cudaFree(k0); cudaFree(k1); cudaFree(tmp); cudaFree(d_bad);
    if (rc != GM_OK) {
        cudaFree(g->offs); cudaFree(g->nbr); cudaFree(g->lab); cudaFree(g->old2new); cudaFree(g->new2old);
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
    info->hub_bytes = 4ull * ((uint64_t)g->nhubs * g->hub_words + (uint64_t)(g->nhubs - g->summ_first) * g->summ_words);
    info->hub_summary_words = g->summ_words;
    info->reserved = 0;
    return GM_OK;
}

// Export in ORIGINAL ids: row v*S + l = original ids of v's label-l neighbours, ascending.
extern "C" int gm_graph_export(const gm_graph *g, uint32_t *offs_host, uint32_t *nbr_host, uint32_t *labels_host) {
    GM_REQ(g, GM_ERR_ARG, "gm_graph_export: NULL graph");
    const uint64_t n = g->n, S = g->S, rows = n * S;
    std::vector<uint32_t> offs(rows + 1), nbr(g->nadj), lab(n), n2o(n), o2n(n);
    GM_CK(cudaMemcpy(offs.data(), g->offs, sizeof(uint32_t) * (rows + 1), cudaMemcpyDeviceToHost));
    if (g->nadj) GM_CK(cudaMemcpy(nbr.data(), g->nbr, sizeof(uint32_t) * g->nadj, cudaMemcpyDeviceToHost));
    if (n) {
        GM_CK(cudaMemcpy(lab.data(), g->lab, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
        GM_CK(cudaMemcpy(n2o.data(), g->new2old, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
        GM_CK(cudaMemcpy(o2n.data(), g->old2new, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
    }
    if (labels_host)
        for (uint64_t v = 0; v < n; ++v) labels_host[v] = lab[o2n[v]];
    if (offs_host || nbr_host) {
        uint64_t pos = 0;
        std::vector<uint32_t> row;
        for (uint64_t v = 0; v < n; ++v) {
            const uint64_t nv = o2n[v];
            for (uint64_t l = 0; l < S; ++l) {
                if (offs_host) offs_host[v * S + l] = (uint32_t)pos;
                const uint64_t r = nv * S + l;
                row.assign(nbr.begin() + offs[r], nbr.begin() + offs[r + 1]);
                for (auto &w : row) w = n2o[w];
                std::sort(row.begin(), row.end());
                if (nbr_host) std::copy(row.begin(), row.end(), nbr_host + pos);
                pos += row.size();
            }
        }
        if (offs_host) offs_host[rows] = (uint32_t)pos;
    }
    return GM_OK;
}

extern "C" void gm_free_graph(gm_graph *g) {
    if (!g) return;
    cudaFree(g->offs); cudaFree(g->nbr); cudaFree(g->lab); cudaFree(g->old2new); cudaFree(g->new2old);
    free_hubs(g);
    delete g;
}
