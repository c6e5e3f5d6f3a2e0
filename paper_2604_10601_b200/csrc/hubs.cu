// hubs.cu -- hub adjacency index: bitmaps of N(v) for the highest-degree vertices.
//
// The DFS's dominant cost is the membership test v in N(M[u'']) (Alg. 2 line 38; §5.2:
// "verifying that v is a neighbor of all data vertices mapped to u's backward neighbors
// ... via binary search, costing O(log |N(M[u'])|)").  On power-law graphs those tests
// concentrate on a few high-degree vertices, whose lists are the longest to search.  For
// the top-K vertices by degree (K bounded by a byte budget sized to stay L2-resident
// beside the CSR) we keep a bitmap over all vertex ids, so a test against a hub costs one
// hub_id load and one bitmap-word load instead of ceil(log2 d) dependent probes.  Lists of
// non-hub vertices are still binary searched.  (an index the
// paper does not use; BEEP's per-centre adjacency matrix, §6.2, is the closest relative.)
#include <cub/cub.cuh>

#include <vector>

#include "gm_internal.cuh"

namespace gm {

__global__ void k_degrees(uint64_t n, uint32_t S, const uint32_t *__restrict__ offs, uint32_t *__restrict__ deg,
                          uint32_t *__restrict__ ids) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        deg[v] = offs[(v + 1) * S] - offs[v * S];
        ids[v] = (uint32_t)v;
    }
}

__global__ void k_fill_u32(uint32_t *__restrict__ p, uint64_t n, uint32_t val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = val;
}

__global__ void k_hub_ids(const uint32_t *__restrict__ order, uint32_t k, uint32_t *__restrict__ hub_id) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) hub_id[order[i]] = i;
}

// One block per hub: set bit w of the hub's bitmap for every neighbour w (all labels).
__global__ void k_hub_bits(const uint32_t *__restrict__ order, uint32_t S, const uint32_t *__restrict__ offs,
                           const uint32_t *__restrict__ nbr, uint32_t words, uint32_t *__restrict__ bits) {
    const uint32_t h = blockIdx.x;
    const uint64_t v = order[h];
    uint32_t *row = bits + (uint64_t)h * words;
    const uint32_t lo = offs[v * S], hi = offs[(v + 1) * S];
    for (uint32_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        const uint32_t w = nbr[e];
        atomicOr(row + (w >> 5), 1u << (w & 31));
    }
}

static int gridn(uint64_t work) {
    uint64_t g = (work + 255) / 256;
    if (g > 148ull * 16) g = 148ull * 16;
    return (int)(g ? g : 1);
}

void free_hubs(gm_graph *g) {
    cudaFree(g->hub_id);
    cudaFree(g->hub_bits);
    g->hub_id = nullptr;
    g->hub_bits = nullptr;
    g->nhubs = 0;
}

int build_hubs(gm_graph *g, uint64_t budget_bytes, uint32_t min_degree, cudaStream_t st) {
    free_hubs(g);
    g->hub_min_degree = min_degree;
    g->hub_words = (uint32_t)((g->n + 31) / 32);
    if (g->n == 0 || budget_bytes == 0 || g->dmax < min_degree) return GM_OK;
    const uint64_t per_hub = 4ull * g->hub_words;
    uint64_t kmax = budget_bytes / per_hub;
    if (kmax > g->n) kmax = g->n;
    if (kmax == 0) return GM_OK;
    uint32_t *deg = nullptr, *ids = nullptr, *deg_s = nullptr, *ids_s = nullptr;
    void *tmp = nullptr;
    size_t tb = 0;
    int rc = GM_OK;
    std::vector<uint32_t> top(kmax);
    uint32_t k = 0;
    do {
        cudaError_t e;
        if ((e = cudaMalloc(&deg, 4 * g->n)) || (e = cudaMalloc(&ids, 4 * g->n)) || (e = cudaMalloc(&deg_s, 4 * g->n)) ||
            (e = cudaMalloc(&ids_s, 4 * g->n))) {
            set_error("build_hubs: %s", cudaGetErrorString(e)); rc = GM_ERR_NOMEM; break;
        }
        k_degrees<<<gridn(g->n), 256, 0, st>>>(g->n, g->S, g->offs, deg, ids);
        cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, deg, deg_s, ids, ids_s, (int64_t)g->n, 0, 32, st);
        if ((e = cudaMalloc(&tmp, tb ? tb : 16))) { set_error("build_hubs: %s", cudaGetErrorString(e)); rc = GM_ERR_NOMEM; break; }
        cub::DeviceRadixSort::SortPairsDescending(tmp, tb, deg, deg_s, ids, ids_s, (int64_t)g->n, 0, 32, st);
        if ((e = cudaMemcpyAsync(top.data(), deg_s, 4 * kmax, cudaMemcpyDeviceToHost, st)) ||
            (e = cudaStreamSynchronize(st))) {
            set_error("build_hubs: %s", cudaGetErrorString(e)); rc = GM_ERR_CUDA; break;
        }
        while (k < kmax && top[k] >= min_degree) ++k;
        if (k == 0) break;
        if ((e = cudaMalloc(&g->hub_id, 4 * g->n)) || (e = cudaMalloc(&g->hub_bits, per_hub * k))) {
            set_error("build_hubs: %s", cudaGetErrorString(e)); rc = GM_ERR_NOMEM; break;
        }
        k_fill_u32<<<gridn(g->n), 256, 0, st>>>(g->hub_id, g->n, 0xffffffffu);
        k_hub_ids<<<gridn(k), 256, 0, st>>>(ids_s, k, g->hub_id);
        cudaMemsetAsync(g->hub_bits, 0, per_hub * k, st);
        k_hub_bits<<<k, 256, 0, st>>>(ids_s, g->S, g->offs, g->nbr, g->hub_words, g->hub_bits);
        if ((e = cudaGetLastError()) || (e = cudaStreamSynchronize(st))) {
            set_error("build_hubs: %s", cudaGetErrorString(e)); rc = GM_ERR_CUDA; break;
        }
        g->nhubs = k;
    } while (0);
    cudaFree(deg); cudaFree(ids); cudaFree(deg_s); cudaFree(ids_s); cudaFree(tmp);
    if (rc != GM_OK) free_hubs(g);
    return rc;
}

}  // namespace gm

extern "C" int gm_graph_build_hubs(gm_graph *g, uint64_t budget_bytes, uint32_t min_degree, void *stream) {
    gm::set_error("");
    GM_REQ(g, GM_ERR_ARG, "gm_graph_build_hubs: NULL graph");
    return gm::build_hubs(g, budget_bytes, min_degree, (cudaStream_t)stream);
}
