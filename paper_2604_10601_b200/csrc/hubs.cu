// hubs.cu -- hub adjacency index: bitmaps of N(v) for the highest-degree vertices.
//
// The DFS's dominant cost is the membership test v in N(M[u'']) (Alg. 2 line 38; §5.2:
// "verifying that v is a neighbor of all data vertices mapped to u's backward neighbors
// ... via binary search, costing O(log |N(M[u'])|)").  On power-law graphs those tests
// concentrate on a few high-degree vertices, whose lists are the longest to search.
// Device ids are ordered by decreasing degree (graph.cu), so the hubs are ids 0..K-1:
// for them we keep a bitmap over all device ids (row h of hub_bits), and a test against
// w < K costs ONE bitmap-word load instead of ceil(log2 d) dependent probes.  K is bounded
// by a byte budget sized to stay L2-resident beside the CSR.  Lists of non-hubs are still
// binary searched.  (an index the paper does not use; BEEP's
// per-centre adjacency matrix, §6.2, is its closest relative.)
#include <algorithm>
#include <vector>

#include "gm_internal.cuh"

namespace gm {

// One block per hub: set bit w of the hub's bitmap for every neighbour w (all labels).
__global__ void k_hub_bits(uint32_t S, const uint32_t *__restrict__ offs, const uint32_t *__restrict__ nbr,
                           uint32_t words, uint32_t *__restrict__ bits) {
    const uint64_t h = blockIdx.x;
    uint32_t *row = bits + h * words;
    const uint32_t lo = offs[h * S], hi = offs[(h + 1) * S];
    for (uint32_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        const uint32_t w = nbr[e];
        atomicOr(row + (w >> 5), 1u << (w & 31));
    }
}

// Summary rows: thread j of hub h reads the 32-byte sector j of the bitmap (vertices
// [256 j, 256 j + 256)), and a warp's ballot over 32 consecutive sectors is summary word j/32.
__global__ void k_hub_summ(uint32_t nhubs, uint32_t words, uint32_t summ_words, const uint32_t *__restrict__ bits,
                           uint32_t *__restrict__ summ) {
    const uint64_t sectors = (uint64_t)summ_words * 32;
    const uint64_t total = (uint64_t)nhubs * sectors;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i - (threadIdx.x & 31) < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        bool any = false;
        if (i < total) {
            const uint64_t h = i / sectors, j = i % sectors;
            const uint32_t *row = bits + h * words;
            for (uint32_t k = 0; k < 8; ++k) {
                const uint64_t w = j * 8 + k;
                if (w < words) any = any || row[w] != 0;
            }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, any);
        if ((threadIdx.x & 31) == 0 && i < total) summ[i / 32] = m;   // sectors is a multiple of 32
    }
}

uint64_t default_hub_budget(const gm_graph *g) {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    const uint64_t csr = 4ull * (g->n * g->S + 1 + g->nadj);
    // measured: on rmat18 (30 MB CSR) the 64 MiB index stays in L2 beside the
    // graph; on rmat24/26 every probe goes to DRAM anyway, and an 8 GiB index (one DRAM
    // word per test against a hub instead of a dependent binary search) doubled tasks/s
    if (csr + kDefaultHubBudget <= (uint64_t)l2) return kDefaultHubBudget;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); return kDefaultHubBudget; }
    const uint64_t cap = fr / 4;
    return cap < kLargeHubBudget ? (cap > kDefaultHubBudget ? cap : kDefaultHubBudget) : kLargeHubBudget;
}

void free_hubs(gm_graph *g) {
    cudaFree(g->hub_bits);
    cudaFree(g->hub_summ);
    g->hub_bits = nullptr;
    g->hub_summ = nullptr;
    g->summ_words = 0;
    g->summ_first = 0;
    g->nhubs = 0;
}

int build_hubs(gm_graph *g, uint64_t budget_bytes, uint32_t min_degree, int summary, cudaStream_t st) {
    free_hubs(g);
    g->hub_min_degree = min_degree;
    g->hub_words = (uint32_t)((g->n + 31) / 32);
    if (g->n == 0 || budget_bytes == 0 || g->dmax < min_degree) return GM_OK;
    const uint64_t per_hub = 4ull * g->hub_words;
    uint64_t kmax = budget_bytes / per_hub;
    if (kmax > g->n) kmax = g->n;
    if (kmax == 0) return GM_OK;
    // degrees of the leading device ids (ordered by decreasing degree at load time)
    std::vector<uint32_t> offs(kmax + 1);
    GM_CK(cudaMemcpy2DAsync(offs.data(), sizeof(uint32_t), g->offs, sizeof(uint32_t) * g->S, sizeof(uint32_t),
                            kmax + 1, cudaMemcpyDeviceToHost, st));   // offs[i*S], i = 0..kmax
    GM_CK(cudaStreamSynchronize(st));
    uint32_t k = 0;
    while (k < kmax && offs[k + 1] - offs[k] >= min_degree) ++k;
    if (k == 0) return GM_OK;
    GM_CK(cudaMalloc(&g->hub_bits, per_hub * k));
    GM_CK(cudaMemsetAsync(g->hub_bits, 0, per_hub * k, st));
    k_hub_bits<<<k, 256, 0, st>>>(g->S, g->offs, g->nbr, g->hub_words, g->hub_bits);
    GM_CK(cudaGetLastError());
    // An index larger than L2 gets a summary level (1 bit per 32-byte bitmap sector, 1/256 of
    // the index): a test whose summary bit is 0 -- most tests fail, and a hub of degree d has
    // neighbours in about d of the n/256 blocks -- is answered from the L2-resident summary
    // instead of a DRAM sector of the bitmap.
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    // Only hubs whose summary is selective get one: a hub of degree d has neighbours in about
    // 1 - exp(-256 d / n) of the blocks; above d = n / 1024 (~22 %) the extra dependent load
    // costs more than the bitmap sectors it saves.  Hubs are in decreasing degree order, so
    // the selective ones are a suffix [summ_first, k).
    uint32_t first = 0;
    if (summary < 1)
        while (first < k && (uint64_t)(offs[first + 1] - offs[first]) * 1024 > g->n) ++first;
    if (first < k && (summary > 0 || (summary < 0 && per_hub * k > (uint64_t)l2))) {
        const uint32_t ks = k - first;
        g->summ_words = (uint32_t)((g->n + 8191) / 8192);
        g->summ_first = first;
        GM_CK(cudaMalloc(&g->hub_summ, 4ull * g->summ_words * ks));
        const uint64_t threads = (uint64_t)ks * g->summ_words * 32;
        const uint64_t blocks = std::min<uint64_t>((threads + 255) / 256, 148ull * 32);
        k_hub_summ<<<(unsigned)blocks, 256, 0, st>>>(ks, g->hub_words, g->summ_words,
                                                     g->hub_bits + (uint64_t)first * g->hub_words, g->hub_summ);
        GM_CK(cudaGetLastError());
    }
    GM_CK(cudaStreamSynchronize(st));
    g->nhubs = k;
    return GM_OK;
}

}  // namespace gm

extern "C" int gm_graph_build_hubs(gm_graph *g, uint64_t budget_bytes, uint32_t min_degree, int summary,
                                   void *stream) {
    gm::set_error("");
    GM_REQ(g, GM_ERR_ARG, "gm_graph_build_hubs: NULL graph");
    return gm::build_hubs(g, budget_bytes, min_degree, summary, (cudaStream_t)stream);
}
