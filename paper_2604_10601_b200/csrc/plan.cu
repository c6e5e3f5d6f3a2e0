// plan.cu -- gm_plan_query: candidate filter (GPU) + matching order (host).
//
// Filter (north_star "LDF/NLF candidate filter"; §6.1 line 681 notes the
// degree-based filtering gMatch runs on the GPU): for query vertex u and data vertex v
//   LABEL: L(v) = L(u)                                     (Definition 1, clause 1)
//   LDF:   LABEL and d(v) >= d(u)
//   NLF:   LDF and, for every label l of a neighbour of u, |N_l(v)| >= |N_l(u)|
// With the label-partitioned CSR, |N_l(v)| = offs[v*S+l+1] - offs[v*S+l]: the NLF test
// reads S+1 consecutive offsets of v, so one warp reads a contiguous 32*(S+1)*4-byte
// span -- the kernel is a single coalesced pass over offs (HBM-bound).
// Results are bitmaps (bit v of cand[u]) built with one __ballot_sync per 32 vertices.
//
// Matching order (§3: "we generate phi on the CPU using the RI
// method"; any connected order is valid, §2.2): RI-style greedy -- first the
// vertex with the fewest candidates per unit degree, then repeatedly the unplaced
// vertex with the most already-placed neighbours (RI's first criterion), ties broken
// by fewer candidates, higher degree, smaller id.  DESIGN.md lists this reading.
#include <string.h>

#include <vector>

#include "gm_internal.cuh"

namespace gm {

struct FilterSpec {
    uint32_t nq, S, filter, words;
    uint32_t qlab[kMaxQ];
    uint32_t qdeg[kMaxQ];
    uint32_t nlf_n[kMaxQ];
    uint32_t nlf_lab[kMaxQ][kMaxQ];
    uint32_t nlf_need[kMaxQ][kMaxQ];
};

__global__ void __launch_bounds__(256) k_filter(uint64_t n, const uint32_t *__restrict__ offs,
                                                const uint32_t *__restrict__ lab,
                                                const FilterSpec *__restrict__ fs,
                                                uint32_t *__restrict__ cand,
                                                unsigned long long *__restrict__ counts) {
    __shared__ unsigned s_cnt[kMaxQ];
    __shared__ FilterSpec s;
    for (int i = threadIdx.x; i < (int)(sizeof(FilterSpec) / 4); i += blockDim.x)
        ((uint32_t *)&s)[i] = ((const uint32_t *)fs)[i];
    if (threadIdx.x < kMaxQ) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t S = s.S;
    for (uint64_t v0 = warp * 32; v0 < n; v0 += nwarps * 32) {
        const uint64_t v = v0 + lane;
        const bool valid = v < n;
        const uint32_t l = valid ? lab[v] : 0xffffffffu;
        const uint64_t row = v * S;
        const uint32_t deg = valid ? offs[row + S] - offs[row] : 0;
        for (uint32_t u = 0; u < s.nq; ++u) {
            bool pred = valid && l == s.qlab[u];
            if (pred && s.filter >= GM_FILTER_LDF) pred = deg >= s.qdeg[u];
            if (pred && s.filter >= GM_FILTER_NLF) {
                for (uint32_t k = 0; k < s.nlf_n[u]; ++k) {
                    const uint32_t ll = s.nlf_lab[u][k];
                    if (offs[row + ll + 1] - offs[row + ll] < s.nlf_need[u][k]) { pred = false; break; }
                }
            }
            const uint32_t word = __ballot_sync(0xffffffffu, pred);
            if (lane == 0) {
                cand[(uint64_t)u * s.words + (v0 >> 5)] = word;
                if (word) atomicAdd(&s_cnt[u], (unsigned)__popc(word));
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < s.nq && s_cnt[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

}  // namespace gm

using namespace gm;

static bool connected_order(const gm_plan *p, const uint32_t *order) {
    uint32_t seen = 0, placed = 0;
    for (uint32_t i = 0; i < p->nq; ++i) {
        uint32_t u = order[i];
        if (u >= p->nq || (seen >> u & 1u)) return false;
        if (i > 0 && (p->qadj[u] & placed) == 0) return false;
        seen |= 1u << u;
        placed |= 1u << u;
    }
    return true;
}

static void ri_order(const gm_plan *p, uint32_t *order) {
    const uint32_t nq = p->nq;
    auto better_root = [&](uint32_t a, uint32_t b) {  // is a a better root than b?
        // fewer candidates per unit degree: c[a]/d[a] < c[b]/d[b]
        long double ra = (long double)p->cand_count[a] / (p->qdeg[a] ? p->qdeg[a] : 1);
        long double rb = (long double)p->cand_count[b] / (p->qdeg[b] ? p->qdeg[b] : 1);
        if (ra != rb) return ra < rb;
        if (p->qdeg[a] != p->qdeg[b]) return p->qdeg[a] > p->qdeg[b];
        return a < b;
    };
    uint32_t r = 0;
    for (uint32_t u = 1; u < nq; ++u)
        if (better_root(u, r)) r = u;
    order[0] = r;
    uint32_t placed = 1u << r;
    for (uint32_t i = 1; i < nq; ++i) {
        int best = -1;
        for (uint32_t u = 0; u < nq; ++u) {
            if (placed >> u & 1u) continue;
            const int nb = __builtin_popcount(p->qadj[u] & placed);
            if (nb == 0) continue;
            if (best < 0) { best = (int)u; continue; }
            const int bb = __builtin_popcount(p->qadj[best] & placed);
            if (nb != bb) { if (nb > bb) best = (int)u; continue; }
            if (p->cand_count[u] != p->cand_count[best]) { if (p->cand_count[u] < p->cand_count[best]) best = (int)u; continue; }
            if (p->qdeg[u] != p->qdeg[best]) { if (p->qdeg[u] > p->qdeg[best]) best = (int)u; continue; }
        }
        order[i] = (uint32_t)best;
        placed |= 1u << best;
    }
}

// ---- symmetry breaking (Appendix A: "we use the same matching order and
// symmetry breaking strategy in gMatch and T-DFS").  Aut(Q) = label- and edge-preserving
// permutations of V(Q), enumerated by backtracking (given up above kMaxAut).  Conditions
// are Grochow-Kellis: while the group is non-trivial, take the vertex v with the largest
// orbit (earliest in phi on ties), require M[v] > M[w] for every other w of its orbit, and
// continue with v's stabilizer.  Exactly one embedding of every Aut(Q)-orbit satisfies
// them (the orbit of an embedding under Aut(Q) has |Aut(Q)| members, injectivity makes the
// action free), so count = |Aut(Q)| * (embeddings satisfying the conditions).
static constexpr size_t kMaxAut = 200000;

static bool aut_search(const gm_plan *p, uint32_t pos, uint8_t *img, uint32_t used,
                       std::vector<std::vector<uint8_t>> &auts) {
    const uint32_t nq = p->nq;
    if (pos == nq) {
        auts.emplace_back(img, img + nq);
        return auts.size() <= kMaxAut;
    }
    for (uint32_t w = 0; w < nq; ++w) {
        if ((used >> w) & 1u) continue;
        if (p->qlab[w] != p->qlab[pos] || p->qdeg[w] != p->qdeg[pos]) continue;
        bool ok = true;
        for (uint32_t x = 0; x < pos && ok; ++x)
            ok = ((p->qadj[pos] >> x) & 1u) == ((p->qadj[w] >> img[x]) & 1u);
        if (!ok) continue;
        img[pos] = (uint8_t)w;
        if (!aut_search(p, pos + 1, img, used | (1u << w), auts)) return false;
    }
    return true;
}

static void symmetry_conditions(gm_plan *p) {
    const uint32_t nq = p->nq;
    memset(p->sb_gt, 0, sizeof(p->sb_gt));
    memset(p->sb_lt, 0, sizeof(p->sb_lt));
    p->aut = 1;
    p->sb_ok = false;
    std::vector<std::vector<uint8_t>> auts;
    uint8_t img[kMaxQ];
    if (!aut_search(p, 0, img, 0u, auts)) return;     // group too large to enumerate: no SB
    p->aut = auts.size();
    std::vector<size_t> S(auts.size());
    for (size_t i = 0; i < S.size(); ++i) S[i] = i;
    while (S.size() > 1) {
        int best = -1;
        uint32_t best_orbit = 0, best_size = 0;
        for (uint32_t l = 0; l < nq; ++l) {                // scan in phi order: earliest wins ties
            const uint32_t v = p->order[l];
            uint32_t orbit = 0;
            for (size_t a : S) orbit |= 1u << auts[a][v];
            const uint32_t sz = (uint32_t)__builtin_popcount(orbit);
            if (sz > best_size) { best = (int)v; best_orbit = orbit; best_size = sz; }
        }
        if (best_size <= 1) break;
        const uint32_t v = (uint32_t)best;
        for (uint32_t w = 0; w < nq; ++w) {
            if (w == v || !((best_orbit >> w) & 1u)) continue;
            // condition M[v] > M[w] on device ids (the orbit representative is its largest
            // image); device ids decrease with degree, so the earliest-ordered vertex is the
            // lowest-degree image and its later orbit-mates are bounded to higher-degree
            // (smaller) ids -- the degree-oriented DAG of triangle counting, generalised.
            // Checked when the later of the two is mapped.
            const uint32_t lv = p->pos[v], lw = p->pos[w];
            if (lv < lw) p->sb_lt[lw] |= 1u << lv;   // at w's level: M[w] < M[v]
            else p->sb_gt[lv] |= 1u << lw;           // at v's level: M[v] > M[w]
        }
        std::vector<size_t> T;
        for (size_t a : S) if (auts[a][v] == v) T.push_back(a);
        S.swap(T);
    }
    p->sb_ok = true;
}

extern "C" int gm_plan_query(const gm_graph *g, uint32_t nq, uint32_t mq, const uint32_t *qedges,
                             const uint32_t *qlabels, const uint32_t *order, uint32_t filter,
                             void *stream_, gm_plan **out) {
    set_error("");
    GM_REQ(g && out && qlabels && (mq == 0 || qedges), GM_ERR_ARG, "gm_plan_query: NULL argument");
    *out = nullptr;
    GM_REQ(nq >= 1 && nq <= (uint32_t)kMaxQ, GM_ERR_LIMIT, "gm_plan_query: nq=%u outside [1,%d]", nq, kMaxQ);
    GM_REQ(filter <= GM_FILTER_NLF, GM_ERR_ARG, "gm_plan_query: bad filter %u", filter);
    cudaStream_t st = (cudaStream_t)stream_;

    gm_plan tmp;
    tmp.g = g;
    tmp.nq = nq;
    tmp.filter = filter;
    memset(tmp.qadj, 0, sizeof(tmp.qadj));
    memset(tmp.qdeg, 0, sizeof(tmp.qdeg));
    for (uint32_t u = 0; u < nq; ++u) {
        GM_REQ(qlabels[u] < 0xffffffffu, GM_ERR_ARG, "gm_plan_query: bad label");
        tmp.qlab[u] = qlabels[u];
    }
    for (uint32_t i = 0; i < mq; ++i) {
        uint32_t a = qedges[2 * i], b = qedges[2 * i + 1];
        GM_REQ(a < nq && b < nq, GM_ERR_ARG, "gm_plan_query: query edge %u has vertex >= nq", i);
        if (a == b) continue;
        tmp.qadj[a] |= 1u << b;
        tmp.qadj[b] |= 1u << a;
    }
    for (uint32_t u = 0; u < nq; ++u) tmp.qdeg[u] = (uint32_t)__builtin_popcount(tmp.qadj[u]);
    {   // connectivity
        uint32_t seen = 1, frontier = 1;
        while (frontier) {
            uint32_t nxt = 0;
            for (uint32_t u = 0; u < nq; ++u) if (frontier >> u & 1u) nxt |= tmp.qadj[u];
            frontier = nxt & ~seen;
            seen |= nxt;
        }
        uint32_t all = nq == 32 ? 0xffffffffu : ((1u << nq) - 1);
        GM_REQ(seen == all, GM_ERR_ARG, "gm_plan_query: query graph is not connected");
    }

    // ---- filter on the GPU
    FilterSpec fs;
    memset(&fs, 0, sizeof(fs));
    fs.nq = nq; fs.S = g->S; fs.filter = filter;
    tmp.words = (uint32_t)((g->n + 31) / 32);
    fs.words = tmp.words;
    for (uint32_t u = 0; u < nq; ++u) {
        fs.qlab[u] = tmp.qlab[u] < g->S ? tmp.qlab[u] : 0xfffffffeu;  // unknown label: no candidates
        fs.qdeg[u] = tmp.qdeg[u];
        uint32_t cnt[kMaxQ], labs[kMaxQ], k = 0;
        for (uint32_t w = 0; w < nq; ++w) {
            if (!(tmp.qadj[u] >> w & 1u)) continue;
            uint32_t l = tmp.qlab[w], j = 0;
            while (j < k && labs[j] != l) ++j;
            if (j == k) { labs[k] = l; cnt[k] = 0; ++k; }
            cnt[j]++;
        }
        fs.nlf_n[u] = k;
        for (uint32_t j = 0; j < k; ++j) {
            // a neighbour label absent from G can never be matched: need > any count
            fs.nlf_lab[u][j] = labs[j] < g->S ? labs[j] : 0;
            fs.nlf_need[u][j] = labs[j] < g->S ? cnt[j] : 0xffffffffu;
        }
    }
    gm_plan *p = new gm_plan(tmp);
    p->cand = nullptr;
    FilterSpec *d_fs = nullptr;
    unsigned long long *d_cnt = nullptr;
    int rc = GM_OK;
    cudaError_t e = cudaSuccess;
    unsigned long long hc[kMaxQ];
    do {
        if ((e = cudaMalloc(&p->cand, sizeof(uint32_t) * (size_t)nq * (p->words ? p->words : 1))) != cudaSuccess) break;
        if ((e = cudaMalloc(&d_fs, sizeof(FilterSpec))) != cudaSuccess) break;
        if ((e = cudaMalloc(&d_cnt, sizeof(unsigned long long) * kMaxQ)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(d_fs, &fs, sizeof(fs), cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
        if ((e = cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * kMaxQ, st)) != cudaSuccess) break;
        if (g->n) {
            uint64_t warps = (g->n + 31) / 32;
            uint64_t blocks = (warps + 7) / 8;
            if (blocks > 148ull * 16) blocks = 148ull * 16;
            k_filter<<<(unsigned)blocks, 256, 0, st>>>(g->n, g->offs, g->lab, d_fs, p->cand, d_cnt);
            if ((e = cudaGetLastError()) != cudaSuccess) break;
        }
        if ((e = cudaMemcpyAsync(hc, d_cnt, sizeof(hc), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        for (uint32_t u = 0; u < nq; ++u) p->cand_count[u] = hc[u];
    } while (0);
    if (e != cudaSuccess) {
        set_error("gm_plan_query: CUDA error: %s", cudaGetErrorString(e));
        rc = e == cudaErrorMemoryAllocation ? GM_ERR_NOMEM : GM_ERR_CUDA;
    }
    cudaFree(d_fs);
    cudaFree(d_cnt);
    if (rc != GM_OK) { cudaFree(p->cand); delete p; return rc; }

    // ---- matching order
    if (order) {
        if (!connected_order(p, order)) {
            set_error("gm_plan_query: order is not a connected permutation of the query vertices");
            cudaFree(p->cand); delete p;
            return GM_ERR_ARG;
        }
        memcpy(p->order, order, sizeof(uint32_t) * nq);
    } else {
        ri_order(p, p->order);
    }
    for (uint32_t l = 0; l < nq; ++l) p->pos[p->order[l]] = l;
    for (uint32_t l = 0; l < nq; ++l) {
        uint32_t m = 0;
        for (uint32_t i = 0; i < l; ++i)
            if (p->qadj[p->order[l]] >> p->order[i] & 1u) m |= 1u << i;
        p->bw[l] = m;
    }
    symmetry_conditions(p);
    *out = p;
    return GM_OK;
}

extern "C" int gm_plan_info(const gm_plan *p, gm_plan_info_t *info) {
    GM_REQ(p && info, GM_ERR_ARG, "gm_plan_info: NULL argument");
    memset(info, 0, sizeof(*info));
    info->nq = p->nq;
    for (uint32_t i = 0; i < p->nq; ++i) {
        info->order[i] = p->order[i];
        info->backward[i] = p->bw[i];
        info->cand_count[i] = p->cand_count[i];
        info->sb_conditions += (uint32_t)(__builtin_popcount(p->sb_gt[i]) + __builtin_popcount(p->sb_lt[i]));
    }
    info->automorphisms = p->sb_ok ? p->aut : 0;
    return GM_OK;
}

extern "C" int gm_plan_candidates(const gm_plan *p, uint32_t u, uint32_t *words_host) {
    GM_REQ(p && words_host, GM_ERR_ARG, "gm_plan_candidates: NULL argument");
    GM_REQ(u < p->nq, GM_ERR_ARG, "gm_plan_candidates: u=%u >= nq", u);
    if (!p->words) return GM_OK;
    // the bitmap is over device ids; report it over the caller's (original) ids
    const uint64_t n = p->g->n;
    std::vector<uint32_t> dev(p->words), n2o(n);
    GM_CK(cudaMemcpy(dev.data(), p->cand + (uint64_t)u * p->words, sizeof(uint32_t) * p->words,
                     cudaMemcpyDeviceToHost));
    GM_CK(cudaMemcpy(n2o.data(), p->g->new2old, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
    memset(words_host, 0, sizeof(uint32_t) * p->words);
    for (uint64_t v = 0; v < n; ++v)
        if ((dev[v >> 5] >> (v & 31)) & 1u) words_host[n2o[v] >> 5] |= 1u << (n2o[v] & 31);
    return GM_OK;
}

extern "C" void gm_free_plan(gm_plan *p) {
    if (!p) return;
    cudaFree(p->cand);
    delete p;
}
