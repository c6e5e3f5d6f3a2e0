// gm_internal.cuh -- shared internals of libgmatch (graph/plan structs, error plumbing).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/gmatch.h"

namespace gm {

void set_error(const char *fmt, ...);

#define GM_CK(call)                                                                   \
    do {                                                                              \
        cudaError_t _e = (call);                                                      \
        if (_e != cudaSuccess) {                                                      \
            ::gm::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                \
                            cudaGetErrorString(_e));                                  \
            return _e == cudaErrorMemoryAllocation ? GM_ERR_NOMEM : GM_ERR_CUDA;      \
        }                                                                             \
    } while (0)

#define GM_REQ(cond, code, ...)                                                       \
    do {                                                                              \
        if (!(cond)) {                                                                \
            ::gm::set_error(__VA_ARGS__);                                             \
            return (code);                                                            \
        }                                                                             \
    } while (0)

constexpr int kWarp = 32;
constexpr int kMaxQ = GM_MAX_QUERY;

}  // namespace gm

// Device data graph: label-partitioned CSR.
struct gm_graph {
    uint64_t n = 0;
    uint32_t S = 1;            // number of labels
    uint64_t nadj = 0;         // stored adjacency entries
    uint32_t dmax = 0;
    int device = 0;
    uint32_t *offs = nullptr;  // n*S + 1 row offsets (row = v*S + label)
    uint32_t *nbr = nullptr;   // nadj neighbour ids, ascending inside each row
    uint32_t *lab = nullptr;   // n vertex labels
    uint64_t bytes = 0;
    // vertex renumbering by decreasing degree (graph.cu): device ids are new ids
    uint32_t *old2new = nullptr;   // n: original id -> device id
    uint32_t *new2old = nullptr;   // n: device id -> original id
    // hub adjacency index (hubs.cu): device ids 0..nhubs-1 (the highest-degree vertices)
    // each have a bitmap of N(v) over device ids, row v of hub_bits
    uint32_t nhubs = 0;
    uint32_t hub_min_degree = 0;
    uint32_t hub_words = 0;        // ceil(n/32) words per hub bitmap
    uint32_t *hub_bits = nullptr;  // nhubs * hub_words
    // two-level index for indexes larger than L2 (hubs.cu): bit b of hub h's summary row is 1
    // iff its bitmap has a set bit among vertices [256 b, 256 b + 256) (one 32-byte sector)
    uint32_t summ_words = 0;       // ceil(n / 8192) words per summary row; 0: no summary
    uint32_t summ_first = 0;       // hubs h >= summ_first have a summary row (selective enough)
    uint32_t *hub_summ = nullptr;  // (nhubs - summ_first) * summ_words
};

namespace gm {
int build_hubs(gm_graph *g, uint64_t budget_bytes, uint32_t min_degree, int summary, cudaStream_t st);
void free_hubs(gm_graph *g);
constexpr uint64_t kDefaultHubBudget = 64ull << 20;   // fits beside the graph in the 126 MB L2
constexpr uint64_t kLargeHubBudget = 8ull << 30;     // graphs whose CSR cannot stay in L2
// default hub budget for a graph: the L2-resident budget when the CSR fits in L2 beside it,
// else the large one (at most a quarter of the free device memory)
uint64_t default_hub_budget(const gm_graph *g);
constexpr uint32_t kDefaultHubMinDegree = 64;
}  // namespace gm

// Query plan: matching order, backward sets, candidate bitmaps.
struct gm_plan {
    const gm_graph *g = nullptr;
    uint32_t nq = 0;
    uint32_t order[gm::kMaxQ];      // phi[l] = query vertex at position l
    uint32_t pos[gm::kMaxQ];        // inverse of order
    uint32_t qlab[gm::kMaxQ];       // label by query vertex id
    uint32_t qdeg[gm::kMaxQ];
    uint32_t qadj[gm::kMaxQ];       // adjacency bitmask by query vertex id
    uint32_t bw[gm::kMaxQ];         // bit i of bw[l]: phi[i] adjacent to phi[l], i < l
    uint64_t cand_count[gm::kMaxQ]; // by query vertex id
    uint32_t filter = 0;
    uint32_t words = 0;             // ceil(n/32)
    uint32_t *cand = nullptr;       // nq * words bitmaps, by query vertex id
    // symmetry breaking (plan.cu): |Aut(Q)| (label-preserving) and, per position l, the
    // positions i < l with a condition M[phi[i]] < M[phi[l]] (sb_gt) or > (sb_lt)
    uint64_t aut = 1;
    bool sb_ok = false;             // conditions computed (|Aut| small enough to enumerate)
    uint32_t sb_gt[gm::kMaxQ];      // v = M[phi[l]] must be greater than M[phi[i]]
    uint32_t sb_lt[gm::kMaxQ];      // v must be smaller than M[phi[i]]
};
