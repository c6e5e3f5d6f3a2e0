/*
 * gmatch.h -- C ABI of the B200-native fine-grained subgraph matcher.
 *
 * The operations follow the problem statement of PAPER.md (gMatch, arXiv 2604.10601):
 *   "Given a query graph Q and a data graph G, subgraph matching aims to find all
 *    embeddings of Q in G" (§1, line 82); an embedding is an injective, label- and
 *    edge-preserving map V(Q) -> V(G) (§2.1, Definition 1).
 * The search itself is the paper's fine-grained DFS extension with warp-level batch
 * exploration (§4.1-4.2, Algorithm 2) and its two-phase load balancing
 * (initial BFS pool of tau partial matches + idle-warp work stealing, §4.3, lines
 * 431-445), re-designed for sm_100a.
 *
 * Conventions for every entry point:
 *   - Return value: GM_OK (0) on success, a positive GM_* code otherwise; a one-line
 *     human-readable reason is then available from gm_last_error() (thread-local).
 *     No entry point aborts the process or prints.
 *   - `mem` arguments say where a caller buffer lives: GM_MEM_HOST (pageable or
 *     pinned host memory) or GM_MEM_DEVICE (memory of the current CUDA device).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls may synchronize `stream` internally where the host needs a device value
 *     (pool sizes, candidate counts); they return only after results are visible in
 *     the caller's output buffers.
 *   - Opaque handles (gm_graph, gm_plan) own device memory on the device that was
 *     current at creation; free them with gm_free_graph / gm_free_plan.  A plan
 *     borrows its graph: free plans before their graph.
 *   - Vertex ids are uint32 in [0, n); labels are uint32 in [0, num_labels).
 *   - Limits: n * num_labels < 2^32, stored adjacency entries < 2^32,
 *     query size 1 <= nq <= GM_MAX_QUERY, and (gm_count / gm_enumerate) maximum degree
 *     < 2^27 and, for queries of more than 8 vertices, n < 2^27 (a DFS stack entry packs a
 *     slice length with its source level, and a vertex id with its parent lane; DESIGN.md
 *     §5).  Exceeding a limit returns GM_ERR_LIMIT.
 */
#ifndef GMATCH_H
#define GMATCH_H

#include <stdint.h>

#if defined(__GNUC__)
#define GM_API __attribute__((visibility("default")))
#else
#define GM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GM_OK            0
#define GM_ERR_ARG       1   /* invalid argument (null pointer, bad id, disconnected query...) */
#define GM_ERR_CUDA      2   /* a CUDA runtime call failed */
#define GM_ERR_NOMEM     3   /* device allocation failed */
#define GM_ERR_LIMIT     4   /* a size limit documented above was exceeded */
#define GM_TIMEOUT       5   /* time limit hit: the reported count is a lower bound */

#define GM_MEM_HOST      0
#define GM_MEM_DEVICE    1

#define GM_MAX_QUERY     32

/* candidate filters (gm_plan_query `filter`) */
#define GM_FILTER_NONE   0   /* label only */
#define GM_FILTER_LDF    1   /* label and degree: L(v)=L(u), d(v) >= d(u) */
#define GM_FILTER_NLF    2   /* LDF + neighbour label frequency: for all labels l,
                                |N(v) with label l| >= |N(u) with label l| */

typedef struct gm_graph gm_graph;
typedef struct gm_plan gm_plan;
typedef struct gm_team gm_team;

/* ------------------------------------------------------------------ graph */

/*
 * gm_load_graph -- build the device data graph G from an edge list.
 *   n            number of vertices.
 *   m            number of (src[i], dst[i]) pairs.  Pairs are undirected edges;
 *                self loops and repeated pairs are dropped (G is simple, as
 *                Definition 1 assumes).
 *   src, dst     m vertex ids each, in `mem`.  Read only; not retained.
 *   labels       n labels in `mem`, or NULL for an unlabelled graph (all label 0).
 *   num_labels   |Sigma| >= 1; every label must be < num_labels.
 * Layout built: row r = v*num_labels + l holds
 * the neighbours of v whose label is l, ascending; offs has n*num_labels+1 entries.
 * On success *out receives a handle.  Needs ~40 bytes of scratch per input pair.
 */
GM_API int gm_load_graph(uint64_t n, uint64_t m, const uint32_t *src, const uint32_t *dst,
                  const uint32_t *labels, uint32_t num_labels, int mem, void *stream,
                  gm_graph **out);

typedef struct {
    uint64_t n;            /* vertices */
    uint64_t num_adj;      /* stored adjacency entries = 2 |E(G)| */
    uint32_t num_labels;
    uint32_t d_max;        /* maximum degree */
    uint64_t device_bytes; /* device memory held by the graph */
    uint32_t hubs;         /* vertices with a hub adjacency bitmap (gm_graph_build_hubs) */
    uint32_t hub_min_degree;
    uint64_t hub_bytes;    /* device bytes of the hub index (bitmaps + summary rows) */
    uint32_t hub_summary_words; /* words per hub summary row (1 bit per 256 vertices); 0 when the
                                   index fits in L2 and has no summary level */
    uint32_t reserved;
} gm_graph_info_t;

GM_API int gm_graph_info(const gm_graph *g, gm_graph_info_t *info);

/*
 * gm_graph_build_hubs -- (re)build the hub adjacency index: for the highest-degree
 * vertices (degree >= min_degree, at most budget_bytes / (4*ceil(n/32)) of them) a bitmap
 * of N(v) over all vertex ids, used by the search to test v in N(w) with one word read
 * instead of a binary search.  An index larger than the L2 cache
 * also gets a summary level: one bit per 256-vertex block of each bitmap (set iff the block
 * holds a neighbour), so most failing tests read an L2-resident summary word instead of a
 * DRAM sector of the bitmap.  summary: -1 = that rule, 0 = never (gm_load_graph's choice:
 * the extra dependent load measured 1-8 % slower on rmat24/26), 1 = always.
 * The search kernels read the summary only in a build with GM_HUB_SUMMARY=1 (the default
 * build compiles the test out: 3-52 % more tasks/s on rmat24/26); without it a summary is
 * built but unused.  gm_load_graph builds it with
 * min_degree 64 and a 64 MiB budget when the CSR fits in L2 beside it, else an 8 GiB budget
 * (at most a quarter of the free device memory); budget_bytes = 0 removes it.  Results
 * never depend on it.
 * Synchronizes `stream`.  Do not call while a search on this graph is running.
 */
GM_API int gm_graph_build_hubs(gm_graph *g, uint64_t budget_bytes, uint32_t min_degree, int summary,
                               void *stream);

/*
 * gm_graph_export -- copy the CSR back to host buffers (tests, debugging).
 *   offs_host: n*num_labels+1 uint32; nbr_host: num_adj uint32; labels_host: n uint32.
 *   Any pointer may be NULL to skip that array.
 */
GM_API int gm_graph_export(const gm_graph *g, uint32_t *offs_host, uint32_t *nbr_host, uint32_t *labels_host);

GM_API void gm_free_graph(gm_graph *g);

/* ------------------------------------------------------------------ query plan */

/*
 * gm_plan_query -- prepare query Q against G: candidate filter, matching order.
 *   nq, mq       |V(Q)| (1..GM_MAX_QUERY) and number of query edges.
 *   qedges       2*mq host uint32: edge i joins qedges[2i] and qedges[2i+1].
 *   qlabels      nq host uint32 labels.
 *   order        NULL for the planner's order (RI-style greedy, §3:
 *                "we generate phi on the CPU using the RI method"), or nq host uint32
 *                giving phi[0..nq-1]; it must be a permutation whose every vertex after
 *                the first has an earlier neighbour ("connected", §2.2),
 *                else GM_ERR_ARG.
 *   filter       GM_FILTER_NONE / _LDF / _NLF; every filter is sound (it never removes
 *                the image of a query vertex under an embedding), so counts do not
 *                depend on it.
 * Q must be connected (GM_ERR_ARG otherwise).  Runs the filter kernel on `stream`
 * and synchronizes it (the order uses the candidate counts).
 */
GM_API int gm_plan_query(const gm_graph *g, uint32_t nq, uint32_t mq, const uint32_t *qedges,
                  const uint32_t *qlabels, const uint32_t *order, uint32_t filter,
                  void *stream, gm_plan **out);

typedef struct {
    uint32_t nq;
    uint32_t order[GM_MAX_QUERY];       /* phi */
    uint32_t backward[GM_MAX_QUERY];    /* bit i of backward[l]: phi[i] is a backward
                                           neighbour of phi[l] (N_+^phi, Table 1) */
    uint64_t cand_count[GM_MAX_QUERY];  /* |C(u)| after filtering, by query vertex id */
    uint64_t automorphisms;             /* |Aut(Q)| (label-preserving), 0 if not enumerated */
    uint32_t sb_conditions;             /* number of symmetry-breaking conditions M[a] < M[b] */
} gm_plan_info_t;

GM_API int gm_plan_info(const gm_plan *p, gm_plan_info_t *info);

/*
 * gm_plan_candidates -- copy the candidate bitmap of query vertex u to the host:
 * bit (v % 32) of word v / 32 is 1 iff v passed the filter for u.  words_host holds
 * ceil(n/32) uint32.
 */
GM_API int gm_plan_candidates(const gm_plan *p, uint32_t u, uint32_t *words_host);

GM_API void gm_free_plan(gm_plan *p);

/* ------------------------------------------------------------------ search */

/* gm_run_opts.flags */
#define GM_FLAG_NO_SET_COUNT 1u  /* gm_count: validate every last-level candidate as its own task
                                    (Alg. 2 as written) instead of set-counting the last level
                                    when phi[last] has a single backward neighbour */
#define GM_FLAG_NO_PAIR_COUNT 4u /* gm_count: do not count the last two levels in bulk when
                                    phi[last-1] and phi[last] are non-adjacent vertices with one
                                    backward neighbour each (pair counting) */
#define GM_FLAG_STOP_AT_CAPACITY 8u /* gm_enumerate: stop the search once `capacity` rows are
                                    written (returns GM_TIMEOUT; *count_host is then the number
                                    found so far, >= capacity) -- for timing row output */
#define GM_FLAG_NO_POOL      16u /* diagnostic (tests): this rank claims no pool batches and gets
                                    work only by stealing (needs steal = 1; with a team, from
                                    other ranks' rings) */
#define GM_FLAG_COUNT_WORDS  32u /* gm_count: also count the algorithmic 4-byte words the DFS reads
                                    (gm_run_stats.words; DESIGN.md §6 defines the unit).  The
                                    counters cost 12-23 % throughput, so without this flag the
                                    search runs a kernel compiled without them and words = 0. */
#define GM_FLAG_NO_SIBLING   64u /* gm_count: never take the last level's candidates from the
                                    recorded siblings of phi[last-1] (GM_PATH_SIBLING) */
#define GM_FLAG_NO_GEN_CACHE 128u /* gm_count/gm_enumerate: GenerateTask at the hot level computes
                                    every backward row itself instead of reusing the part cached
                                    per grandparent (diagnostic: results are identical) */
#define GM_FLAG_NO_SYMMETRY  2u  /* gm_count: search every embedding instead of one per
                                    Aut(Q)-orbit (symmetry breaking, Appendix A) times |Aut(Q)|.
                                    Symmetry breaking is also skipped when `roots` is given. */

typedef struct {
    uint64_t tau;            /* initial task-pool threshold (§4.3); 0 = 1e6 */
    uint32_t rank, world;    /* this rank's share of the root candidates: vertex v is
                                owned by rank (v / root_chunk) % world; world 0 = 1 */
    uint32_t root_chunk;     /* 0 = 64 */
    uint32_t steal;          /* 1 = idle-warp work stealing on (gm_default_opts), 0 = off */
    uint32_t blocks_per_sm;  /* 0 = as many as fit */
    uint32_t warps_per_block;/* DFS warps per block: 0 (default) = the block size that keeps
                                the most warps resident for this query's shared memory; else
                                1..4 (<= 8-vertex queries) or 1..14 (larger ones); more:
                                GM_ERR_ARG; a block over 227 KB: GM_ERR_LIMIT */
    double   time_limit_ms;  /* 0 = none; on expiry the call returns GM_TIMEOUT */
    const uint32_t *roots;   /* optional host list of DISTINCT vertices restricting phi[0]'s
                                images to them (still filtered and rank-partitioned);
                                non-NULL with num_roots = 0 means no roots (count 0) */
    uint64_t num_roots;
    uint64_t pool_bytes_max; /* cap on the BFS pool's device bytes; 0 = 1 GiB */
    uint32_t flags;          /* GM_FLAG_* bits */
    void    *shared_pool_ctr;/* optional device pointer to a pool counter shared by several
                                ranks (gm_pool_counter_*): every rank then builds the SAME
                                initial pool (rank/world are ignored) and their DFS kernels
                                claim pool batches from this one counter -- dynamic chunk
                                assignment across GPUs through NVLink peer atomics */
    uint64_t root_seed;      /* 0: root candidates in device-id order (degree-descending: hubs
                                first, the heaviest subtrees claimed first); else a seeded
                                pseudo-random permutation of them, so a time-limited run
                                explores a uniform sample of the roots (the BFS pool keeps the
                                root order).  Counts of completed runs never depend on it; ranks
                                sharing a pool counter must pass the same seed. */
    gm_team *team;           /* optional stealing team (gm_team_open): idle warps also pop the
                                steal rings of the other ranks and post requests to them, and
                                the DFS ends when the whole team is out of work (cross-GPU
                                stealing, §4.3 "replicated at the block level
                                using global memory", one level up).  Every rank of the team
                                runs the same query with the same shared_pool_ctr slot (needed)
                                and the same options (time limits included); see gm_team_open
                                for the protocol.  NULL: stealing stays within this GPU. */
} gm_run_opts;

GM_API void gm_default_opts(gm_run_opts *o);

typedef struct {
    uint64_t count;           /* embeddings found by this rank */
    uint64_t roots;           /* root candidates owned by this rank */
    uint64_t pool_size;       /* partial matches in the initial pool */
    uint32_t pool_depth;      /* their length */
    uint32_t timed_out;
    uint64_t donations;       /* work items handed to idle warps (stealing) */
    uint64_t tasks;           /* candidate checks T_M(u,v) performed by the DFS kernel */
    uint64_t rounds;          /* warp scatter rounds (32-wide task batches) */
    float    dfs_ms;          /* device time of the DFS kernel launch (CUDA events) */
    float    total_ms;        /* device time of the whole call on `stream` */
    uint32_t dfs_launches;    /* DFS kernel launches in this call (0 or 1) */
    uint32_t kernel_launches; /* all kernels this call launched */
    uint32_t grid, block;     /* DFS launch shape */
    uint64_t words;           /* 4-byte words the DFS kernel read from the CSR and the candidate
                                 bitmaps: candidate reads + row-offset pairs + binary-search
                                 probes + bitmap words (algorithmic bytes = 4 * words); 0 unless
                                 GM_FLAG_COUNT_WORDS was set */
    uint64_t automorphisms;   /* |Aut(Q)| the count was scaled by (1: no symmetry breaking) */
    uint32_t paths;           /* GM_PATH_* bits: the exact shortcuts this call's DFS used */
    uint32_t stack_levels;    /* levels D of the k_dfs stack instantiation (8, 16, 24 (count only) or 32); 0: no DFS */
} gm_run_stats;

/* gm_run_stats.paths */
#define GM_PATH_SET_COUNT   1u  /* last level set-counted (count_last) */
#define GM_PATH_PAIR_COUNT  2u  /* last two levels pair-counted (count_two) */
#define GM_PATH_PAR_CHECKS  4u  /* per-parent check lists at the hot level (prep_checks) */
#define GM_PATH_SYMMETRY    8u  /* symmetry-breaking conditions enforced (count x |Aut(Q)|) */
#define GM_PATH_GEN_CACHE  32u  /* GenerateTask at the hot level reused a part cached per
                                   grandparent (gen_prep) */
#define GM_PATH_SIBLING    16u  /* last level's candidates from the recorded valid siblings of
                                   phi[last-1] (clique-like last levels) */

/*
 * gm_count -- count all embeddings of the plan's Q in G (this rank's share).
 *   count_out   one uint64 in `mem` receiving the count (device memory lets the
 *               caller all-reduce it across ranks without a host round trip).
 *   stats       optional host struct.
 * Returns GM_OK, or GM_TIMEOUT (count is the number found before the limit), or
 * GM_ERR_LIMIT when the count does not fit in 64 bits (count_out = UINT64_MAX).
 */
GM_API int gm_count(const gm_plan *p, const gm_run_opts *opts, uint64_t *count_out, int mem,
             gm_run_stats *stats, void *stream);

/*
 * gm_enumerate -- list embeddings: row k of `out` (nq uint32, in `mem`) holds the data
 * vertex of query vertex u at column u.  At most `capacity` rows are written, in no
 * particular order; *count_host receives the total number of embeddings (which may
 * exceed capacity: rows past capacity are counted but not written).
 */
GM_API int gm_enumerate(const gm_plan *p, const gm_run_opts *opts, uint32_t *out, uint64_t capacity,
                 int mem, uint64_t *count_host, gm_run_stats *stats, void *stream);

/* ------------------------------------------------------------------ multi-GPU pool counters */

/*
 * An array of 64-bit counters in one GPU's memory that the DFS kernels of several ranks
 * (processes, one per GPU) atomically claim pool batches from, over NVLink peer memory -- the
 * north_star's "root-level candidates ... partitioned across the 8 GPUs with dynamic chunk
 * assignment" (§4.3, 445: warps fetch from the pool with an atomic counter;
 * the inter-block mechanism is "replicated at the block level using global memory").
 * Slot k lives at (char *)counter_dev + k * GM_POOL_COUNTER_STRIDE (its own 128-byte line),
 * so a step of several queries gives each query its own slot and resets them all once.
 *   gm_pool_counter_create: allocate `slots` counters on the current device (zeroed); copies
 *       a GM_IPC_HANDLE_BYTES CUDA IPC handle into ipc_handle_out for the other ranks.
 *       slots in [1, 2^20], else GM_ERR_ARG.
 *   gm_pool_counter_open:   map another process's counters (any GPU of the node, or the same
 *       GPU) into this process; *counter_dev (+ k * stride) is then usable as shared_pool_ctr.
 *   gm_pool_counter_reset:  zero the first `slots` counters on `stream` (one rank).
 *   gm_pool_counter_close:  owner = 1 frees the allocation, owner = 0 unmaps it.
 * Memory model: the DFS claims with system-scope atomics (atomicAdd_system) and polls with
 * relaxed system-scope loads whenever shared_pool_ctr is set: a device-scope atomic is only
 * atomic among the threads of one GPU.
 * Protocol per step: reset all slots on one rank and synchronize that stream, barrier, then
 * every rank runs gm_count for query i with shared_pool_ctr = slot i and the same plan
 * inputs (no barrier between queries: slots are independent); sum the per-rank counts (one
 * all-reduce).  A slot must not be reset while a rank may still claim from it.
 */
#define GM_IPC_HANDLE_BYTES 64
#define GM_POOL_COUNTER_STRIDE 128
GM_API int gm_pool_counter_create(uint32_t slots, void **counter_dev, void *ipc_handle_out);
GM_API int gm_pool_counter_open(const void *ipc_handle, void **counter_dev);
GM_API int gm_pool_counter_reset(void *counter_dev, uint32_t slots, void *stream);
GM_API int gm_pool_counter_close(void *counter_dev, int owner);

/* ------------------------------------------------------------------ cross-GPU stealing team */

/*
 * A team of ranks (processes, one per GPU of a node) whose DFS kernels steal from each other
 * over NVLink peer memory, the paper's dynamic balancing phase (§4.3:
 * idle warps receive half of a busy warp's execution stack; "the same mechanism is replicated
 * at the block level using global memory") taken one level further, to GPUs.
 *   gm_team_export: allocate this device's search workspace (control block + steal ring) if
 *       needed and copy GM_TEAM_HANDLE_BYTES of CUDA IPC handles for it into handle_out.
 *   gm_team_open: world (1..8) ranks' exported handles, concatenated in rank order
 *       (world * GM_TEAM_HANDLE_BYTES bytes); maps every other rank's workspace into this
 *       process and returns a team handle for gm_run_opts.team.  Call on the device the
 *       searches will run on, after every rank exported.
 *   gm_team_free: unmap (call after the last search that uses the team).
 * Protocol: the ranks run the same sequence of searches with the team; search k runs on every
 * rank with the same plan inputs, options and shared_pool_ctr slot (a shared pool counter is
 * required: every rank then builds the same pool).  No barrier is needed between searches:
 * the team numbers its searches (epoch k, the same on every rank), every steal item carries
 * its epoch and is popped only by warps of that epoch, and each rank's work word is
 * (epoch << 32) | count.  Termination: a unit of work is counted in the lineage rank that
 * claimed its pool batch, wherever it runs; once the pool is exhausted a lineage count only
 * decreases, and a word tagged with another epoch holds none of this search's units, so a
 * rank ends its DFS when every rank's word reads zero for its epoch.  Memory model: the
 * team's counters, ring positions and slot sequence numbers use system-scope atomics and
 * acquire loads; items are written before a __threadfence_system() and the slot's sequence
 * store that publishes them.
 */
#define GM_TEAM_HANDLE_BYTES 256
GM_API int gm_team_export(void *handle_out);
GM_API int gm_team_open(uint32_t world, uint32_t rank, const void *handles, gm_team **out);
GM_API void gm_team_free(gm_team *t);

/* Thread-local description of the last error (empty string if none). */
GM_API const char *gm_last_error(void);

/* Library version string. */
GM_API const char *gm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GMATCH_H */
