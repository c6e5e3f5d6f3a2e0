/*
 * gm_oracle.c -- plain, slow, obviously-correct CPU reference for subgraph matching.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this code.  The product
 * path (paper_2604_10601_b200/) never links, imports or executes anything here,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (§2.1, Definition 1):
 *   an embedding (match) of Q in G is an injective M : V(Q) -> V(G) with
 *     1) L(u) = L(M[u])                     for every query vertex u,
 *     2) e(M[u], M[u']) in E(G)             for every query edge e(u, u').
 *   "The goal of subgraph matching is to find all matches of Q in G" (line 143).
 *   Matches are NOT deduplicated by automorphisms (no symmetry breaking).
 *
 * How: textbook backtracking (Alg. 1's DFS-Search idea, lines 223-237, written
 * sequentially): query vertices are assigned one at a time in a connected order
 * chosen here (fixed vertex first, then smallest-id vertex adjacent to the
 * assigned set), each candidate is checked for label, injectivity and every
 * edge to an already-assigned query neighbour.  No filtering, no ordering
 * heuristics, no intersection tricks: slowness is the price of independence.
 *
 * Also here, written from their definitions (used as pins for the GPU filter):
 *   LDF (label-and-degree filter):   v in C(u)  iff  L(v)=L(u) and d(v) >= d(u)
 *   NLF (neighbour-label-frequency): additionally, for every label l,
 *        |{w in N(v) : L(w)=l}| >= |{u' in N(u) : L(u')=l}|
 *   (the north_star's "LDF/NLF candidate filter"; the paper only cites the
 *    filtering literature, §6.1 line 576 / Appendix C.)
 *
 * Parity status: pinned -- see tests/test_oracle.py (brute force over all
 * injective maps on <= 8-vertex graphs, K_k in K_n = n!/(n-k)!, cycles and
 * paths in C_n, stars, isomorphism invariance, the Figure 1 example reading).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t n;
    int64_t *off;   /* n+1 */
    uint32_t *adj;  /* sorted, deduplicated, symmetric, no self loops */
    uint32_t *lab;  /* n */
} or_graph;

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

static int cmp_u32(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

/* Build the simple undirected graph on the given (src,dst) pairs. */
or_graph *or_graph_new(int64_t n, int64_t m, const uint32_t *src, const uint32_t *dst,
                       const uint32_t *labels) {
    or_graph *g = (or_graph *)calloc(1, sizeof(or_graph));
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
    int64_t k = 0;
    for (int64_t i = 0; i < m; i++) {
        if (src[i] == dst[i]) continue;              /* simple graph: no self loops */
        key[k++] = ((uint64_t)src[i] << 32) | dst[i];
        key[k++] = ((uint64_t)dst[i] << 32) | src[i]; /* undirected: both directions */
    }
    qsort(key, (size_t)k, sizeof(uint64_t), cmp_u64);
    int64_t u = 0;
    for (int64_t i = 0; i < k; i++)                  /* drop parallel edges */
        if (i == 0 || key[i] != key[i - 1]) key[u++] = key[i];
    g->n = n;
    g->off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    g->adj = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(u + 1));
    g->lab = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < u; i++) {
        g->off[(key[i] >> 32) + 1]++;
        g->adj[i] = (uint32_t)(key[i] & 0xffffffffu);
    }
    for (int64_t v = 0; v < n; v++) g->off[v + 1] += g->off[v];
    for (int64_t v = 0; v < n; v++) g->lab[v] = labels ? labels[v] : 0;
    free(key);
    return g;
}

void or_graph_free(or_graph *g) {
    if (!g) return;
    free(g->off); free(g->adj); free(g->lab); free(g);
}

int64_t or_graph_num_adj(const or_graph *g) { return g->off[g->n]; }

void or_graph_export(const or_graph *g, int64_t *off, uint32_t *adj) {
    memcpy(off, g->off, sizeof(int64_t) * (size_t)(g->n + 1));
    memcpy(adj, g->adj, sizeof(uint32_t) * (size_t)g->off[g->n]);
}

static int has_edge(const or_graph *g, uint32_t a, uint32_t b) {
    const uint32_t *base = g->adj + g->off[a];
    size_t len = (size_t)(g->off[a + 1] - g->off[a]);
    return bsearch(&b, base, len, sizeof(uint32_t), cmp_u32) != NULL;
}

/* ---------------------------------------------------------------- matcher */

/* Embeddings found by the last or_count/or_count_budget call on this thread, including a
 * call whose node budget ran out (then a lower bound) -- lets bench.py time the oracle on
 * a bounded amount of search work.  Never used as an expected value. */
static _Thread_local uint64_t g_last_found;
uint64_t or_last_found(void) { return g_last_found; }

typedef struct {
    const or_graph *g;
    int nq;
    const uint32_t *qlab;
    int qadj[64][64];          /* query adjacency matrix */
    int order[64];             /* oracle's own assignment order */
    int first_back[64];        /* an earlier-ordered neighbour, or -1 */
    uint32_t map[64];          /* map[u] = data vertex of query vertex u */
    uint8_t *used;             /* used[v] = 1 if v is the image of some query vertex */
    uint64_t count, limit;
    uint64_t nodes, max_nodes;  /* search-tree nodes visited; budget (0 = none) */
    uint32_t *out;
    uint64_t out_cap;
    int fixed_u;
    uint32_t fixed_v;
} or_ctx;

static int feasible(or_ctx *c, int depth, uint32_t v) {
    int u = c->order[depth];
    if (c->g->lab[v] != c->qlab[u]) return 0;             /* Def. 1 clause 1 */
    if (c->used[v]) return 0;                             /* injectivity     */
    for (int i = 0; i < depth; i++) {                     /* Def. 1 clause 2 */
        int w = c->order[i];
        if (c->qadj[u][w] && !has_edge(c->g, c->map[w], v)) return 0;
    }
    return 1;
}

static void emit(or_ctx *c) {
    if (c->out && c->count < c->out_cap)
        for (int u = 0; u < c->nq; u++) c->out[c->count * (uint64_t)c->nq + (uint64_t)u] = c->map[u];
    c->count++;
}

static void search(or_ctx *c, int depth) {
    if (c->limit && c->count >= c->limit) return;
    if (c->max_nodes && ++c->nodes > c->max_nodes) return;   /* budget exhausted: caller discards */
    if (depth == c->nq) { emit(c); return; }
    int u = c->order[depth];
    if (depth == 0 && c->fixed_u >= 0) {
        uint32_t v = c->fixed_v;
        if (v < (uint64_t)c->g->n && feasible(c, 0, v)) {
            c->map[u] = v; c->used[v] = 1;
            search(c, 1);
            c->used[v] = 0;
        }
        return;
    }
    if (c->first_back[depth] >= 0) {
        uint32_t w = c->map[c->first_back[depth]];
        for (int64_t e = c->g->off[w]; e < c->g->off[w + 1]; e++) {
            uint32_t v = c->g->adj[e];
            /* the budget also counts candidates examined, so a budgeted call is bounded even
               when every node scans a hub's adjacency (budget only: no effect on results) */
            if (c->max_nodes && ++c->nodes > c->max_nodes) return;
            if (!feasible(c, depth, v)) continue;
            c->map[u] = v; c->used[v] = 1;
            search(c, depth + 1);
            c->used[v] = 0;
        }
    } else {
        for (int64_t v = 0; v < c->g->n; v++) {
            if (c->max_nodes && ++c->nodes > c->max_nodes) return;
            if (!feasible(c, depth, (uint32_t)v)) continue;
            c->map[u] = (uint32_t)v; c->used[v] = 1;
            search(c, depth + 1);
            c->used[v] = 0;
        }
    }
}

/*
 * Count (and optionally list) all embeddings of Q in G.
 *   qedges: mq pairs (u, u') of query vertex ids in [0, nq); qlabels: nq labels.
 *   fixed_u >= 0 restricts to embeddings with M[fixed_u] = fixed_v.
 *   limit > 0 stops after `limit` embeddings.  out (nullable) receives up to
 *   out_cap embeddings, each nq data-vertex ids indexed by query vertex id.
 * Returns the number of embeddings found (-1 on bad arguments, as UINT64_MAX).
 */
uint64_t or_count_budget(const or_graph *g, int nq, int mq, const uint32_t *qedges,
                         const uint32_t *qlabels, int fixed_u, uint32_t fixed_v, uint64_t limit,
                         uint32_t *out, uint64_t out_cap, uint64_t max_nodes);

uint64_t or_count(const or_graph *g, int nq, int mq, const uint32_t *qedges,
                  const uint32_t *qlabels, int fixed_u, uint32_t fixed_v, uint64_t limit,
                  uint32_t *out, uint64_t out_cap) {
    return or_count_budget(g, nq, mq, qedges, qlabels, fixed_u, fixed_v, limit, out, out_cap, 0);
}

/*
 * Same as or_count, with a budget of max_nodes units of search work (0 = none): one unit per
 * visited search-tree node and per candidate examined.
 * Returns UINT64_MAX - 1 when the budget ran out (the count is then unknown); used only to
 * pick samples the oracle can finish, never to produce a partial expected value.
 */
uint64_t or_count_budget(const or_graph *g, int nq, int mq, const uint32_t *qedges,
                         const uint32_t *qlabels, int fixed_u, uint32_t fixed_v, uint64_t limit,
                         uint32_t *out, uint64_t out_cap, uint64_t max_nodes) {
    if (nq <= 0 || nq > 64) return UINT64_MAX;
    or_ctx *c = (or_ctx *)calloc(1, sizeof(or_ctx));
    c->g = g; c->nq = nq; c->qlab = qlabels; c->limit = limit; c->out = out; c->out_cap = out_cap;
    c->fixed_u = fixed_u; c->fixed_v = fixed_v; c->max_nodes = max_nodes;
    for (int i = 0; i < mq; i++) {
        uint32_t a = qedges[2 * i], b = qedges[2 * i + 1];
        if (a >= (uint32_t)nq || b >= (uint32_t)nq) { free(c); return UINT64_MAX; }
        if (a != b) c->qadj[a][b] = c->qadj[b][a] = 1;
    }
    int placed[64] = {0};
    c->order[0] = fixed_u >= 0 ? fixed_u : 0;
    placed[c->order[0]] = 1;
    for (int d = 1; d < nq; d++) {
        int pick = -1;
        for (int u = 0; u < nq && pick < 0; u++) {
            if (placed[u]) continue;
            for (int i = 0; i < d; i++) if (c->qadj[u][c->order[i]]) { pick = u; break; }
        }
        if (pick < 0) for (int u = 0; u < nq; u++) if (!placed[u]) { pick = u; break; }
        c->order[d] = pick; placed[pick] = 1;
    }
    for (int d = 0; d < nq; d++) {
        c->first_back[d] = -1;
        for (int i = 0; i < d; i++)
            if (c->qadj[c->order[d]][c->order[i]]) { c->first_back[d] = c->order[i]; break; }
    }
    c->used = (uint8_t *)calloc((size_t)g->n + 1, 1);
    search(c, 0);
    g_last_found = c->count;
    uint64_t r = (c->max_nodes && c->nodes > c->max_nodes) ? UINT64_MAX - 1 : c->count;
    free(c->used); free(c);
    return r;
}

/* ---------------------------------------------------------------- filters */

/*
 * kind = 1: LDF only; kind = 2: LDF and NLF.
 * out[u * n + v] = 1 iff data vertex v passes the filter for query vertex u.
 */
int or_filter(const or_graph *g, int nq, int mq, const uint32_t *qedges, const uint32_t *qlabels,
              int kind, uint32_t num_labels, uint8_t *out) {
    if (nq <= 0 || nq > 64) return -1;
    int qdeg[64] = {0};
    uint32_t *qnlf = (uint32_t *)calloc((size_t)nq * num_labels, sizeof(uint32_t));
    int qadj[64][64];
    memset(qadj, 0, sizeof(qadj));
    for (int i = 0; i < mq; i++) {
        uint32_t a = qedges[2 * i], b = qedges[2 * i + 1];
        if (a == b || qadj[a][b]) continue;
        qadj[a][b] = qadj[b][a] = 1;
        qdeg[a]++; qdeg[b]++;
        qnlf[a * num_labels + qlabels[b]]++;
        qnlf[b * num_labels + qlabels[a]]++;
    }
    uint32_t *cnt = (uint32_t *)calloc(num_labels, sizeof(uint32_t));
    for (int64_t v = 0; v < g->n; v++) {
        int64_t d = g->off[v + 1] - g->off[v];
        if (kind >= 2) {
            memset(cnt, 0, sizeof(uint32_t) * num_labels);
            for (int64_t e = g->off[v]; e < g->off[v + 1]; e++) cnt[g->lab[g->adj[e]]]++;
        }
        for (int u = 0; u < nq; u++) {
            int ok = g->lab[v] == qlabels[u] && d >= qdeg[u];
            if (ok && kind >= 2)
                for (uint32_t l = 0; l < num_labels; l++)
                    if (cnt[l] < qnlf[u * num_labels + l]) { ok = 0; break; }
            out[(int64_t)u * g->n + v] = (uint8_t)ok;
        }
    }
    free(cnt); free(qnlf);
    return 0;
}
