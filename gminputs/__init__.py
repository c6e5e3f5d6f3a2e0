"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module is the ONE piece of code both sides of the parity check may use
(task rule: "only the seeded input generators serve both, from a module of
their own").  It holds no subgraph-matching arithmetic: it only draws graphs,
labels and query graphs.  Every random number comes from a counter-based
generator (``rng_u64``) so that the numpy implementation here and the CUDA
implementation in ``gminputs/gen_gpu.cu`` (used for graphs too large for host
generation) produce bit-identical edge lists for the same seed.

Workload shapes follow PAPER.md §6.1 "Datasets" / "Query Sets" (lines 582-677):
  * R-MAT graphs (PaRMAT-style, a,b,c,d = 0.57,0.19,0.19,0.05, Graph500 values),
  * Erdős–Rényi graphs G(n, M) with M = n*avg_deg/2 sampled edges,
  * labels "assigned with a label uniformly at random" (§6.1) or Zipf-skewed
    (Appendix A: P(label=l) ∝ (l+1)^-alpha),
  * query graphs: "start with a random seed vertex from the data graph and
    iteratively expand it by adding random neighboring vertices, along with all
    their connecting edges" (§6.1) -> ``random_query``; and a sparse
    random-walk variant keeping only the walked edges -> ``random_walk_query``.

Edge lists are returned as directed (src, dst) uint32 pairs of an UNDIRECTED
graph; duplicates and self loops may be present and are removed by every
consumer (the oracle and gm_load_graph both define the graph as the simple
undirected graph on the given pairs).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_STREAM_MUL = np.uint64(0xD1B54A32D192ED03)

# stream ids (part of the generator contract shared with gen_gpu.cu)
STREAM_RMAT = 1
STREAM_ER = 2
STREAM_LABEL = 3
STREAM_QUERY = 4

RMAT_ABC = (0.57, 0.19, 0.19)  # d = 0.05
RMAT_SCRAMBLE_MUL = 0x5851F42D4C957F2D  # odd => x -> (A*x + B) mod 2^scale is a bijection
RMAT_SCRAMBLE_ADD = 0x14057B7EF767814F


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def rng_u64(seed: int, stream: int, idx) -> np.ndarray:
    """Counter-based 64-bit random words: mix64(mix64(seed ^ stream*K) + idx*GOLDEN)."""
    with np.errstate(over="ignore"):
        key = _mix64(np.array([(seed ^ (stream * 0xD1B54A32D192ED03)) & M64], dtype=np.uint64))[0]
        i = np.asarray(idx, dtype=np.uint64)
        return _mix64(key + i * _GOLDEN)


def rng_unit(seed: int, stream: int, idx) -> np.ndarray:
    """Uniform doubles in [0,1) with 53 random bits."""
    return (rng_u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


# ----------------------------------------------------------------------------- graphs

def rmat_edges(scale: int, edge_factor: int, seed: int, chunk: int = 1 << 22):
    """R-MAT edge list with n = 2^scale vertices and m = edge_factor * n sampled edges.

    Edge e draws one uniform per recursion level k (counter e*scale + k) and
    descends into quadrant a/b/c/d; vertex ids are then scrambled with the
    affine bijection v -> (A v + B) mod 2^scale so hubs are not all at id 0.
    """
    n = 1 << scale
    m = edge_factor * n
    a, b, c = RMAT_ABC
    src = np.empty(m, dtype=np.uint32)
    dst = np.empty(m, dtype=np.uint32)
    mask = np.uint64(n - 1)
    A = np.uint64(RMAT_SCRAMBLE_MUL & M64)
    B = np.uint64(RMAT_SCRAMBLE_ADD & M64)
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        e = np.arange(lo, hi, dtype=np.uint64)
        s = np.zeros(hi - lo, dtype=np.uint64)
        d = np.zeros(hi - lo, dtype=np.uint64)
        for k in range(scale):
            u = rng_unit(seed, STREAM_RMAT, e * np.uint64(scale) + np.uint64(k))
            bit = np.uint64(1) << np.uint64(scale - 1 - k)
            sb = u >= (a + b)                      # quadrants c, d set the src bit
            db = ((u >= a) & (u < a + b)) | (u >= a + b + c)  # quadrants b, d set the dst bit
            s |= np.where(sb, bit, np.uint64(0))
            d |= np.where(db, bit, np.uint64(0))
        with np.errstate(over="ignore"):
            s = (s * A + B) & mask
            d = (d * A + B) & mask
        src[lo:hi] = s.astype(np.uint32)
        dst[lo:hi] = d.astype(np.uint32)
    return n, src, dst


def er_edges(n: int, avg_deg: float, seed: int):
    """Erdős–Rényi G(n, M) with M = round(n*avg_deg/2) uniformly drawn vertex pairs."""
    m = int(round(n * avg_deg / 2))
    e = np.arange(m, dtype=np.uint64)
    src = (rng_u64(seed, STREAM_ER, 2 * e) % np.uint64(n)).astype(np.uint32)
    dst = (rng_u64(seed, STREAM_ER, 2 * e + np.uint64(1)) % np.uint64(n)).astype(np.uint32)
    return n, src, dst


def uniform_labels(n: int, num_labels: int, seed: int) -> np.ndarray:
    """§6.1: 'each vertex is assigned with a label uniformly at random'."""
    if num_labels <= 1:
        return np.zeros(n, dtype=np.uint32)
    v = np.arange(n, dtype=np.uint64)
    return (rng_u64(seed, STREAM_LABEL, v) % np.uint64(num_labels)).astype(np.uint32)


def zipf_labels(n: int, num_labels: int, alpha: float, seed: int) -> np.ndarray:
    """Appendix A: P(label = l) = (l+1)^-alpha / sum_i i^-alpha, l in [0, |Sigma|-1]."""
    w = (np.arange(num_labels, dtype=np.float64) + 1.0) ** (-alpha)
    cdf = np.cumsum(w / w.sum())
    cdf[-1] = 1.0
    u = rng_unit(seed, STREAM_LABEL, np.arange(n, dtype=np.uint64))
    return np.searchsorted(cdf, u, side="right").astype(np.uint32)


def complete_graph(n: int):
    s, d = np.triu_indices(n, 1)
    return n, s.astype(np.uint32), d.astype(np.uint32)


def cycle_graph(n: int):
    v = np.arange(n, dtype=np.uint32)
    return n, v, ((v + 1) % n).astype(np.uint32)


def path_graph(n: int):
    v = np.arange(n - 1, dtype=np.uint32)
    return n, v, v + 1


def star_graph(leaves: int):
    v = np.arange(1, leaves + 1, dtype=np.uint32)
    return leaves + 1, np.zeros(leaves, dtype=np.uint32), v


def simple_adjacency(n: int, src: np.ndarray, dst: np.ndarray):
    """Sorted, deduplicated, symmetric adjacency (offsets, neighbors) of the simple graph.

    Used only to draw query graphs (random_query) — an input-side helper, not
    the oracle's or the GPU path's graph representation.
    """
    s = np.concatenate([src, dst]).astype(np.uint64)
    d = np.concatenate([dst, src]).astype(np.uint64)
    keep = s != d
    key = np.unique((s[keep] << np.uint64(32)) | d[keep])
    s = (key >> np.uint64(32)).astype(np.int64)
    nb = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    offs = np.zeros(n + 1, dtype=np.int64)
    offs[1:] = np.cumsum(np.bincount(s, minlength=n))
    return offs, nb


# ----------------------------------------------------------------------------- queries

class Query:
    """A small labelled query graph Q: vertices 0..n-1, undirected edge list, labels."""

    def __init__(self, n, edges, labels, name=""):
        self.n = int(n)
        e = sorted({(min(a, b), max(a, b)) for a, b in edges if a != b})
        self.edges = np.array(e, dtype=np.uint32).reshape(-1, 2)
        self.labels = np.asarray(labels, dtype=np.uint32).reshape(self.n)
        self.name = name

    @property
    def avg_degree(self) -> float:
        return 2.0 * len(self.edges) / max(self.n, 1)

    def __repr__(self):
        return f"Query({self.name!r}, n={self.n}, m={len(self.edges)})"


class HostAdjacency:
    """neighbors(v) of the simple graph, from host CSR arrays (simple_adjacency)."""

    def __init__(self, offs, nbrs):
        self.offs, self.nbrs = offs, nbrs
        self.n = len(offs) - 1

    def neighbors(self, v):
        return self.nbrs[int(self.offs[v]):int(self.offs[v + 1])]


def random_query(offs, nbrs, labels, size: int, seed: int, **kw) -> Query:
    """grow_query over host CSR arrays."""
    return grow_query(HostAdjacency(offs, nbrs), labels, size, seed, **kw)


def grow_query(adj, labels, size: int, seed: int, max_restarts: int = 1000,
               dense: bool = False, min_avg_degree: float = 0.0, with_vertices: bool = False):
    """§6.1 procedure: random seed vertex, repeatedly add a uniformly random vertex
    adjacent to the current set, keep ALL edges among chosen vertices (induced).
    `adj` provides .n and .neighbors(v) (sorted, simple graph): HostAdjacency or the
    device-scanning gminputs.gpu.DeviceNeighbors -- both give identical queries.

    dense=True draws the next vertex uniformly among the frontier vertices with the MOST
    neighbours in the chosen set (on sparse power-law graphs the plain procedure almost
    always returns trees; Appendix A's "dense" class needs d_avg >= 3).  Restarts until
    the query's average degree reaches min_avg_degree.  with_vertices=True also returns the
    data vertices the query was grown from (query vertex i = chosen[i]: one embedding)."""
    n = adj.n
    ctr = 0
    for _ in range(max_restarts):
        r = int(rng_u64(seed, STREAM_QUERY, ctr)); ctr += 1
        v0 = r % n
        chosen = [v0]
        cset = {v0}
        while len(chosen) < size:
            conn = {}
            for v in chosen:
                for w in adj.neighbors(v):
                    w = int(w)
                    if w not in cset:
                        conn[w] = conn.get(w, 0) + 1
            if not conn:
                break
            if dense:
                best = max(conn.values())
                fr = sorted(w for w, c in conn.items() if c == best)
            else:
                fr = sorted(conn)
            r = int(rng_u64(seed, STREAM_QUERY, ctr)); ctr += 1
            w = fr[r % len(fr)]
            chosen.append(w)
            cset.add(w)
        if len(chosen) == size:
            idx = {v: i for i, v in enumerate(chosen)}
            edges = []
            for v in chosen:
                for w in adj.neighbors(v):
                    w = int(w)
                    if w in idx and idx[v] < idx[w]:
                        edges.append((idx[v], idx[w]))
            if 2.0 * len(edges) / size < min_avg_degree:
                continue
            q = Query(size, edges, [int(labels[v]) for v in chosen], name=f"rq{size}_s{seed}")
            return (q, chosen) if with_vertices else q
    raise RuntimeError("random_query: could not grow a connected query (isolated region)")


def random_walk_query(offs, nbrs, labels, size: int, seed: int, **kw) -> Query:
    """walk_query over host CSR arrays."""
    return walk_query(HostAdjacency(offs, nbrs), labels, size, seed, **kw)


def walk_query(adj, labels, size: int, seed: int, max_steps: int = 100000) -> Query:
    """Sparse variant: a random walk from a random vertex until `size` distinct vertices
    are visited; only the traversed edges are kept (a spanning tree plus revisits)."""
    n = adj.n
    ctr = 0
    for _ in range(1000):
        r = int(rng_u64(seed, STREAM_QUERY, ctr)); ctr += 1
        cur = r % n
        if len(adj.neighbors(cur)) == 0:
            continue
        idx = {cur: 0}
        order = [cur]
        edges = set()
        steps = 0
        while len(order) < size and steps < max_steps:
            nb = adj.neighbors(cur)
            deg = len(nb)
            r = int(rng_u64(seed, STREAM_QUERY, ctr)); ctr += 1
            nxt = int(nb[r % deg])
            if nxt not in idx:
                idx[nxt] = len(order)
                order.append(nxt)
            a, b = idx[cur], idx[nxt]
            edges.add((min(a, b), max(a, b)))
            cur = nxt
            steps += 1
        if len(order) == size:
            return Query(size, sorted(edges), [int(labels[v]) for v in order], name=f"wq{size}_s{seed}")
    raise RuntimeError("random_walk_query: walk did not reach the requested size")


# fixed unlabelled patterns (small-pattern regime, §6.1 "predefined query graphs")
def triangle() -> Query:
    return Query(3, [(0, 1), (1, 2), (0, 2)], [0, 0, 0], "triangle")


def clique(k: int) -> Query:
    return Query(k, [(i, j) for i in range(k) for j in range(i + 1, k)], [0] * k, f"clique{k}")


def cycle(k: int) -> Query:
    return Query(k, [(i, (i + 1) % k) for i in range(k)], [0] * k, f"cycle{k}")


def path(k: int) -> Query:
    return Query(k, [(i, i + 1) for i in range(k - 1)], [0] * k, f"path{k}")


def star(leaves: int) -> Query:
    return Query(leaves + 1, [(0, i) for i in range(1, leaves + 1)], [0] * (leaves + 1), f"star{leaves}")


def tailed_triangle(labels=(0, 1, 2, 3)) -> Query:
    """Config 1's 4-vertex tailed triangle: triangle 0-1-2 with tail 2-3."""
    return Query(4, [(0, 1), (1, 2), (0, 2), (2, 3)], list(labels), "tailed_triangle")
