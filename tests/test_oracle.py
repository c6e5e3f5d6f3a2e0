"""Pins for the CPU oracle (oracle/gm_oracle.c) against things other than itself.

Each pin is chosen so that a plausible bug in the oracle (a dropped edge check,
a missing injectivity test, a label test on the wrong side, an off-by-one in the
order, a wrong fixed-root path) fails at least one of them:
  * brute force over ALL injective maps V(Q)->V(G) on <= 8-vertex graphs
    (Definition 1 evaluated literally);
  * closed forms: K_k in K_n = n!/(n-k)!  (every injective map is an embedding),
    C_n in C_n = 2n, P_k in C_n = 2n, C_k in C_n = 0 (k<n), stars
    sum_v d(v)!/(d(v)-s)!, triangles = trace(A^3), labelled triangles
    = trace(P_a A P_b A P_c A), 4-cycles = tr(A^4) - 2 sum d^2 + sum d;
  * the Figure 1 example (tests/golden/fig1_example.txt, its values quoted from
    the paper text: 112 matches, the example embedding, the candidate sets);
  * invariants: isomorphism invariance, sum over fixed roots = total.
"""
import itertools
import math

import numpy as np
import pytest

import gminputs as gi
from conftest import load_fig1
from oracle import OracleGraph


def brute_force(n, src, dst, labels, q):
    """All injective maps checked clause by clause against Definition 1."""
    E = {(int(a), int(b)) for a, b in zip(src, dst) if a != b}
    E |= {(b, a) for a, b in E}
    out = []
    for img in itertools.permutations(range(n), q.n):
        if any(labels[img[u]] != q.labels[u] for u in range(q.n)):
            continue
        if all((img[a], img[b]) in E for a, b in q.edges):
            out.append(img)
    return sorted(out)


def small_random_graph(seed, n, p, nl):
    rs = np.random.default_rng(seed)
    pairs = [(a, b) for a in range(n) for b in range(a + 1, n) if rs.random() < p]
    src = np.array([a for a, _ in pairs], np.uint32)
    dst = np.array([b for _, b in pairs], np.uint32)
    lab = rs.integers(0, nl, n).astype(np.uint32)
    return n, src, dst, lab


def small_random_query(seed, k, nl, connected=True):
    rs = np.random.default_rng(seed + 7777)
    edges = set()
    for v in range(1, k):
        if connected:
            edges.add((int(rs.integers(0, v)), v))
    for a in range(k):
        for b in range(a + 1, k):
            if rs.random() < 0.35:
                edges.add((a, b))
    return gi.Query(k, sorted(edges), rs.integers(0, nl, k).tolist())


@pytest.mark.parametrize("seed", range(120))
def test_brute_force_small(seed):
    n = 5 + seed % 4                     # 5..8 data vertices
    nl = 1 + seed % 3
    n, src, dst, lab = small_random_graph(seed, n, 0.35 + 0.1 * (seed % 3), nl)
    q = small_random_query(seed, 2 + seed % 4, nl, connected=(seed % 5 != 0))
    g = OracleGraph(n, src, dst, lab)
    bf = brute_force(n, src, dst, lab, q)
    assert g.count(q) == len(bf)
    got = [tuple(int(x) for x in r) for r in g.enumerate(q)]
    assert got == bf


def test_duplicates_and_self_loops_ignored():
    src = np.array([0, 1, 1, 1, 2, 0], np.uint32)
    dst = np.array([1, 0, 1, 2, 0, 2], np.uint32)
    g = OracleGraph(3, src, dst)
    off, adj = g.csr()
    assert off.tolist() == [0, 2, 4, 6]
    assert adj.tolist() == [1, 2, 0, 2, 0, 1]
    assert g.count(gi.triangle()) == 6


@pytest.mark.parametrize("n,k", [(4, 3), (5, 3), (6, 4), (7, 2), (8, 5), (9, 4), (6, 6), (5, 1)])
def test_clique_in_clique(n, k):
    g = OracleGraph(*gi.complete_graph(n))
    assert g.count(gi.clique(k)) == math.factorial(n) // math.factorial(n - k)


@pytest.mark.parametrize("n", [3, 4, 5, 8, 13])
def test_cycles_and_paths_in_cycle(n):
    g = OracleGraph(*gi.cycle_graph(n))
    assert g.count(gi.cycle(n)) == 2 * n
    for k in range(3, n):
        assert g.count(gi.cycle(k)) == 0
    for k in range(2, n + 1):
        assert g.count(gi.path(k)) == 2 * n
    assert g.count(gi.path(1)) == n


@pytest.mark.parametrize("seed", range(6))
def test_star_closed_form(seed):
    n, src, dst = gi.er_edges(40, 6.0, seed)
    g = OracleGraph(n, src, dst)
    off, _ = g.csr()
    deg = np.diff(off)
    for s in (1, 2, 3):
        expect = sum(math.perm(int(d), s) for d in deg)
        assert g.count(gi.star(s)) == expect


def _adj_matrix(n, src, dst):
    A = np.zeros((n, n), dtype=np.int64)
    for a, b in zip(src, dst):
        if a != b:
            A[a, b] = A[b, a] = 1
    return A


@pytest.mark.parametrize("seed", range(5))
def test_triangles_and_4cycles_trace(seed):
    n, src, dst = gi.er_edges(60, 8.0, seed)
    g = OracleGraph(n, src, dst)
    A = _adj_matrix(n, src, dst)
    d = A.sum(1)
    assert g.count(gi.triangle()) == int(np.trace(A @ A @ A))
    A4 = np.trace(np.linalg.matrix_power(A, 4))
    assert g.count(gi.cycle(4)) == int(A4 - 2 * (d * d).sum() + d.sum())


@pytest.mark.parametrize("seed", range(4))
def test_labelled_triangle_trace(seed):
    n, src, dst = gi.er_edges(80, 10.0, seed)
    lab = gi.uniform_labels(n, 3, seed)
    g = OracleGraph(n, src, dst, lab)
    A = _adj_matrix(n, src, dst)
    P = [np.diag((lab == c).astype(np.int64)) for c in range(3)]
    for la, lb, lc in [(0, 1, 2), (0, 0, 1), (2, 2, 2), (1, 0, 1)]:
        q = gi.Query(3, [(0, 1), (1, 2), (0, 2)], [la, lb, lc])
        assert g.count(q) == int(np.trace(P[la] @ A @ P[lb] @ A @ P[lc] @ A))


def test_figure1_example():
    n, src, dst, lab, q, exp = load_fig1()
    g = OracleGraph(n, src, dst, lab)
    off, adj = g.csr()
    assert g.count(q) == exp["count"] == 112                       # line 149
    rows = {tuple(int(x) for x in r) for r in g.enumerate(q)}
    assert tuple(exp["match"]) in rows                              # line 149
    v, dv = exp["degree"]
    assert off[v + 1] - off[v] == dv                                # line 304
    a, b = exp["degree_less"]
    assert off[a + 1] - off[a] < off[b + 1] - off[b]                # line 384
    for (m1, m2), feas in exp["feasible"]:                          # lines 197, 281
        # feasible u3 candidates given (u1,u2) = (m1,m2): matches of the prefix triangle
        tri = gi.Query(3, [(0, 1), (1, 2), (0, 2)], q.labels[:3].tolist())
        got = sorted(int(r[2]) for r in g.enumerate(tri) if r[0] == m1 and r[1] == m2)
        assert got == feas


@pytest.mark.parametrize("seed", range(8))
def test_isomorphism_invariance_and_fixed_roots(seed):
    n, src, dst = gi.er_edges(50, 7.0, seed)
    lab = gi.uniform_labels(n, 2, seed)
    q = small_random_query(seed, 4, 2)
    g = OracleGraph(n, src, dst, lab)
    total = g.count(q)
    perm = np.random.default_rng(seed).permutation(n).astype(np.uint32)
    lab2 = np.empty_like(lab)
    lab2[perm] = lab
    g2 = OracleGraph(n, perm[src], perm[dst], lab2)
    assert g2.count(q) == total
    for u in range(q.n):
        assert sum(g.count(q, fixed=(u, v)) for v in range(n)) == total


def test_query_equals_data_counts_automorphisms():
    # P3 (path on 3 vertices) has 2 automorphisms; the 5-cycle has 10.
    g = OracleGraph(*gi.path_graph(3))
    assert g.count(gi.path(3)) == 2
    g = OracleGraph(*gi.cycle_graph(5))
    assert g.count(gi.cycle(5)) == 10


@pytest.mark.parametrize("seed", range(10))
def test_filters_sound_and_nested(seed):
    n, src, dst = gi.er_edges(60, 6.0, seed)
    lab = gi.uniform_labels(n, 3, seed)
    g = OracleGraph(n, src, dst, lab)
    q = small_random_query(seed, 4, 3)
    ldf = g.filter(q, "ldf", 3)
    nlf = g.filter(q, "nlf", 3)
    assert np.all(nlf <= ldf)
    for row in g.enumerate(q):
        for u in range(q.n):
            assert nlf[u, row[u]] == 1      # soundness: embedded images always pass


def test_filter_hand_example():
    # Data: path a(0)-b(1)-c(0) plus vertex d(0) adjacent to b and e(0).  Query: u0(0)-u1(1)-u2(0).
    # Hand-derived: d(u1)=2 with two label-0 neighbours.  b has neighbours a,c,d (label 0) -> passes.
    # Vertex e has label 0, degree 1: LDF needs d>=1 for u0 -> passes LDF; NLF needs one
    # label-1 neighbour, e's only neighbour is d (label 0) -> fails NLF.
    src = np.array([0, 1, 1, 3], np.uint32)
    dst = np.array([1, 2, 3, 4], np.uint32)
    lab = np.array([0, 1, 0, 0, 0], np.uint32)
    g = OracleGraph(5, src, dst, lab)
    q = gi.Query(3, [(0, 1), (1, 2)], [0, 1, 0])
    ldf, nlf = g.filter(q, "ldf", 2), g.filter(q, "nlf", 2)
    assert ldf[0].tolist() == [1, 0, 1, 1, 1]
    assert nlf[0].tolist() == [1, 0, 1, 1, 0]
    assert ldf[1].tolist() == [0, 1, 0, 0, 0] == nlf[1].tolist()


def test_node_budget_only_discards():
    n, src, dst = gi.er_edges(60, 8.0, 1)
    g = OracleGraph(n, src, dst)
    full = g.count(gi.path(4))
    assert g.count(gi.path(4), max_nodes=10 ** 9) == full
    assert g.count(gi.path(4), max_nodes=5) is None
