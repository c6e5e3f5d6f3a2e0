"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Counts must be bit-exact; enumerations must equal the oracle's sorted embedding set;
CSR and candidate bitmaps must be bit-exact against definitions computed by the oracle.
Inputs are the seeded generators of gminputs (shared by both sides).
"""
import math

import numpy as np
import pytest

import gminputs as gi
from conftest import load_fig1
from oracle import OracleGraph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_10601_b200 as gm
    return gm


def sorted_rows(a):
    a = np.asarray(a, dtype=np.uint32)
    if len(a) == 0:
        return a.reshape(0, a.shape[1] if a.ndim == 2 else 0)
    return a[np.lexsort(a.T[::-1])]


def small_random_query(seed, k, nl):
    rs = np.random.default_rng(seed + 991)
    edges = {(int(rs.integers(0, v)), v) for v in range(1, k)}
    for a in range(k):
        for b in range(a + 1, k):
            if rs.random() < 0.3:
                edges.add((a, b))
    return gi.Query(k, sorted(edges), rs.integers(0, nl, k).tolist())


# ------------------------------------------------------------------ graph build

@pytest.mark.parametrize("seed,nl", [(0, 1), (1, 3), (2, 8)])
def test_csr_matches_oracle(gm, seed, nl):
    n, s, d = gi.rmat_edges(10, 8, seed)
    lab = gi.uniform_labels(n, nl, seed)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    offs, nbr, glab = g.export()
    off_o, adj_o = OracleGraph(n, s, d, lab).csr()
    assert np.array_equal(glab, lab)
    assert g.info()["num_adj"] == len(adj_o)
    assert g.info()["d_max"] == int(np.diff(off_o).max())
    for v in range(n):
        row = adj_o[off_o[v]:off_o[v + 1]]
        # label-partitioned: rows v*nl + l are the label-l neighbours of v, ascending
        for l in range(nl):
            mine = nbr[offs[v * nl + l]:offs[v * nl + l + 1]]
            assert np.array_equal(mine, row[lab[row] == l])


def test_csr_edge_cases(gm):
    # self loops, duplicates, isolated vertices, empty graph
    g = gm.gm_load_graph(5, np.array([0, 0, 1, 3, 1], np.uint32), np.array([0, 1, 0, 3, 2], np.uint32))
    offs, nbr, _ = g.export()
    assert offs.tolist() == [0, 1, 3, 4, 4, 4] and nbr.tolist() == [1, 0, 2, 1]
    g0 = gm.gm_load_graph(4, np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert g0.info()["num_adj"] == 0
    with pytest.raises(gm.GMError):
        gm.gm_load_graph(3, np.array([0], np.uint32), np.array([5], np.uint32))
    with pytest.raises(gm.GMError):
        gm.gm_load_graph(3, np.array([0], np.uint32), np.array([1], np.uint32), np.array([0, 1, 7], np.uint32), 2)


def test_gpu_generator_matches_numpy(gm):
    import gminputs.gpu as gg
    n, s, d = gi.rmat_edges(12, 4, seed=9)
    n2, s2, d2 = gg.rmat_edges(12, 4, seed=9)
    assert n == n2
    assert np.array_equal(s, s2.cpu().numpy().view(np.uint32)) and np.array_equal(d, d2.cpu().numpy().view(np.uint32))
    n, s, d = gi.er_edges(3000, 6, seed=4)
    _, s2, d2 = gg.er_edges(3000, 6, seed=4)
    assert np.array_equal(s, s2.cpu().numpy().view(np.uint32)) and np.array_equal(d, d2.cpu().numpy().view(np.uint32))
    assert np.array_equal(gi.uniform_labels(5000, 7, 3), gg.uniform_labels(5000, 7, 3).cpu().numpy().view(np.uint32))


def test_device_resident_load_equals_host_load(gm):
    import gminputs.gpu as gg
    n, s, d = gg.rmat_edges(11, 8, seed=3)
    lab = gg.uniform_labels(n, 4, 3)
    g1 = gm.gm_load_graph(n, s, d, lab, 4)
    g2 = gm.gm_load_graph(n, s.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32),
                          lab.cpu().numpy().view(np.uint32), 4)
    for a, b in zip(g1.export(), g2.export()):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ filter

@pytest.mark.parametrize("seed", range(4))
def test_filter_bitmaps_match_oracle(gm, seed):
    n, s, d = gi.er_edges(700, 7, seed)
    nl = 3
    lab = gi.uniform_labels(n, nl, seed)
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    q = small_random_query(seed, 6, nl)
    for kind in ("ldf", "nlf"):
        ref = og.filter(q, kind, nl)
        p = gm.gm_plan_query(g, q, filter=kind)
        for u in range(q.n):
            assert np.array_equal(p.candidates(u), ref[u].astype(bool)), (kind, u)
        assert p.info()["cand_count"] == [int(x) for x in ref.sum(1)]
    p = gm.gm_plan_query(g, q, filter="none")
    for u in range(q.n):
        assert np.array_equal(p.candidates(u), lab == q.labels[u])


def test_plan_order_is_connected_and_user_order_validated(gm):
    n, s, d = gi.er_edges(200, 6, 1)
    g = gm.gm_load_graph(n, s, d)
    q = gi.Query(4, [(0, 1), (1, 2), (2, 3)], [0, 0, 0, 0])
    info = gm.gm_plan_query(g, q).info()
    order = info["order"]
    assert sorted(order) == [0, 1, 2, 3]
    for i in range(1, 4):
        assert info["backward"][i] != 0
    with pytest.raises(gm.GMError):
        gm.gm_plan_query(g, q, order=[0, 2, 1, 3])      # 2 has no earlier neighbour
    with pytest.raises(gm.GMError):
        gm.gm_plan_query(g, gi.Query(4, [(0, 1), (2, 3)], [0] * 4))   # disconnected query


# ------------------------------------------------------------------ counts and enumeration

def run_both(gm, n, s, d, lab, nl, q, **kw):
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    p = gm.gm_plan_query(g, q, filter=kw.pop("filter", "nlf"), order=kw.pop("order", None))
    c, st = gm.gm_count(p, **kw)
    return og.count(q), c, st, og, g, p


@pytest.mark.parametrize("seed", range(40))
def test_count_random_small(gm, seed):
    nl = [1, 2, 4][seed % 3]
    if seed % 2:
        n, s, d = gi.er_edges(300 + 20 * seed, 6 + seed % 5, seed)
    else:
        n, s, d = gi.rmat_edges(9, 6, seed)
    lab = gi.uniform_labels(n, nl, seed)
    k = 3 + seed % 4
    q = small_random_query(seed, k, nl)
    tau = [1, 64, 1000000][seed % 3]
    ref, c, st, og, g, p = run_both(gm, n, s, d, lab, nl, q, tau=tau, steal=bool(seed % 4 != 1))
    assert c == ref, (q.edges.tolist(), q.labels.tolist(), st)
    c2, _ = gm.gm_count(p, tau=tau, set_count=False)      # every last-level task validated
    assert c2 == ref
    c3, st3 = gm.gm_count(p, tau=tau, count_words=True)   # the word-counting kernel instantiation
    assert c3 == ref
    c4, _ = gm.gm_count(p, tau=tau, gen_cache=False)       # GenerateTask without the cached part
    assert c4 == ref
    assert st["words"] == 0 and (st3["words"] > 0 or st3["dfs_launches"] == 0)


@pytest.mark.parametrize("seed", range(16))
def test_set_count_trees_same_labels(gm, seed):
    """Trees (last vertex has one backward neighbour) with few labels, so mapped vertices of the
    last label often lie in the counted slice -- adjacent or not to the backward neighbour."""
    n, s, d = gi.rmat_edges(8, 6, seed)
    lab = gi.uniform_labels(n, 2, seed)
    rs = np.random.default_rng(seed)
    k = 4 + seed % 3
    q = gi.Query(k, [(int(rs.integers(0, v)), v) for v in range(1, k)], rs.integers(0, 2, k).tolist())
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, 2)
    p = gm.gm_plan_query(g, q)
    ref = og.count(q)
    for tau in (1, 10 ** 6):
        assert gm.gm_count(p, tau=tau)[0] == ref
        assert gm.gm_count(p, tau=tau, set_count=False)[0] == ref


@pytest.mark.parametrize("seed", range(24))
def test_pair_count_two_leaves(gm, seed):
    """Pair counting: queries whose last two order positions are leaves with one backward
    neighbour each (same or different parents, same or different labels), on power-law graphs
    with few labels, with the hub index forced on (intersection through bitmaps), default, and
    off (binary search); with and without symmetry breaking; against the oracle and against
    the one-level (set_count) and task-per-candidate paths."""
    nl = [1, 2, 3][seed % 3]
    n, s, d = gi.rmat_edges(8 + seed % 2, 8, seed)
    lab = gi.uniform_labels(n, nl, seed)
    rs = np.random.default_rng(seed + 7)
    k = 4 + seed % 3
    core = [(int(rs.integers(0, v)), v) for v in range(1, k - 2)]          # a tree on 0..k-3
    extra = [(a, b) for a in range(k - 2) for b in range(a + 1, k - 2) if rs.random() < 0.3]
    p6 = int(rs.integers(0, k - 2))
    p7 = p6 if seed % 4 == 0 else int(rs.integers(0, k - 2))
    edges = sorted(set(core + extra + [(p6, k - 2), (p7, k - 1)]))
    labels = rs.integers(0, nl, k).tolist()
    if seed % 2:
        labels[k - 1] = labels[k - 2]              # same-label leaves: the intersection term
    q = gi.Query(k, edges, labels)
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    ref = og.count(q)
    order = list(range(k))                         # the two leaves last
    for budget, mindeg, summ in ((64 << 20, 2, 0), (64 << 20, 2, 1), (64 << 20, 64, -1), (0, 64, -1)):
        g.build_hubs(budget, mindeg, summ)
        p = gm.gm_plan_query(g, q, order=order)
        for tau in (1, 10 ** 6):
            assert gm.gm_count(p, tau=tau)[0] == ref
            assert gm.gm_count(p, tau=tau, symmetry=False)[0] == ref
        assert gm.gm_count(p, pair_count=False, symmetry=False)[0] == ref
        assert gm.gm_count(p, set_count=False, symmetry=False)[0] == ref


@pytest.mark.parametrize("seed", range(12))
def test_enumerate_random_small(gm, seed):
    nl = [1, 2, 3][seed % 3]
    n, s, d = gi.er_edges(150, 6, seed)
    lab = gi.uniform_labels(n, nl, seed)
    q = small_random_query(seed, 3 + seed % 3, nl)
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    p = gm.gm_plan_query(g, q)
    ref = og.enumerate(q)
    rows, total, _ = gm.gm_enumerate(p, capacity=len(ref) + 5, tau=[1, 32, 10 ** 6][seed % 3])
    assert total == len(ref)
    assert np.array_equal(sorted_rows(rows), ref)


def test_figure1_example(gm):
    n, s, d, lab, q, exp = load_fig1()
    g = gm.gm_load_graph(n, s, d, lab, 4)
    for tau in (1, 4, 10 ** 6):
        p = gm.gm_plan_query(g, q)
        c, _ = gm.gm_count(p, tau=tau)
        assert c == 112
        rows, total, _ = gm.gm_enumerate(p, capacity=200, tau=tau)
        assert total == 112 and tuple(exp["match"]) in {tuple(int(x) for x in r) for r in rows}
    # the paper's order phi = (u1,u2,u3,u4) (line 197)
    p = gm.gm_plan_query(g, q, order=[0, 1, 2, 3])
    assert gm.gm_count(p, tau=1)[0] == 112


@pytest.mark.parametrize("n,k", [(6, 3), (8, 4), (9, 5), (10, 6), (12, 3)])
def test_clique_closed_form(gm, n, k):
    nn, s, d = gi.complete_graph(n)
    g = gm.gm_load_graph(nn, s, d)
    for tau in (1, 10 ** 6):
        c, _ = gm.gm_count(gm.gm_plan_query(g, gi.clique(k)), tau=tau)
        assert c == math.factorial(n) // math.factorial(n - k)


def test_cycle_and_path_closed_forms(gm):
    n = 40
    g = gm.gm_load_graph(*gi.cycle_graph(n))
    assert gm.gm_count(gm.gm_plan_query(g, gi.cycle(n // 2)))[0] == 0
    for k in (2, 5, 17, 32):                       # 32 = GM_MAX_QUERY
        assert gm.gm_count(gm.gm_plan_query(g, gi.path(k)), tau=1)[0] == 2 * n
    g = gm.gm_load_graph(*gi.cycle_graph(32))
    assert gm.gm_count(gm.gm_plan_query(g, gi.cycle(32)), tau=1)[0] == 64


def test_star_closed_form_with_hub(gm):
    # star with a 5000-leaf hub: d_max >> 32, one root -> relies on batching + stealing
    n, s, d = gi.star_graph(5000)
    g = gm.gm_load_graph(n, s, d)
    for steal in (True, False):
        c, st = gm.gm_count(gm.gm_plan_query(g, gi.star(2)), tau=1, steal=steal)
        assert c == 5000 * 4999 + 0
    c, _ = gm.gm_count(gm.gm_plan_query(g, gi.path(3)), tau=1)
    assert c == 5000 * 4999


def test_edge_cases(gm):
    n, s, d = gi.er_edges(100, 4, 2)
    lab = gi.uniform_labels(n, 2, 2)
    g = gm.gm_load_graph(n, s, d, lab, 2)
    og = OracleGraph(n, s, d, lab)
    # single-vertex query: every vertex with the label
    q1 = gi.Query(1, [], [1])
    assert gm.gm_count(gm.gm_plan_query(g, q1))[0] == int((lab == 1).sum())
    rows, total, _ = gm.gm_enumerate(gm.gm_plan_query(g, q1), capacity=1000)
    assert sorted(rows[:, 0].tolist()) == np.flatnonzero(lab == 1).tolist()
    # label absent from G
    q = gi.Query(3, [(0, 1), (1, 2)], [0, 5, 0])
    assert gm.gm_count(gm.gm_plan_query(g, q))[0] == 0
    # single edge query
    q2 = gi.Query(2, [(0, 1)], [0, 1])
    assert gm.gm_count(gm.gm_plan_query(g, q2))[0] == og.count(q2)
    # query larger than any component
    gsmall = gm.gm_load_graph(*gi.path_graph(4))
    assert gm.gm_count(gm.gm_plan_query(gsmall, gi.path(5)))[0] == 0
    # empty graph
    g0 = gm.gm_load_graph(10, np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert gm.gm_count(gm.gm_plan_query(g0, gi.triangle()))[0] == 0


def test_enumerate_capacity_overflow(gm):
    g = gm.gm_load_graph(*gi.complete_graph(7))
    p = gm.gm_plan_query(g, gi.clique(4))
    rows, total, _ = gm.gm_enumerate(p, capacity=100, tau=1)
    assert total == 840 and len(rows) == 100
    rows = rows.astype(np.int64)
    assert all(len(set(r)) == 4 for r in rows.tolist())


@pytest.mark.parametrize("world", [2, 3])
def test_rank_partition_sums_to_total(gm, world):
    n, s, d = gi.rmat_edges(11, 8, 5)
    lab = gi.uniform_labels(n, 2, 5)
    q = gi.tailed_triangle((0, 1, 0, 1))
    g = gm.gm_load_graph(n, s, d, lab, 2)
    p = gm.gm_plan_query(g, q)
    total = gm.gm_count(p)[0]
    parts = [gm.gm_count(p, rank=r, world=world, root_chunk=16, tau=128)[0] for r in range(world)]
    assert sum(parts) == total == OracleGraph(n, s, d, lab).count(q)


def test_user_roots_match_oracle_fixed_root(gm):
    n, s, d = gi.rmat_edges(12, 8, 7)
    q = gi.clique(4)
    g = gm.gm_load_graph(n, s, d)
    og = OracleGraph(n, s, d)
    p = gm.gm_plan_query(g, q)
    u0 = p.info()["order"][0]
    rs = np.random.default_rng(0)
    roots = rs.choice(n, 30, replace=False).astype(np.uint32)
    c, _ = gm.gm_count(p, roots=roots, tau=1)
    assert c == sum(og.count(q, fixed=(u0, int(v))) for v in roots)


def test_count_to_device_tensor(gm):
    import torch
    g = gm.gm_load_graph(*gi.complete_graph(6))
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    gm.gm_count(gm.gm_plan_query(g, gi.clique(3)), out=out)
    assert int(out.item()) == 120


def test_time_limit_reports_timeout(gm):
    n, s, d = gi.rmat_edges(14, 16, 1)
    g = gm.gm_load_graph(n, s, d)
    p = gm.gm_plan_query(g, gi.path(8))
    c, st = gm.gm_count(p, time_limit_ms=5, tau=1000)
    assert st["timed_out"] == 1


# ------------------------------------------------------------------ BASELINE configs (sampled)

def test_config1_full(gm):
    """configs[0]: ER(1000, avg deg 8, 4 labels), tailed triangle -- full enumeration parity."""
    n, s, d = gi.er_edges(1000, 8, 11)
    lab = gi.uniform_labels(n, 4, 11)
    q = gi.tailed_triangle((0, 1, 2, 3))
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, 4)
    p = gm.gm_plan_query(g, q)
    ref = og.enumerate(q)
    rows, total, _ = gm.gm_enumerate(p, capacity=len(ref) + 1)
    assert total == len(ref) and np.array_equal(sorted_rows(rows), ref)


def _device_graph(cfg):
    import bench
    n, s, d, lab = bench.make_graph_device(cfg)
    return n, s, d, lab


def test_config3_sampled_roots(gm):
    """configs[2]: R-MAT scale 22 unlabelled (64M sampled edges), triangle / 4-clique / 5-cycle in
    the bench configuration: per-root counts on sampled roots equal the oracle's; the full
    triangle count with symmetry breaking equals the full search without it."""
    import bench
    cfg = bench.CONFIGS["rmat22"]
    n, s, d, lab = _device_graph(cfg)
    sh, dh = s.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32)
    g = gm.gm_load_graph(n, s, d, lab, 1)
    og = OracleGraph(n, sh, dh)
    rs = np.random.default_rng(3)
    checked = nonzero = 0
    for q in (gi.triangle(), gi.clique(4), gi.cycle(5)):
        p = gm.gm_plan_query(g, q)
        u0 = p.info()["order"][0]
        roots, ref = [], 0
        for v in rs.choice(n, 400, replace=False):
            c = og.count(q, fixed=(u0, int(v)), max_nodes=4_000_000)
            if c is not None:
                roots.append(int(v)); ref += c; nonzero += c > 0
            if len(roots) == 12:
                break
        assert gm.gm_count(p, roots=np.array(roots, np.uint32))[0] == ref
        checked += len(roots)
    assert checked >= 24 and nonzero >= 6
    p = gm.gm_plan_query(g, gi.triangle())
    c_sb, st = gm.gm_count(p)
    assert st["automorphisms"] == 6 and st["timed_out"] == 0
    assert c_sb == gm.gm_count(p, symmetry=False)[0]


def test_config4_enumerated_rows_valid(gm):
    """configs[3]: R-MAT scale 24, 16 labels, the bench's 16-vertex dense queries: rows listed by
    gm_enumerate (time-limited) are distinct embeddings -- labels, injectivity, and every query
    edge checked against the device edge list by an independent scan (gminputs.gpu)."""
    import bench
    import gminputs.gpu as gg
    cfg = bench.CONFIGS["rmat24"]
    n, s, d, lab = _device_graph(cfg)
    lh = lab.cpu().numpy().view(np.uint32)
    adj = gg.DeviceNeighbors(n, s, d)
    queries = bench.build_queries(cfg, adj, lh)[:2]
    g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
    for q in queries:
        p = gm.gm_plan_query(g, q)
        rows, total, st = gm.gm_enumerate(p, capacity=256, time_limit_ms=500)
        assert len(rows) == min(256, total) and len(rows) > 0
        assert len({tuple(r) for r in rows.tolist()}) == len(rows)
        for r in rows[:6].astype(np.int64):
            assert len(set(r.tolist())) == q.n and np.array_equal(lh[r], q.labels)
            for a, b in q.edges.tolist():
                nb = adj.neighbors(int(r[a]))
                i = np.searchsorted(nb, r[b])
                assert i < len(nb) and nb[i] == r[b]


def test_config2_sampled_roots(gm):
    """configs[1]: R-MAT scale 18 (16 edges/vertex), 8 labels, 8-vertex queries (§6.1 generator):
    GPU count restricted to sampled roots == sum of the oracle's per-root counts.  Roots are
    sampled among phi[0]'s candidates whose oracle count stays under a budget (the oracle
    must finish); the GPU runs in the bench launch configuration (tau = 1e6, stealing on)."""
    import bench
    cfg = bench.CONFIGS["rmat18"]
    n, s, d, lab = bench.make_graph_host(cfg)
    off, nb = gi.simple_adjacency(n, s, d)
    queries = bench.build_queries(cfg, gi.HostAdjacency(off, nb), lab)          # the bench's query set
    g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
    og = OracleGraph(n, s, d, lab)
    rs = np.random.default_rng(1)
    budget = 2_000_000          # oracle work units (tree nodes + candidates examined) per sampled root
    checked, nonzero = 0, 0
    for q in queries:
        p = gm.gm_plan_query(g, q)
        u0 = p.info()["order"][0]
        cands = np.flatnonzero(p.candidates(u0))
        roots, ref = [], 0
        for v in rs.permutation(cands)[:300]:
            c = og.count(q, fixed=(u0, int(v)), max_nodes=budget)
            if c is not None:
                roots.append(int(v)); ref += c
                nonzero += c > 0
            if len(roots) == 6:
                break
        c, st = gm.gm_count(p, roots=np.array(roots, np.uint32), time_limit_ms=60000)
        assert st["timed_out"] == 0
        assert c == ref, (q, roots)
        checked += len(roots)
        # the 5-vertex prefix of the planner's order (an induced, connected sub-query) has
        # per-root counts the oracle finishes: exact parity on sampled roots
        order = p.info()["order"][:5]
        idx = {u: i for i, u in enumerate(order)}
        sub = gi.Query(5, [(idx[a], idx[b]) for a, b in q.edges.tolist() if a in idx and b in idx],
                       [int(q.labels[u]) for u in order])
        ps = gm.gm_plan_query(g, sub)
        s0 = ps.info()["order"][0]
        sroots, sref = [], 0
        for v in rs.permutation(np.flatnonzero(ps.candidates(s0)))[:100]:
            cc = og.count(sub, fixed=(s0, int(v)), max_nodes=20_000_000)
            if cc is not None:
                sroots.append(int(v)); sref += cc
                nonzero += cc > 0
            if len(sroots) == 6:
                break
        assert gm.gm_count(ps, roots=np.array(sroots, np.uint32))[0] == sref
        checked += len(sroots)
    assert checked >= 24 and nonzero >= 8
    # an explicit empty root list means no roots at all
    p = gm.gm_plan_query(g, queries[0])
    assert gm.gm_count(p, roots=np.zeros(0, np.uint32))[0] == 0
    # full queries at full size through gm_enumerate: every listed row is a distinct embedding
    off_o, adj_o = og.csr()
    for q in queries:
        p = gm.gm_plan_query(g, q)
        rows, total, st = gm.gm_enumerate(p, capacity=4096, time_limit_ms=300)
        assert len(rows) == min(4096, total) and len(rows) > 0
        assert len({tuple(r) for r in rows.tolist()}) == len(rows)
        for r in rows[:512].astype(np.int64):
            assert len(set(r.tolist())) == q.n                              # injective
            assert np.array_equal(lab[r], q.labels)                         # labels
            for a, b in q.edges.tolist():                                   # edges
                nb_a = adj_o[off_o[r[a]]:off_o[r[a] + 1]]
                i = np.searchsorted(nb_a, r[b])
                assert i < len(nb_a) and nb_a[i] == r[b]


@pytest.mark.parametrize("seed", range(6))
def test_hub_index_does_not_change_results(gm, seed):
    """Counts with the hub bitmap index (all vertices of degree >= 2 as hubs), with the default
    index and with no index all equal the oracle."""
    nl = [2, 3, 4][seed % 3]
    n, s, d = gi.rmat_edges(8, 6, seed)
    lab = gi.uniform_labels(n, nl, seed)
    q = small_random_query(seed + 50, 4, nl)
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    ref = og.count(q)
    assert g.info()["hubs"] > 0
    for budget, mindeg, summ in ((64 << 20, 2, 0), (64 << 20, 2, 1), (0, 64, -1), (64 << 20, 64, -1)):
        g.build_hubs(budget, mindeg, summ)
        assert (g.info()["hub_summary_words"] > 0) == (summ == 1 and budget > 0)
        if budget == 0:
            assert g.info()["hubs"] == 0
        p = gm.gm_plan_query(g, q)
        assert gm.gm_count(p, tau=[1, 1000][seed % 2])[0] == ref
        assert gm.gm_count(p, tau=1, set_count=False)[0] == ref
        rows, total, _ = gm.gm_enumerate(p, capacity=min(ref, 20000) + 1)
        assert total == ref


def test_symmetry_breaking_at_scale(gm):
    """R-MAT scale 16 (65k vertices, 1M edges): symmetric patterns counted with symmetry
    breaking + id-range slice cuts equal the full search (different code path, same library)
    and, on sampled roots, the oracle (test_symmetry_breaking_counts pins the small cases)."""
    n, s, d = gi.rmat_edges(16, 16, 21)
    g = gm.gm_load_graph(n, s, d)
    for q in (gi.triangle(), gi.clique(4), gi.cycle(4)):
        p = gm.gm_plan_query(g, q)
        c_sb, st = gm.gm_count(p)
        c_full, st2 = gm.gm_count(p, symmetry=False)
        assert st["automorphisms"] > 1 and st2["automorphisms"] == 1
        assert c_sb == c_full and c_sb > 0


def _aut_brute(q):
    """|Aut(Q)|: label- and edge-preserving permutations, by brute force."""
    import itertools
    E = {(int(a), int(b)) for a, b in q.edges} | {(int(b), int(a)) for a, b in q.edges}
    return sum(1 for pm in itertools.permutations(range(q.n))
               if all(q.labels[pm[u]] == q.labels[u] for u in range(q.n))
               and all((pm[a], pm[b]) in E for a, b in E))


SYM_QUERIES = [gi.path(2), gi.triangle(), gi.clique(4), gi.clique(5), gi.cycle(4), gi.cycle(5), gi.cycle(6), gi.star(3),
               gi.path(4), gi.Query(3, [(0, 1), (1, 2), (0, 2)], [0, 0, 1]),
               gi.Query(4, [(0, 1), (1, 2), (2, 3), (3, 0)], [0, 1, 0, 1]),
               gi.Query(5, [(0, 1), (0, 2), (0, 3), (0, 4), (1, 2)], [0, 1, 1, 2, 2])]


@pytest.mark.parametrize("qi", range(len(SYM_QUERIES)))
def test_symmetry_breaking_counts(gm, qi):
    """gm_count with symmetry breaking (one embedding per Aut(Q)-orbit, times |Aut(Q)|, as in
    Appendix A) equals the oracle and the unbroken search; |Aut(Q)| equals brute force."""
    q = SYM_QUERIES[qi]
    nl = int(q.labels.max()) + 1
    for seed in range(3):
        n, s, d = (gi.rmat_edges(7, 6, seed) if seed % 2 == 0 else gi.er_edges(150, 9, seed))
        lab = gi.uniform_labels(n, nl, seed)
        og = OracleGraph(n, s, d, lab)
        g = gm.gm_load_graph(n, s, d, lab, nl)
        p = gm.gm_plan_query(g, q)
        info = p.info()
        assert info["automorphisms"] == _aut_brute(q)
        ref = og.count(q)
        for tau in (1, 10 ** 6):
            c, st = gm.gm_count(p, tau=tau)
            # symmetry breaking is used unless it would disable last-level set counting
            assert c == ref and st["automorphisms"] in (1, info["automorphisms"])
            assert gm.gm_count(p, tau=tau, symmetry=False)[0] == ref
            assert gm.gm_count(p, tau=tau, set_count=False)[0] == ref


def test_config5_local_parity(gm):
    """configs[4]: Friendster-shaped R-MAT scale 26 (2.1 G adjacency entries, 16 labels) with the
    bench's 24/32-vertex dense queries.  (a) Exact parity at full size: for the sub-query induced
    by a query vertex c and up to 4 of its Q-neighbours, every embedding with M[c] = v lies in
    the closed neighbourhood N[v]; the oracle counts it on that local graph (edges gathered by
    an independent scan of the device edge list) and the GPU counts it on the whole graph with
    root v.  (b) Rows listed by gm_enumerate for the full queries are distinct embeddings."""
    import bench
    import gminputs.gpu as gg
    cfg = bench.CONFIGS["rmat26"]
    n, s, d, lab = _device_graph(cfg)
    lh = lab.cpu().numpy().view(np.uint32)
    adj = gg.DeviceNeighbors(n, s, d)
    queries = bench.build_queries(cfg, adj, lh)
    queries = [queries[0], queries[2]]                       # one 24- and one 32-vertex query
    g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
    rs = np.random.default_rng(26)
    checked = nonzero = 0
    for q in queries:
        qe = q.edges.tolist()
        qn = {u: sorted({b for a, b in qe if a == u} | {a for a, b in qe if b == u}) for u in range(q.n)}
        c = max(range(q.n), key=lambda u: (len(qn[u]), -u))
        for k in (2, 4):
            keep = [c] + qn[c][:k]
            idx = {u: i for i, u in enumerate(keep)}
            sub = gi.Query(len(keep), [(idx[a], idx[b]) for a, b in qe if a in idx and b in idx],
                           [int(q.labels[u]) for u in keep])
            ps = gm.gm_plan_query(g, sub, order=list(range(len(keep))))
            cands = np.flatnonzero(ps.candidates(0))
            roots, ref = [], 0
            for v in rs.permutation(cands)[:200]:
                nv = adj.neighbors(int(v))
                if not 2 <= len(nv) <= 160:
                    continue
                ball = [int(v)] + nv.tolist()
                loc = {w: i for i, w in enumerate(ball)}
                es = np.array([(loc[a], loc[b]) for a, b in adj.induced_edges(ball).tolist()], np.uint32).reshape(-1, 2)
                og = OracleGraph(len(ball), es[:, 0].copy(), es[:, 1].copy(), lh[np.array(ball, np.int64)])
                cnt = og.count(sub, fixed=(0, 0))
                roots.append(int(v)); ref += cnt; nonzero += cnt > 0
                assert gm.gm_count(ps, roots=np.array([v], np.uint32))[0] == cnt, (q.name, k, int(v))
                if len(roots) == 4:
                    break
            assert gm.gm_count(ps, roots=np.array(roots, np.uint32))[0] == ref
            checked += len(roots)
        p = gm.gm_plan_query(g, q)
        rows, total, st = gm.gm_enumerate(p, capacity=128, time_limit_ms=500)
        assert len(rows) == min(128, total) and len(rows) > 0
        assert len({tuple(r) for r in rows.tolist()}) == len(rows)
        for r in rows[:4].astype(np.int64):
            assert len(set(r.tolist())) == q.n and np.array_equal(lh[r], q.labels)
            for a, b in qe:
                nb = adj.neighbors(int(r[a]))
                i = np.searchsorted(nb, r[b])
                assert i < len(nb) and nb[i] == r[b]
    assert checked >= 12 and nonzero >= 3


@pytest.mark.parametrize("seed", range(4))
def test_pool_depth_sweep_counting_paths(gm, seed):
    """tau sweeps the depth of the initial pool (Alg. 2 line 1, §4.3) across every level, so the
    DFS starts at, below and above the pair-counting (last-2) and set-counting (last-1)
    levels, with and without stealing; every count equals the oracle's."""
    nl = 2
    n, s, d = gi.rmat_edges(9, 8, 40 + seed)
    lab = gi.uniform_labels(n, nl, 40 + seed)
    rs = np.random.default_rng(60 + seed)
    k = 5 + seed % 2
    # a tree on 0..k-3 plus two non-adjacent leaves last (pair counting applies in the given order)
    edges = [(int(rs.integers(0, v)), v) for v in range(1, k - 2)]
    edges += [(int(rs.integers(0, k - 2)), k - 2), (int(rs.integers(0, k - 2)), k - 1)]
    q = gi.Query(k, sorted(set(edges)), rs.integers(0, nl, k).tolist())
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    ref = og.count(q)
    p = gm.gm_plan_query(g, q, order=list(range(k)))
    depths = set()
    for tau in (1, 4, 16, 64, 256, 1024, 4096, 16384, 65536, 10 ** 6):
        for steal in (True, False):
            c, st = gm.gm_count(p, tau=tau, steal=steal, symmetry=False)
            assert c == ref, (tau, steal, st["pool_depth"])
            depths.add(st["pool_depth"] if st["dfs_launches"] else k)
        assert gm.gm_count(p, tau=tau)[0] == ref
    # the DFS started below the pair-counting level and at the set-counting level (depth k-2)
    assert min(depths) <= k - 3 and (k - 2) in depths, depths


def test_launch_shape_options(gm):
    """warps_per_block 1/2/4 and blocks_per_sm give the oracle's count; more warps per block
    than k_dfs is compiled for (4 for the 8-level kernels, 14 for the deeper ones) is an
    argument error, not a failed launch."""
    n, s, d = gi.rmat_edges(9, 8, 5)
    lab = gi.uniform_labels(n, 2, 5)
    q = small_random_query(5, 5, 2)
    ref, c, st, og, g, p = run_both(gm, n, s, d, lab, 2, q)
    assert c == ref
    for wpb in (1, 2, 4):
        for bps in (0, 1, 3):
            assert gm.gm_count(p, warps_per_block=wpb, blocks_per_sm=bps, tau=16)[0] == ref
    for wpb in (8, 15):
        with pytest.raises(gm.GMError) as e:
            gm.gm_count(p, warps_per_block=wpb, tau=16)
        assert "warps_per_block" in str(e.value)


def test_pair_count_long_lists_closed_form(gm):
    """Pair counting with both leaf lists long (>= 128: the 16-byte-load intersection rounds)
    on R-MAT 13 unlabelled: 4-vertex paths x-a-b-y in the order [a, b, x, y] (the two leaves
    hang off different vertices and share a label, so |A n R| is intersected).  The count is
    pinned by a closed form, not the oracle: ordered walks a-b with x in N(a) \\ {b},
    y in N(b) \\ {a}, x != y number sum over ordered edges of (d_a - 1)(d_b - 1) - t(a, b),
    and sum over ordered edges of t(a, b) = |N(a) n N(b)| is trace(A^3)."""
    import scipy.sparse as sp
    n, s, d = gi.rmat_edges(13, 16, 77)
    off, nb = gi.simple_adjacency(n, s, d)
    deg = np.diff(off).astype(np.int64)
    rows = np.repeat(np.arange(n), deg)
    A = sp.csr_matrix((np.ones(len(nb), np.int64), (rows, nb.astype(np.int64))), shape=(n, n))
    tr3 = int((A @ A).multiply(A).sum())
    want = int(((deg[rows] - 1) * (deg[nb] - 1)).sum()) - tr3
    assert deg.max() >= 512                      # hub lists: many 128-element rounds
    g = gm.gm_load_graph(n, s, d)
    q = gi.Query(4, [(0, 1), (1, 2), (2, 3)], [0, 0, 0, 0])
    for budget, mindeg, summ in ((64 << 20, 64, 0), (64 << 20, 64, 1), (0, 64, -1)):   # bitmaps / + summary / search
        g.build_hubs(budget, mindeg, summ)
        p = gm.gm_plan_query(g, q, order=[1, 2, 0, 3])
        for tau in (1, 10 ** 6):
            c, st = gm.gm_count(p, tau=tau, symmetry=False)
            assert st["paths"] & 2, st             # pair counting ran
            assert c == want, (budget, tau, c, want)
        assert gm.gm_count(p, pair_count=False, symmetry=False)[0] == want
        assert gm.gm_count(p)[0] == want


def test_enumerate_stop_at_capacity(gm):
    """GM_FLAG_STOP_AT_CAPACITY: the search stops once the buffer is full; every written row is
    a distinct embedding (a subset of the oracle's set) and the reported count is >= capacity."""
    n, s, d = gi.rmat_edges(10, 8, 31)
    lab = gi.uniform_labels(n, 2, 31)
    q = small_random_query(31, 5, 2)
    og = OracleGraph(n, s, d, lab)
    ref = og.enumerate(q)
    assert len(ref) > 5000
    g = gm.gm_load_graph(n, s, d, lab, 2)
    p = gm.gm_plan_query(g, q)
    refset = {tuple(r) for r in ref.tolist()}
    for tau in (1, 10 ** 6):
        rows, total, st = gm.gm_enumerate(p, capacity=1000, tau=tau, stop_at_capacity=True)
        assert total >= 1000 and len(rows) == 1000
        got = {tuple(r) for r in rows.tolist()}
        assert len(got) == 1000 and got <= refset
    rows, total, st = gm.gm_enumerate(p, capacity=len(ref) + 10, stop_at_capacity=True)
    assert total == len(ref) and st["timed_out"] == 0


# ------------------------------------------------------------------ sibling prefixes

def _sib_queries():
    """Clique-like last levels (GM_PATH_SIBLING applies) and near misses (it must not)."""
    qs = [gi.clique(4), gi.clique(5), gi.clique(6)]
    # K4 plus a pendant vertex on the clique: last level is still clique-like under phi
    qs.append(gi.Query(5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4)], [0] * 5, "k4tail"))
    # diamond (K4 minus an edge): two triangles sharing an edge
    qs.append(gi.Query(4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], [0] * 4, "diamond"))
    # labelled K4: two labels (the last two share one label or not, depending on the order)
    qs.append(gi.Query(4, [(i, j) for i in range(4) for j in range(i + 1, 4)], [0, 0, 1, 1], "k4lab"))
    qs.append(gi.Query(5, [(i, j) for i in range(5) for j in range(i + 1, 5)], [0, 0, 0, 1, 1], "k5lab"))
    return qs


@pytest.mark.parametrize("seed", range(6))
def test_sibling_prefix_counts(gm, seed):
    """Sibling prefixes: counts with and without them equal the oracle's, on
    R-MAT and ER graphs with hubs whose sibling lists overflow the per-parent buffer, with
    the pool starting below the sibling level (tau = 1) or not, stealing on and off."""
    if seed % 2:
        n, s, d = gi.er_edges(100, 36.0, seed)
    else:
        n, s, d = gi.rmat_edges(9, 8, seed)
    nl = 1 if seed < 4 else 2
    lab = gi.uniform_labels(n, nl, seed)
    og = OracleGraph(n, s, d, lab)
    g = gm.gm_load_graph(n, s, d, lab, nl)
    seen = 0
    for q in _sib_queries():
        if nl == 1 and len(set(q.labels.tolist())) > 1:
            continue
        if q.name == "clique6" and nl == 1 and seed % 2 == 0:
            continue                                  # (the oracle needs ~25 s for it there)
        ref = og.count(q)
        p = gm.gm_plan_query(g, q)
        for kw in (dict(tau=1), dict(tau=1, steal=False), dict(tau=64), dict(tau=10 ** 6),
                   dict(tau=1, sibling=False), dict(tau=1, count_words=True), dict(tau=1, sibling=False, gen_cache=False)):
            c, st = gm.gm_count(p, **kw)
            assert c == ref, (q.name, kw, st)
            seen |= st["paths"]
    assert seen & 16, "no query took the sibling-prefix path"


def test_sibling_prefix_closed_forms(gm):
    """K_k in K_n = n!/(n-k)! with sibling prefixes (every sibling list of K_60 is long)."""
    for n, k in ((60, 4), (40, 5), (24, 6), (300, 4)):   # K_300: sibling lists overflow the buffer
        nn, s, d = gi.complete_graph(n)
        g = gm.gm_load_graph(nn, s, d)
        p = gm.gm_plan_query(g, gi.clique(k))
        c, st = gm.gm_count(p, tau=1)
        assert c == math.factorial(n) // math.factorial(n - k)
        assert st["paths"] & 16


@pytest.mark.parametrize("seed", range(4))
def test_generate_cache_counts(gm, seed):
    """Cached GenerateTask part (gen_prep): symmetric unlabelled patterns whose
    hot level has a backward row and symmetry bounds from levels <= l-2 (cycles, a house, a
    bowtie), with and without the cache, against the oracle."""
    n, s, d = gi.rmat_edges(7, 6, seed) if seed % 2 == 0 else gi.er_edges(60, 6.0, seed)
    og = OracleGraph(n, s, d)
    g = gm.gm_load_graph(n, s, d)
    qs = [gi.cycle(5), gi.cycle(6)] + ([gi.cycle(7)] if seed % 2 else []) + [
          gi.Query(5, [(0, 1), (1, 2), (2, 3), (3, 0), (2, 4), (3, 4)], [0] * 5, "house"),
          gi.Query(5, [(0, 1), (1, 2), (0, 2), (2, 3), (3, 4), (2, 4)], [0] * 5, "bowtie")]
    seen = 0
    for q in qs:
        ref = og.count(q)
        p = gm.gm_plan_query(g, q)
        for kw in (dict(tau=1), dict(tau=1, steal=False), dict(tau=64), dict(tau=1, gen_cache=False),
                   dict(tau=1, count_words=True)):
            c, st = gm.gm_count(p, **kw)
            assert c == ref, (q.name, kw, st)
            seen |= st["paths"]
    assert seen & 32, "no query took the cached GenerateTask path"
