"""GPU parity for 9-32-vertex queries: the D=16, D=24 (count) and D=32 instantiations of k_dfs.

The bench's configs 4 and 5 run 16-, 24- and 32-vertex dense queries (BASELINE.json
configs[3..4]; the paper evaluates 8-, 12- and 16-vertex random queries, PAPER.md:883,
and Definition 1, does not get easier with |V(Q)|).  These tests
compare gm_count and gm_enumerate with the oracle on graphs where the oracle finishes in
seconds, for every counting path the library has:

  * dense queries grown by the §6.1 procedure with the dense rule of
    gminputs.grow_query -- many backward neighbours per level, i.e. many adjacency checks
    per task, and (16 labels over 24-32 query vertices) same-label injectivity rows at
    levels >= 16;
  * the same dense cores with one or two pendant leaves, so set counting (one leaf) and
    pair counting (two non-adjacent leaves, same or different labels) run at D=16/32;

each under default options, set_count=False, pair_count=False and symmetry=False, with
tau in {1, 64, 1e6} and stealing on and off.  Small results are also enumerated and the
sorted embedding set compared element by element.
"""
import numpy as np
import pytest

import gminputs as gi
from oracle import OracleGraph

pytestmark = pytest.mark.gpu

GRAPH = dict(scale=12, ef=8, labels=16, seed=7)     # R-MAT 12 (4096 vertices), 16 uniform labels
ENUM_MAX = 200_000                                   # enumerate and compare sets up to this many rows


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_10601_b200 as gm
    n, s, d = gi.rmat_edges(GRAPH["scale"], GRAPH["ef"], GRAPH["seed"])
    lab = gi.uniform_labels(n, GRAPH["labels"], GRAPH["seed"])
    og = OracleGraph(n, s, d, lab)
    adj = gi.HostAdjacency(*gi.simple_adjacency(n, s, d))
    g = gm.gm_load_graph(n, s, d, lab, GRAPH["labels"])
    return dict(gm=gm, n=n, lab=lab, og=og, adj=adj, g=g, ref={})


def with_leaves(core, k_leaves, same, seed):
    """core + k_leaves pendant vertices (leaf i hangs off core vertex a or b).  Leaves are never
    adjacent to each other; `same` gives the two leaves one label (pair counting's
    intersection term)."""
    rs = np.random.default_rng(seed)
    n = core.n
    edges = core.edges.tolist()
    labels = core.labels.tolist()
    a = int(rs.integers(0, n))
    b = a if seed % 2 == 0 else int(rs.integers(0, n))
    la = int(rs.integers(0, GRAPH["labels"]))
    for i, p in enumerate([a, b][:k_leaves]):
        edges.append((p, n + i))
        labels.append(la if (same or i == 0) else int(rs.integers(0, GRAPH["labels"])))
    return gi.Query(n + k_leaves, edges, labels, name=f"{core.name}+{k_leaves}l{'s' if same else ''}")


# (core size, seed, leaves, same-label leaves); every case verified to finish in the oracle in
# a few seconds (R-MAT 12, 16 labels).  Sizes 10..32 cover k_dfs<16> (9-16), k_dfs<24> (17-24, count) and k_dfs<32>
# (25-32; 17-32 when enumerating).
DENSE = [(10, 1), (10, 3), (12, 1), (12, 3), (16, 1), (16, 3), (24, 1), (24, 3), (32, 1), (32, 2), (32, 3)]
LEAVES = [(k, s, nl, same) for k in (10, 14, 22, 30) for s in (1, 3, 4) for nl, same in ((1, False), (2, False), (2, True))
          if not (k == 14 and s == 4 and same)]


def query(env, core_size, seed, leaves=0, same=False):
    core = gi.grow_query(env["adj"], env["lab"], core_size, seed=seed, dense=True, min_avg_degree=3.0)
    return with_leaves(core, leaves, same, seed) if leaves else core


def oracle_count(env, q):
    key = (q.n, tuple(map(tuple, q.edges.tolist())), tuple(q.labels.tolist()))
    if key not in env["ref"]:
        env["ref"][key] = env["og"].count(q)
    return env["ref"][key]


def sorted_rows(a):
    a = np.asarray(a, dtype=np.uint32)
    return a[np.lexsort(a.T[::-1])] if len(a) else a


def check_all_paths(env, q, order=None, expect_paths=0):
    gm = env["gm"]
    ref = oracle_count(env, q)
    assert ref > 0                                  # the query was grown from G: at least the identity
    p = gm.gm_plan_query(env["g"], q, order=order)
    seen = 0
    for tau in (1, 64, 10 ** 6):
        for steal in (True, False):
            c, st = gm.gm_count(p, tau=tau, steal=steal)
            assert c == ref, (q.name, tau, steal, st)
            if st["dfs_launches"]:
                assert st["stack_levels"] == (16 if q.n <= 16 else (24 if q.n <= 24 else 32))
            seen |= st["paths"]
    for kw in (dict(set_count=False), dict(pair_count=False), dict(symmetry=False),
               dict(set_count=False, symmetry=False), dict(count_words=True), dict(gen_cache=False)):
        for tau in (1, 64):
            c, st = gm.gm_count(p, tau=tau, **kw)
            assert c == ref, (q.name, kw, tau, st)
            seen |= st["paths"]
    assert seen & expect_paths == expect_paths, (q.name, seen)
    if ref <= ENUM_MAX:
        want = env["og"].enumerate(q)
        for tau in (1, 10 ** 6):
            rows, total, _ = gm.gm_enumerate(p, capacity=ref + 3, tau=tau)
            assert total == ref
            assert np.array_equal(sorted_rows(rows), want), q.name
    return ref, seen


@pytest.mark.parametrize("k,seed", DENSE)
def test_dense_query_counts_and_sets(env, k, seed):
    """Dense grown queries of 10-32 vertices (many checks per task, same-label injectivity rows
    at high levels) on every counting path, tau and stealing setting."""
    q = query(env, k, seed)
    check_all_paths(env, q)


@pytest.mark.parametrize("k,seed,leaves,same", [(12, 1, 0, False), (14, 3, 1, False), (14, 1, 2, True),
                                                 (22, 1, 2, False), (30, 2, 1, False), (32, 1, 0, False)])
def test_block_shapes_deep_kernels(env, k, seed, leaves, same):
    """The 16/24/32-level kernels are compiled for blocks of up to 14 warps; the default picks
    the block size with the most resident warps for the query's shared memory (stack levels
    the query touches + scratch rows).  Every explicit block size, with stealing and a small
    pool (many warps share few items), gives the oracle's count; 15 warps is an argument error."""
    gm = env["gm"]
    q = query(env, k, seed, leaves, same)
    ref = oracle_count(env, q)
    p = gm.gm_plan_query(env["g"], q)
    c, st = gm.gm_count(p, tau=1)
    assert c == ref and st["dfs_launches"] and st["block"] % 32 == 0 and 32 <= st["block"] <= 14 * 32, st
    for wpb in (1, 3, 5, 7, 14):
        for bps in (0, 1):
            try:
                c, st = gm.gm_count(p, tau=64, warps_per_block=wpb, blocks_per_sm=bps)
            except gm.GMError as e:      # a block of wpb warps larger than 227 KB of shared memory
                assert wpb >= 7 and "no block fits" in str(e), (q.name, wpb, e)
                continue
            assert c == ref, (q.name, wpb, bps, st)
            if st["dfs_launches"]:
                assert st["block"] == 32 * wpb
    with pytest.raises(gm.GMError):
        gm.gm_count(p, warps_per_block=15)


@pytest.mark.parametrize("k,seed,leaves,same", LEAVES)
def test_dense_core_with_leaves(env, k, seed, leaves, same):
    """Dense cores plus one or two pendant leaves, in the planner's order and with the leaves
    placed last (set counting with one leaf, pair counting with two) at D=16/32."""
    from paper_2604_10601_b200 import _lib as L
    q = query(env, k, seed, leaves, same)
    check_all_paths(env, q)
    # leaves last in a connected order of the core (BFS from vertex 0 of the core)
    core_n = q.n - leaves
    adjq = {u: set() for u in range(q.n)}
    for a, b in q.edges.tolist():
        adjq[a].add(b); adjq[b].add(a)
    order, seen = [0], {0}
    i = 0
    while i < len(order):
        for w in sorted(adjq[order[i]]):
            if w < core_n and w not in seen:
                seen.add(w); order.append(w)
        i += 1
    order += list(range(core_n, q.n))
    expect = L.GM_PATH_SET_COUNT | (L.GM_PATH_PAIR_COUNT if leaves == 2 else 0)
    check_all_paths(env, q, order=order, expect_paths=expect)


def test_stealing_happens_at_d16_and_d32(env):
    """With a one-item pool (tau = 1) the only way to keep the GPU busy is stealing: donations
    happen in both the 16- and the 32-level stack, and the counts stay exact."""
    gm = env["gm"]
    for k, seed in ((14, 3), (30, 2)):
        q = query(env, k, seed, 2, False)
        ref = oracle_count(env, q)
        p = gm.gm_plan_query(env["g"], q)
        don = 0
        for kw in (dict(), dict(set_count=False, symmetry=False), dict(pair_count=False)):
            c, st = gm.gm_count(p, tau=1, steal=True, **kw)
            assert c == ref, (q.name, kw)
            don += st["donations"]
        assert don > 0, q.name


def test_root_restricted_counts_large(env):
    """User root lists (no symmetry breaking) at D=16/32: the count over sampled roots equals the
    oracle's per-root counts summed."""
    gm = env["gm"]
    og = env["og"]
    rs = np.random.default_rng(5)
    for k, seed, leaves in ((12, 1, 0), (22, 3, 2), (30, 4, 1)):
        q = query(env, k, seed, leaves)
        p = gm.gm_plan_query(env["g"], q)
        u0 = p.info()["order"][0]
        cands = np.flatnonzero(p.candidates(u0))
        roots = rs.permutation(cands)[:24]
        ref = sum(og.count(q, fixed=(u0, int(v))) for v in roots)
        for tau in (1, 10 ** 6):
            assert gm.gm_count(p, roots=roots.astype(np.uint32), tau=tau)[0] == ref


def test_config4_sampled_roots_full_queries():
    """configs[3] at full size: R-MAT scale 24 (16.8 M vertices, ~265 M adjacency entries, 16
    labels) with the bench's own 16-vertex dense queries and their 12- and 9-vertex prefixes
    in the planner's order (induced, connected sub-queries: the same k_dfs<16, false>
    kernel), counted on sampled roots of phi[0] -- the query's own seed image first, so
    nonzero counts are covered -- equal the oracle's per-root counts on the whole graph
    (roots whose oracle search stays under a work budget)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import time
    import bench
    import gminputs.gpu as gg
    import paper_2604_10601_b200 as gm
    t0 = time.time()
    cfg = bench.CONFIGS["rmat24"]
    n, s, d, lab = bench.make_graph_device(cfg)
    lh = lab.cpu().numpy().view(np.uint32)
    adj = gg.DeviceNeighbors(n, s, d)
    queries = bench.build_queries(cfg, adj, lh)
    seeds = [gi.grow_query(adj, lh, q.n, seed=sd, dense=True, min_avg_degree=3.0, with_vertices=True)[1]
             for q, sd in zip(queries, cfg["dense"])]
    g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
    print(f"[config4] graph + queries {time.time() - t0:.1f}s", flush=True)
    og = OracleGraph(n, s.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32), lh)
    print(f"[config4] oracle graph {time.time() - t0:.1f}s", flush=True)
    del adj, s, d
    torch.cuda.empty_cache()
    rs = np.random.default_rng(24)
    checked = nonzero = 0
    for q, chosen in zip(queries, seeds):
        order = gm.gm_plan_query(g, q).info()["order"]
        for k in (16, 12, 9):
            keep = order[:k]
            idx = {u: i for i, u in enumerate(keep)}
            sub = gi.Query(k, [(idx[a], idx[b]) for a, b in q.edges.tolist() if a in idx and b in idx],
                           [int(q.labels[u]) for u in keep], name=f"{q.name}[:{k}]")
            p = gm.gm_plan_query(g, sub, order=list(range(k)))
            cands = np.flatnonzero(p.candidates(0))
            roots, ref = [], 0
            for v in [int(chosen[keep[0]])] + [int(x) for x in rs.permutation(cands)[:120]]:
                if v in roots:
                    continue
                c = og.count(sub, fixed=(0, v), max_nodes=4_000_000)
                if c is not None:
                    roots.append(v); ref += c; nonzero += c > 0
                    # tau = 1: the single root goes straight to k_dfs<16, false> (no BFS levels)
                    c1, st1 = gm.gm_count(p, roots=np.array([v], np.uint32), tau=1, time_limit_ms=60000)
                    assert c1 == c, (sub.name, v)
                    assert st1["stack_levels"] == 16 or st1["dfs_launches"] == 0
                if len(roots) == 4:
                    break
            c, st = gm.gm_count(p, roots=np.array(roots, np.uint32), time_limit_ms=60000)
            print(f"[config4] {sub.name}: {len(roots)} roots, count {ref}, {time.time() - t0:.1f}s", flush=True)
            assert st["timed_out"] == 0
            assert c == ref, (sub.name, roots)
            checked += len(roots)
    assert checked >= 24 and nonzero >= 1, (checked, nonzero)


@pytest.mark.parametrize("k,seed,leaves,same", [(10, 3, 2, True), (14, 4, 2, False), (22, 4, 2, True), (30, 2, 1, False),
                                                (16, 3, 0, False), (32, 3, 0, False)])
def test_two_level_hub_index(env, k, seed, leaves, same):
    """The hub index's summary level (1 bit per 256-vertex block, used by default only when the
    index exceeds L2) forced on, with every vertex of degree >= 2 a hub: counts at D=16/32 on
    every counting path equal the oracle's; then the default index is restored."""
    gm = env["gm"]
    q = query(env, k, seed, leaves, same)
    g = env["g"]
    g.build_hubs(64 << 20, 2, 1)
    try:
        assert g.info()["hub_summary_words"] > 0
        check_all_paths(env, q)
    finally:
        g.build_hubs(64 << 20, 64, -1)
