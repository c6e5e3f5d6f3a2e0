"""Properties of the seeded input generators (gminputs)."""
import numpy as np

import gminputs as gi


def test_mix64_is_splitmix64():
    # splitmix64 with state 0: first output is 0xE220A8397B1DCDAF (Vigna's reference values)
    z = np.array([0x9E3779B97F4A7C15], dtype=np.uint64)
    assert int(gi._mix64(z)[0]) == 0xE220A8397B1DCDAF
    z = np.array([(2 * 0x9E3779B97F4A7C15) & gi.M64], dtype=np.uint64)
    assert int(gi._mix64(z)[0]) == 0x6E789E6AA1B965F4


def test_deterministic():
    a = gi.rmat_edges(10, 8, seed=5)
    b = gi.rmat_edges(10, 8, seed=5)
    c = gi.rmat_edges(10, 8, seed=6)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert not np.array_equal(a[1], c[1])


def test_rmat_heavy_tail():
    n, s, d = gi.rmat_edges(14, 8, seed=1)
    off, _ = gi.simple_adjacency(n, s, d)
    deg = np.sort(np.diff(off))[::-1]
    top = deg[: n // 100].sum()
    assert top > 0.10 * deg.sum()          # top-1% vertices hold >10% of adjacency
    assert deg[0] > 20 * deg.mean()


def test_uniform_and_zipf_labels():
    lab = gi.uniform_labels(200000, 16, seed=3)
    cnt = np.bincount(lab, minlength=16)
    exp = 200000 / 16
    assert np.all(np.abs(cnt - exp) < 5 * np.sqrt(exp))
    z = gi.zipf_labels(200000, 16, 1.0, seed=3)
    cz = np.bincount(z, minlength=16)
    assert 16 * 0.8 < cz[0] / cz[15] < 16 * 1.2    # Appendix A ratio (1/1)/(1/16)


def test_random_query_connected_and_induced():
    n, s, d = gi.er_edges(500, 8, seed=2)
    lab = gi.uniform_labels(n, 4, 2)
    off, nb = gi.simple_adjacency(n, s, d)
    for seed in range(20):
        q = gi.random_query(off, nb, lab, 8, seed)
        assert q.n == 8
        # connected
        seen, stack = {0}, [0]
        adj = {i: set() for i in range(q.n)}
        for a, b in q.edges:
            adj[int(a)].add(int(b)); adj[int(b)].add(int(a))
        while stack:
            x = stack.pop()
            for y in adj[x] - seen:
                seen.add(y); stack.append(y)
        assert len(seen) == 8
        w = gi.random_walk_query(off, nb, lab, 8, seed)
        assert w.n == 8 and len(w.edges) >= 7


def test_er_size():
    n, s, d = gi.er_edges(1000, 8, seed=0)
    assert n == 1000 and len(s) == 4000
