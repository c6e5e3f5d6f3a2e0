"""Multi-rank GPU paths (2 processes; they share GPU 0 when the box has one): the static root
partition and the cross-rank shared pool counter (CUDA IPC + peer atomics) both give per-rank
counts that sum, with one all-reduce, to the single-rank count and to the oracle."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gminputs as gi
        import paper_2604_10601_b200 as gm
        n, s, d = gi.rmat_edges(11, 8, 13)
        lab = gi.uniform_labels(n, 3, 13)
        g = gm.gm_load_graph(n, s, d, lab, 3)
        queries = [gi.tailed_triangle((0, 1, 2, 0)), gi.Query(4, [(0, 1), (1, 2), (2, 3)], [0, 1, 1, 2]),
                   gi.clique(3), gi.cycle(4)]
        # shared pool counter: rank 0 owns it, the others map it through CUDA IPC
        if rank == 0:
            ptr, handle = gm.gm_pool_counter_create(len(queries))
        else:
            ptr, handle = None, None
        box = [handle]
        dist.broadcast_object_list(box, src=0)
        if rank != 0:
            ptr = gm.gm_pool_counter_open(box[0])
        static = torch.zeros(len(queries), dtype=torch.int64)
        shared = torch.zeros(len(queries), dtype=torch.int64)
        # one counter slot per query, all reset once; no barrier between queries
        if rank == 0:
            gm.gm_pool_counter_reset(ptr, len(queries))
            torch.cuda.synchronize()
        dist.barrier()
        for i, q in enumerate(queries):
            p = gm.gm_plan_query(g, q)
            static[i] = gm.gm_count(p, rank=rank, world=world, root_chunk=8, tau=64)[0]
            shared[i] = gm.gm_count(p, shared_pool_ctr=gm.pool_counter_slot(ptr, i), tau=256)[0]
        dist.all_reduce(static)
        dist.all_reduce(shared)
        if rank == 0:
            from oracle import OracleGraph
            og = OracleGraph(n, s, d, lab)
            single = [gm.gm_count(gm.gm_plan_query(g, q))[0] for q in queries]
            ref = [og.count(q) for q in queries]
            out.put((static.tolist(), shared.tolist(), single, ref))
        dist.barrier()
        gm.gm_pool_counter_close(ptr, owner=(rank == 0))
    finally:
        dist.destroy_process_group()


def test_two_ranks_static_and_shared_pool():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    static, shared, single, ref = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert static == ref
    assert shared == ref
    assert single == ref


def _p4_closed_form(n, s, d):
    """4-vertex paths (ordered embeddings of P4) in the simple graph: sum over ordered edges
    (a, b) of (d_a - 1)(d_b - 1) minus trace(A^3) (tests/test_gpu_parity.py pins it)."""
    import gminputs as gi
    import scipy.sparse as sp
    off, nb = gi.simple_adjacency(n, s, d)
    deg = np.diff(off).astype(np.int64)
    rows = np.repeat(np.arange(n), deg)
    A = sp.csr_matrix((np.ones(len(nb), np.int64), (rows, nb.astype(np.int64))), shape=(n, n))
    return int(((deg[rows] - 1) * (deg[nb] - 1)).sum()) - int((A @ A).multiply(A).sum())


def _team_worker(rank, world, port, out):
    """Cross-GPU stealing team (gm_team): in mode 0 rank 1 takes no pool batches
    (GM_FLAG_NO_POOL), so every embedding it counts came from rank 0's steal ring over peer
    memory; in mode 1 both ranks claim from the shared pool and steal from each other.  The
    per-rank counts sum to the closed form.  The work is made long (every embedding of P4
    validated task by task: set/pair counting and symmetry breaking off) because two
    processes on ONE GPU time-slice it: rank 1's warps run while rank 0's are parked with
    items in its ring."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gminputs as gi
        import paper_2604_10601_b200 as gm
        n, s, d = gi.rmat_edges(13, 16, 77)
        g = gm.gm_load_graph(n, s, d)
        q = gi.Query(4, [(0, 1), (1, 2), (2, 3)], [0, 0, 0, 0])
        handles = [None] * world
        dist.all_gather_object(handles, gm.gm_team_export())
        team = gm.gm_team_open(world, rank, handles)
        if rank == 0:
            ptr, handle = gm.gm_pool_counter_create(4)
        else:
            ptr, handle = None, None
        box = [handle]
        dist.broadcast_object_list(box, src=0)
        if rank != 0:
            ptr = gm.gm_pool_counter_open(box[0])
        if rank == 0:
            gm.gm_pool_counter_reset(ptr, 4)
            torch.cuda.synchronize()
        dist.barrier()
        res = []
        p = gm.gm_plan_query(g, q, order=[1, 2, 0, 3])
        for mode in (0, 1):
            kw = dict(tau=4096, team=team, shared_pool_ctr=gm.pool_counter_slot(ptr, mode), set_count=False,
                      pair_count=False, symmetry=False)
            if mode == 0 and rank == 1:
                kw["no_pool"] = True
            c, st = gm.gm_count(p, **kw)
            res.append((c, st["donations"], st["tasks"]))     # (no barrier between searches: epochs)
        allres = [None] * world
        dist.all_gather_object(allres, res)
        if rank == 0:
            out.put((allres, _p4_closed_form(n, s, d)))
        dist.barrier()
        team.free()
        gm.gm_pool_counter_close(ptr, owner=(rank == 0))
    finally:
        dist.destroy_process_group()


def test_two_rank_team_cross_rank_stealing():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_team_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allres, ref = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for mode in (0, 1):
        c0, c1 = allres[0][mode][0], allres[1][mode][0]
        assert c0 + c1 == ref, (mode, c0, c1, ref)
    # rank 1 took no pool batch in mode 0: whatever it counted, it stole from rank 0's ring
    assert allres[1][0][0] > 0 and allres[1][0][2] > 0, allres
