#!/usr/bin/env python
"""bench.py -- device-timed subgraph-matching throughput (embeddings/s, query ms).

Workload (BASELINE.json configs[1], the single-GPU headline config): R-MAT scale 18,
16 sampled edges/vertex (262,144 vertices, ~3.8M undirected edges), 8 uniform labels, and
a query set of 8-vertex queries drawn with the §6.1 procedure: 4 dense (greedy-dense
growth, average degree >= 3) + 4 sparse (random-walk trees).  A step = the whole hot path
for every query of the set: gm_plan_query (candidate filter + order) and gm_count
(BFS init pool + fine-grained DFS), each query under a per-query time limit (sparse
8-vertex trees on a power-law graph have ~1e13 embeddings; the limit bounds the step).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config rmat18|er1k|rmat22]

N > 1 (torchrun): root candidates are split over ranks ((v / 64) % N == rank), every
rank holds a replica of the graph, per-query counts are summed with ONE NCCL all-reduce
per step; time = max over ranks of the device time.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (generator, params, labels, query size, dense seeds, sparse seeds, time limit ms)
    "rmat18": dict(kind="rmat", scale=18, ef=16, labels=8, qsize=8, dense=[1000, 1001, 1002, 1003],
                   sparse=[2000, 2001, 2002, 2003], limit_ms=1000.0, seed=2,
                   # the dense queries that complete (profiles/r02/explore_bench18.log: rq8_s1000
                   # and the four random-walk trees are still unsolved after 30 s), run without a
                   # binding limit once per bench as the latency leg
                   complete=dict(sizes=[8, 8, 8], seeds=[1001, 1002, 1003]), complete_limit_ms=60000.0,
                   complete_desc="rq8_s1001..1003 (dense 8-vertex, solved in 0.5-5 s); rq8_s1000 and "
                                 "wq8_s2000..2003 exceed 30 s",
                   desc="R-MAT scale 18 (262k vertices, ~3.8M edges, 8 labels), 8-vertex dense+sparse queries"),
    "er1k": dict(kind="er", n=1000, deg=8, labels=4, qsize=4, dense=[], sparse=[], fixed="tailed_triangle",
                 limit_ms=0.0, seed=11, desc="Erdos-Renyi G(n=1000, avg deg 8, 4 labels), tailed triangle"),
    "rmat22": dict(kind="rmat", scale=22, ef=16, labels=1, qsize=0, dense=[], sparse=[],
                   fixed=["triangle", "clique4", "cycle5"], limit_ms=5000.0, seed=3,
                   desc="R-MAT scale 22 unlabelled (4.2M vertices, ~64M edges): triangle / 4-clique / 5-cycle",
                   note="5-cycle: >= 3.9e14 embeddings (a uniform 0.2 % root sample, 3688 of 1.84M roots, found "
                        "7.8e11 before its 60 s limit: profiles/r02/rmat22_sample.log), i.e. >= 3.9e13 "
                        "symmetry-breaking representatives, each a validated last-level task: it cannot "
                        "complete within the 5 s limit at any rate this path reaches (~7e9 per second)"),
    "rmat24": dict(kind="rmat", scale=24, ef=8, labels=16, qsize=16, dense=[1000, 1001, 1002, 1003],
                   sparse=[], limit_ms=2000.0, seed=4,
                   desc="LiveJournal-shaped R-MAT scale 24 (16.8M vertices, ~265M adjacency entries, 16 labels), "
                        "16-vertex dense queries"),
    "rmat26": dict(kind="rmat", scale=26, ef=16, labels=16, qsize=[24, 24, 32, 32], dense=[1000, 1001, 1002, 1003],
                   sparse=[], limit_ms=2000.0, seed=5,
                   desc="Friendster-shaped R-MAT scale 26 (67M vertices, ~2.1B adjacency entries, 16 labels), "
                        "24/32-vertex dense queries under a per-query time limit"),
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def build_queries(cfg, adj, lab):
    """The config's query set; adj = gminputs.HostAdjacency or gminputs.gpu.DeviceNeighbors."""
    import gminputs as gi
    qs = []
    sizes = cfg["qsize"] if isinstance(cfg["qsize"], list) else [cfg["qsize"]] * len(cfg.get("dense", []))
    for s, k in zip(cfg.get("dense", []), sizes):
        qs.append(gi.grow_query(adj, lab, k, seed=s, dense=True, min_avg_degree=3.0))
    for s in cfg.get("sparse", []):
        qs.append(gi.walk_query(adj, lab, cfg["qsize"], seed=s))
    fx = cfg.get("fixed")
    if fx:
        for name in ([fx] if isinstance(fx, str) else fx):
            if name == "tailed_triangle":
                qs.append(gi.tailed_triangle((0, 1, 2, 3)))
            elif name == "triangle":
                qs.append(gi.triangle())
            elif name.startswith("clique"):
                qs.append(gi.clique(int(name[6:])))
            elif name.startswith("cycle"):
                qs.append(gi.cycle(int(name[5:])))
    for i, q in enumerate(qs):
        q.name = q.name or f"q{i}"
    return qs


def build_complete_queries(cfg, adj, lab):
    """The config's complete-run query set (no time limit binds: query ms is a latency)."""
    import gminputs as gi
    c = cfg.get("complete")
    if not c:
        return []
    qs = [gi.grow_query(adj, lab, k, seed=sd, dense=True, min_avg_degree=3.0) for k, sd in zip(c["sizes"], c["seeds"])]
    return qs


def make_graph_host(cfg):
    import gminputs as gi
    if cfg["kind"] == "rmat":
        n, s, d = gi.rmat_edges(cfg["scale"], cfg["ef"], cfg["seed"])
    else:
        n, s, d = gi.er_edges(cfg["n"], cfg["deg"], cfg["seed"])
    lab = gi.uniform_labels(n, cfg["labels"], cfg["seed"])
    return n, s, d, lab


def make_graph_device(cfg):
    import gminputs.gpu as gg
    if cfg["kind"] == "rmat":
        n, s, d = gg.rmat_edges(cfg["scale"], cfg["ef"], cfg["seed"])
    else:
        n, s, d = gg.er_edges(cfg["n"], cfg["deg"], cfg["seed"])
    lab = gg.uniform_labels(n, cfg["labels"], cfg["seed"])
    return n, s, d, lab


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, val in zip(names, p[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, cfg, world, rank):
    """The oracle (plain C, one host core) on a bounded sample of the same workload."""
    if rank != 0:
        return
    import gminputs as gi
    from oracle import OracleGraph
    n, s, d, lab = make_graph_host(cfg)
    qs = build_queries(cfg, gi.HostAdjacency(*gi.simple_adjacency(n, s, d)), lab)
    og = OracleGraph(n, s, d, lab)
    budget_s = float(os.environ.get("GM_REF_STEP_S", "4.0"))
    rs = np.random.default_rng(0)
    times, counts, samples = [], [], []
    for step in range(args.warmup + args.steps):
        c, dt, nroots = oracle_sample(og, qs, lab, rs, budget_s)
        if step >= args.warmup:
            times.append(dt); counts.append(c); samples.append(nroots)
    value = sum(counts) / sum(times)
    line = {
        "impl": "reference", "metric": "embeddings/sec", "value": value, "unit": "embeddings/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak" if cfg["limit_ms"] > 0 else "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"]},
        "cpu_baseline": {"value": value, "unit": "embeddings/s", "cores": 1, "kind": "oracle",
                         "sample": f"per step: embeddings found by the oracle rooted at "
                                   f"{int(np.mean(samples))} random roots (query vertex 0 pinned, <= "
                                   f"{ORACLE_MAX_NODES:.0e} search-tree nodes per root) across {len(qs)} queries, "
                                   f"~{budget_s:.0f}s of one host core"},
        "e2e": {"value": value, "unit": "embeddings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


ORACLE_MAX_NODES = 200_000     # search-tree nodes per sampled root (both oracle legs)


def oracle_sample(og, qs, lab, rs, budget_s, max_nodes=ORACLE_MAX_NODES):
    """The oracle on bounded work, like the GPU arm's time-limited queries: for each query,
    random roots for query vertex 0, each searched for at most max_nodes tree nodes, until
    budget_s/len(qs) seconds of one core are spent.  Returns (embeddings found, seconds,
    roots searched)."""
    c, t_all, nroots = 0, 0.0, 0
    per_q = budget_s / len(qs)
    for q in qs:
        tq = time.perf_counter()
        cand = np.flatnonzero(lab == q.labels[0])
        for v in rs.permutation(cand):
            found, _ = og.count_budgeted(q, fixed=(0, int(v)), max_nodes=max_nodes)
            c += found
            nroots += 1
            if time.perf_counter() - tq > per_q:
                break
        t_all += time.perf_counter() - tq
    return c, max(t_all, 1e-9), nroots


def cpu_baseline(cfg, qs, n, s, d, lab, budget_s=12.0):
    """Oracle (one host core) on a bounded sample of this workload."""
    from oracle import OracleGraph
    og = OracleGraph(n, s, d, lab)
    c, dt, nroots = oracle_sample(og, qs, lab, np.random.default_rng(0), budget_s)
    return {"value": c / dt, "unit": "embeddings/s", "cores": 1, "kind": "oracle",
            "sample": f"embeddings found by the oracle rooted at {nroots} random roots (query vertex 0 "
                      f"pinned, <= {ORACLE_MAX_NODES:.0e} search-tree nodes per root) across the {len(qs)} queries of this "
                      f"workload, {dt:.1f}s of one host core"}


# ----------------------------------------------------------------------------- our arm

# The paper's own numbers, quoted with the GPU it names (context only, not a target): Table 2
# (PAPER.md:626-666), gMatch (GM) search time in ms on an RTX 4090 (PAPER.md:579, 128 SMs, 24 GB),
# unlabelled small patterns P1-P9 (Figure 8, an image: the patterns are not defined in the text);
# lj is LiveJournal (config 4's shape), fr is Friendster (config 5's shape).
PAPER_CONTEXT = {
    "gpu": "NVIDIA RTX 4090 (PAPER.md:579)",
    "source": "PAPER.md Table 2 (lines 626-666), gMatch column, search time ms",
    "lj_ms": {"P1": 31, "P2": 422, "P3": 2080, "P4": 4127, "P5": 334373, "P6": 637667, "P7": 305968,
              "P8": 221493, "P9": 25114},
    "fr_ms": {"P1": 4354, "P2": 12132, "P3": 53556, "P4": 2806445, "P5": 1068031, "P6": 1519540,
              "P7": 731884, "P8": 235798, "P9": 33776},
    "idle_rate": "< 5 % on 12-vertex queries (PAPER.md:744, Table 5)",
}


def idle_rate(tasks, rounds):
    """Idle lane-slots of the DFS's scatter rounds: 1 - tasks / (32 * rounds).  The batched
    analogue of the paper's idle rate (the mean over partial matches of
    (32 - |C_M^L(u)|) / 32): the share of lanes a round leaves without a task."""
    return 1.0 - tasks / (32.0 * rounds) if rounds else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="rmat18", choices=sorted(CONFIGS))
    ap.add_argument("--time-limit-ms", type=float, default=None)
    ap.add_argument("--tau", type=float, default=1e6)
    ap.add_argument("--no-steal", action="store_true")
    ap.add_argument("--root-order", default="shuffled", choices=["shuffled", "hubs"],
                    help="pool order of the timed steps: seeded root permutation (default: a time-limited "
                         "query explores a uniform sample of its roots) or device-id order (hubs first)")
    ap.add_argument("--static-roots", action="store_true",
                    help="N > 1: static (v/64) %% N root partition instead of the shared pool counter")
    ap.add_argument("--no-team", action="store_true",
                    help="N > 1: no cross-GPU stealing (idle warps steal only within their GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-context", action="store_true", help="skip the context legs (hubs-first order, "
                    "Alg. 2 as written, gm_enumerate, the complete query set)")
    ap.add_argument("--per-query", action="store_true", help="also print the per-query list to stderr")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    limit = cfg["limit_ms"] if args.time_limit_ms is None else args.time_limit_ms
    root_seed = 1 if args.root_order == "shuffled" else 0

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import torch
    import torch.distributed as dist
    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    gpu = local_rank % torch.cuda.device_count()   # one rank per GPU (ranks share a GPU only when
    torch.cuda.set_device(gpu)                     # testing the multi-rank path on a 1-GPU box)
    dev = torch.device("cuda", gpu)
    if world > 1:
        backend = os.environ.get("GM_DIST_BACKEND", "nccl")   # gloo: several ranks on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import gminputs as gi
    import paper_2604_10601_b200 as gm
    from paper_2604_10601_b200 import partition

    # ---- inputs: graph generated on this GPU (replica per rank); queries from host adjacency
    n, s_dev, d_dev, lab_dev = make_graph_device(cfg)
    lab_h = lab_dev.cpu().numpy().view(np.uint32)
    small = cfg["kind"] != "rmat" or cfg["scale"] <= 20
    s_h = d_h = None
    if small:                                    # host copy for query growth + the oracle baseline
        s_h = s_dev.cpu().numpy().view(np.uint32)
        d_h = d_dev.cpu().numpy().view(np.uint32)
        adj = gi.HostAdjacency(*gi.simple_adjacency(n, s_h, d_h))
    else:                                        # grow queries by scanning the device edge list
        import gminputs.gpu as gg
        adj = gg.DeviceNeighbors(n, s_dev, d_dev)
    qs = build_queries(cfg, adj, lab_h)
    cq = build_complete_queries(cfg, adj, lab_h) if not args.no_context else []
    del adj
    g = gm.gm_load_graph(n, s_dev, d_dev, lab_dev, cfg["labels"])
    del s_dev, d_dev
    torch.cuda.empty_cache()
    ginfo = g.info()
    stream = torch.cuda.current_stream()
    run_kw = dict(tau=int(args.tau), rank=rank, world=world, steal=not args.no_steal, time_limit_ms=limit,
                  root_seed=root_seed)
    # N > 1: dynamic chunk assignment -- every rank's DFS claims pool batches from counters in
    # rank 0's memory (CUDA IPC + NVLink peer atomics, one slot per query, reset once per
    # step); --static-roots: (v/64) % N partition
    shared_ptr = None
    nslots = max(len(qs), len(cq), 1)
    if world > 1 and not args.static_roots:
        if rank == 0:
            shared_ptr, handle = gm.gm_pool_counter_create(nslots)
        box = [handle if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        if rank != 0:
            shared_ptr = gm.gm_pool_counter_open(box[0])
        run_kw = dict(tau=int(args.tau), steal=not args.no_steal, time_limit_ms=limit, root_seed=root_seed)
        if not args.no_team and not args.no_steal:
            # cross-GPU stealing: every rank maps every other rank's steal ring and work word
            handles = [None] * world
            dist.all_gather_object(handles, gm.gm_team_export())
            team = gm.gm_team_open(world, rank, handles)
            run_kw["team"] = team

    counts_dev = torch.zeros(nslots, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def reset_slots():
        """Shared pool counters: zeroed by rank 0 before a step; every rank waits (outside the
        timed region) so no rank claims from a slot before its reset."""
        if shared_ptr is not None:
            if rank == 0:
                gm.gm_pool_counter_reset(shared_ptr, nslots)
            torch.cuda.synchronize()
            dist.barrier()

    def step(queries, kw_extra=None):
        """One pass of the hot path over a query set: per query gm_plan_query (filter + order)
        and gm_count (BFS pool + DFS).  Returns per-query (stats, start event, end event) and
        the reduced count halves (the step's one collective for N > 1)."""
        out = []
        for i, q in enumerate(queries):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            p = gm.gm_plan_query(g, q, filter="nlf")
            kw = dict(run_kw, **(kw_extra or {}))
            if shared_ptr is not None:          # query i claims from its own slot (reset per step)
                kw["shared_pool_ctr"] = gm.pool_counter_slot(shared_ptr, i)
            _, st = gm.gm_count(p, out=counts_dev[i:i + 1], **kw)
            e1.record(stream)
            out.append((st, e0, e1))
            del p
        halves = partition.reduce_count_halves(counts_dev[:len(queries)])
        return out, halves

    def rank_sums(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t)
        return t.tolist()

    def rank_max(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def summarize(queries, res, exact):
        """Per-query list (exact counts summed over ranks; work counters summed; times max over
        ranks)."""
        loc = []
        for st, e0, e1 in res:
            loc += [st["tasks"], st["rounds"], st["words"], st["donations"], st["timed_out"]]
        sums = rank_sums(loc)
        tmax = rank_max([e0.elapsed_time(e1) for _, e0, e1 in res] + [st["dfs_ms"] for st, _, _ in res])
        nq = len(queries)
        rows = []
        for i, (q, (st, _, _)) in enumerate(zip(queries, res)):
            tasks, rounds, words, don, to = sums[5 * i:5 * i + 5]
            rows.append({"q": q.name, "n": int(q.n), "m": int(len(q.edges)), "embeddings": exact[i],
                         "completed": to == 0, "ms": round(tmax[i], 3), "dfs_ms": round(tmax[nq + i], 3),
                         "tasks": int(tasks), "rounds": int(rounds), "words": int(words),
                         "idle_rate": None if not rounds else round(idle_rate(tasks, rounds), 4),
                         "aut": st["automorphisms"], "paths": st["paths"], "D": st["stack_levels"],
                         "pool": st["pool_size"], "depth": st["pool_depth"], "donations": int(don)})
        return rows

    def one_pass(queries, kw_extra=None):
        """Untimed-by-contract context leg: one flushed pass, device-timed per query."""
        flush.zero_()
        reset_slots()
        torch.cuda.synchronize()
        res, halves = step(queries, kw_extra)
        torch.cuda.synchronize()
        exact = partition.count_totals(halves)
        rows = summarize(queries, res, exact)
        t = sum(r["ms"] for r in rows)
        return {"value": sum(exact) / (t / 1e3) if t else None, "unit": "embeddings/s",
                "ms": round(t, 3), "tasks_per_s": sum(r["tasks"] for r in rows) / (t / 1e3) if t else None,
                "solved": sum(r["completed"] for r in rows), "queries": len(rows), "per_query": rows}

    for _ in range(args.warmup):
        flush.zero_()
        reset_slots()
        step(qs)
    torch.cuda.synchronize()

    clocks = ClockSampler(gpu)
    clocks.start()
    step_ms, dfs_ms, dfs_launches, kernel_launches = [], [], 0, 0
    total_emb, timeouts, tasks, rounds = 0, 0, 0, 0
    tasks_q = [0] * len(qs)
    q_ms_all, q_ms_solved = [], []
    per_query = None
    for k in range(args.steps):
        flush.zero_()                                # L2 flush outside the timed region
        reset_slots()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        res, halves = step(qs)
        s1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        step_ms.append(s0.elapsed_time(s1))
        exact = partition.count_totals(halves)       # exact uint64 sums (no int64 wrap)
        total_emb += sum(exact)
        for i, (st, e0, e1) in enumerate(res):
            dfs_ms.append(st["dfs_ms"])
            dfs_launches += st["dfs_launches"]
            tasks_q[i] += st["tasks"]
            tasks += st["tasks"]
            rounds += st["rounds"]
            kernel_launches += st["kernel_launches"] + 1       # + the filter kernel of the plan
            timeouts += st["timed_out"]
        rows = summarize(qs, res, exact)             # (collectives outside the timed region)
        for r in rows:
            q_ms_all.append(r["ms"])
            if r["completed"]:
                q_ms_solved.append(r["ms"])
        if per_query is None:
            per_query = rows
    clk = clocks.stop()

    # ---- max over ranks
    T_ms, T_dfs = rank_max([sum(step_ms), sum(dfs_ms)])
    tasks_all, rounds_all, launches_all, timeouts_all = rank_sums([tasks, rounds, kernel_launches, timeouts])
    tasks_q_all = rank_sums(tasks_q)

    # ---- algorithmic words per task (the roofline's per-unit figure): one flushed counting pass
    # of the same workload with GM_FLAG_COUNT_WORDS (the timed searches run the kernel compiled
    # without the per-probe counters, which cost 12-23 % throughput); algorithmic bytes of the
    # timed launches = sum over queries of tasks done x 4 x words per task of that query
    cal = one_pass(qs, dict(count_words=True))["per_query"]
    wpt = [r["words"] / r["tasks"] if r["tasks"] else 0.0 for r in cal]
    words_all = sum(t * w for t, w in zip(tasks_q_all, wpt))
    for r, w in zip(per_query, wpt):
        r.pop("words", None)
        r["words_per_task"] = round(w, 3)
    emb_per_step = total_emb / args.steps
    value = total_emb / (T_ms / 1e3)

    # ---- end to end through the public API with host buffers (rank-local share, wall clock)
    e2e_emb, e2e_s, h2d, d2h = 0, 0.0, 0, 0
    e2e_steps = max(1, min(args.steps, 5))
    for k in range(e2e_steps):
        flush.zero_()
        reset_slots()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        local = []
        for i, q in enumerate(qs):
            p = gm.gm_plan_query(g, q, filter="nlf")      # query arrays copied H2D by the library
            kw = dict(run_kw)
            if shared_ptr is not None:
                kw["shared_pool_ctr"] = gm.pool_counter_slot(shared_ptr, i)
            c, _ = gm.gm_count(p, **kw)                    # count read back D2H
            local.append(c)
            h2d += q.edges.nbytes + q.labels.nbytes
            d2h += 8
        if world > 1:
            t = torch.tensor(partition.as_int64_bits(local), dtype=torch.int64, device=dev)
            local = partition.reduce_counts(t)
            d2h += 8 * len(qs)
        dt = time.perf_counter() - t0
        dt = rank_max([dt])[0]
        e2e_s += dt
        e2e_emb += sum(local)
    e2e = {"value": e2e_emb / e2e_s, "unit": "embeddings/s", "h2d_bytes_per_step": h2d // e2e_steps,
           "d2h_bytes_per_step": d2h // e2e_steps, "steps": e2e_steps}
    if s_h is not None:
        # gm_load_graph from host (pinned) edge arrays: the transfer + CSR build a user pays once
        # per graph (PAPER.md:681 counts t_transfer in t_query), reported beside e2e
        sp = torch.from_numpy(s_h.view(np.int32)).pin_memory().numpy().view(np.uint32)
        dp = torch.from_numpy(d_h.view(np.int32)).pin_memory().numpy().view(np.uint32)
        lp = torch.from_numpy(lab_h.view(np.int32)).pin_memory().numpy().view(np.uint32)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g2 = gm.gm_load_graph(n, sp, dp, lp, cfg["labels"])
        torch.cuda.synchronize()
        e2e["graph_load_ms"] = round(1e3 * (time.perf_counter() - t0), 3)
        e2e["graph_load_h2d_bytes"] = int(sp.nbytes + dp.nbytes + lp.nbytes)
        g2.free()
        del g2

    # ---- context legs (one flushed pass each, device-timed; not the headline)
    context = None
    if not args.no_context:
        context = {
            "root_order_of_headline": args.root_order,
            "hubs_first": one_pass(qs, dict(root_seed=0)) if root_seed else one_pass(qs, dict(root_seed=1)),
            "alg2_as_written": one_pass(qs, dict(set_count=False, pair_count=False)),
            "complete_set": one_pass(cq, dict(time_limit_ms=cfg.get("complete_limit_ms", 60000.0))) if cq else None,
            "paper": PAPER_CONTEXT,
        }
        if not args.root_order == "shuffled":
            context["shuffled"] = context.pop("hubs_first")
        context["alg2_as_written"]["note"] = ("set counting and pair counting off: every last-level "
                                              "candidate validated as its own task (Alg. 2 lines 12-13)")
        if context["complete_set"]:
            context["complete_set"]["desc"] = cfg.get("complete_desc")
        # gm_enumerate: embeddings written as rows (nq uint32 each, original ids) to a device
        # buffer of `cap` rows; the search stops when the buffer is full (stop_at_capacity) or
        # at the time limit, so rows/s is the output rate of the enumerate kernel
        enum = []
        cap = (1 << 26) // max(q.n for q in qs)
        for q in qs:
            p = gm.gm_plan_query(g, q, filter="nlf")
            buf = torch.empty(cap * q.n, dtype=torch.int32, device=dev)
            flush.zero_()
            torch.cuda.synchronize()
            _, tot, st = gm.gm_enumerate(p, cap, out=buf, time_limit_ms=limit, root_seed=root_seed,
                                         tau=int(args.tau), rank=rank, world=world, stop_at_capacity=True)
            enum.append((q.name, tot, min(tot, cap), st["total_ms"], st["timed_out"]))
            del buf, p
        tms = sum(e[3] for e in enum)
        context["enumerate"] = {"value": sum(e[2] for e in enum) / (tms / 1e3), "unit": "embeddings/s",
                                "rows_bytes_per_s": sum(e[2] * q.n * 4 for e, q in zip(enum, qs)) / (tms / 1e3),
                                "capacity_rows_per_query": cap,
                                "per_query": [{"q": a, "found": b, "rows": c, "ms": round(d, 3),
                                               "stopped": e} for a, b, c, d, e in enum],
                                "note": "gm_enumerate writing rows to a device buffer until it is full "
                                        "(GM_FLAG_STOP_AT_CAPACITY) or the time limit; value = rows written "
                                        "per second, rank-local"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_kind = peaks()
    # roofline of the dominant kernel (k_dfs): algorithmic bytes = 4 * words per launch
    dfs_launch_ms = T_dfs / max(1, dfs_launches) if dfs_launches else None
    bytes_per_launch = 4.0 * words_all / max(1, dfs_launches * (world if world > 1 else 1)) if dfs_launches else 0
    achieved = (4.0 * words_all / world) / (T_dfs / 1e3) / 1e9 if T_dfs > 0 else 0.0
    traffic, ncu = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(args.config)
        ncu = tj.get("ncu", {}).get(args.config)
    except Exception:
        pass
    solved = len(q_ms_solved)
    line = {
        "metric": "embeddings/sec", "value": value, "unit": "embeddings/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": T_ms / args.steps, "higher_is_better": True,
        # each rank searches its share of every query for up to the same per-query time limit:
        # per-GPU work (a time budget) is fixed as N grows
        "scaling": "weak" if limit > 0 else "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "queries": len(qs),
                   **({"note": cfg["note"]} if cfg.get("note") else {}),
                   "per_query_time_limit_ms": limit,
                   "root_order": ("seeded pseudo-random root permutation (root_seed=1): a time-limited query "
                                  "counts the embeddings of a uniform sample of its roots"
                                  if root_seed else "device-id order (hubs first)"),
                   "solved_queries_per_step": solved / args.steps,
                   "unsolved_queries_per_step": (len(q_ms_all) - solved) / args.steps,
                   "query_ms_mean": statistics.mean(q_ms_all),
                   "query_ms_mean_solved": statistics.mean(q_ms_solved) if q_ms_solved else None,
                   "embeddings_per_step": emb_per_step, "tau": int(args.tau), "steal": not args.no_steal,
                   "filter": "nlf", "graph": {k: ginfo[k] for k in ("n", "num_adj", "num_labels", "d_max", "hubs")},
                   "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": ("1 GPU, whole pool on one device" if world == 1 else
                                   f"{world} GPU(s), CSR replicated, " +
                                   ("pool batches claimed from shared counters (NVLink peer system-scope atomics)"
                                    + (", cross-GPU stealing (gm_team)" if "team" in run_kw else "")
                                    if shared_ptr is not None else "static root partition") +
                                   ", 1 all-reduce of the counts per step")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_dfs", "launch_ms_mean": dfs_launch_ms,
                     "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": peak_kind,
                     "unit_of_work": "task T_M(u, v) (one candidate validation, PAPER.md:374)",
                     "bytes_per_task": {r["q"]: round(4 * w, 3) for r, w in zip(cal, wpt)},
                     "bytes_method": "4 x words per task (a flushed GM_FLAG_COUNT_WORDS pass of the same queries "
                                     "and limits) x tasks done in the timed launches",
                     "share_of_step": T_dfs / T_ms if T_ms else None, "ncu": ncu},
        "gpu_launches": int(launches_all),
        "tasks_per_s": tasks_all / (T_ms / 1e3),
        "idle_rate": idle_rate(tasks_all, rounds_all),
        "clocks": clk,
        "e2e": e2e,
        "per_query": per_query,
    }
    if context is not None:
        line["context"] = context
    if not args.no_cpu_baseline and world == 1:
        if s_h is not None:
            line["cpu_baseline"] = cpu_baseline(cfg, qs, n, s_h, d_h, lab_h)
        else:
            line["cpu_baseline"] = {"value": None, "unit": "embeddings/s", "cores": 1, "kind": "oracle",
                                    "sample": "not run: building the oracle's host CSR for this graph size "
                                              "exceeds the bench time budget"}
    if args.per_query:
        print(json.dumps(per_query), file=sys.stderr)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
