"""Per-batch exploit time at the bench workload (configs[2]: 6-D 1M gamma_k,
S = 4096) and at configs[1] (2-D 50k gamma*, S = 1) under a sweep of
persistent-grid sizes and incremental-Improve modes -- the per-batch exploit
is barrier-latency bound, so the grid size sets the barrier cost.
    python tools/grid_probe.py > gpurun_out/grid_probe.jsonl"""
import json
import os
import statistics
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402
from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED, batches  # noqa: E402

a = types.SimpleNamespace(workload="cfg3", d=6, n=1_000_000, S=4096, gamma="k", boxes=20, seed=0,
                          warmup=0, steps=20, graph_cache="/tmp/g1m_bench.npz")
g, gm, _ = bench.make_graph(a, 0, 1)
S, K = a.S, 24
n0 = a.n - K * S
ENVS = ("PIRRT_INC_IMPROVE", "PIRRT_INC_MAX")


def run(gb, env):
    for k in ENVS:
        os.environ.pop(k, None)
    os.environ.update(env)
    ctx = pirrt.Context(h_root=g.h_root(), vertex_capacity=g.n + 1024,
                        edge_capacity=int(2.4 * g.off[-1]) + 4096, grid_blocks=gb)
    for lo, hi in batches(n0, S):
        if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
            ctx.exploit()
    ex = []
    for k in range(K):
        lo, hi = n0 + k * S, n0 + (k + 1) * S
        if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
            ex.append(ctx.exploit())
    ex = ex[4:]
    ms = [s.device_ms for s in ex]
    rec = {"workload": "cfg3", "grid_blocks": ex[0].grid_blocks, "env": env,
           "exploit_ms_mean": round(statistics.mean(ms), 4), "median": round(statistics.median(ms), 4),
           "iterations": round(statistics.mean([s.iterations for s in ex]), 2),
           "barriers": round(statistics.mean([s.barriers for s in ex]), 1),
           "improve_ms": round(statistics.mean([s.improve_ms for s in ex]), 4),
           "evaluate_ms": round(statistics.mean([s.evaluate_ms for s in ex]), 4)}
    print(json.dumps(rec), flush=True)


def run_cfg2(gb, env):
    for k in ENVS:
        os.environ.pop(k, None)
    os.environ.update(env)
    r = gen.rrg(2, 50000, gen.gamma_star(2), n_boxes=30, seed=gen.seed_of("cfg2", 0))
    ctx = pirrt.Context(h_root=r.h_root(), vertex_capacity=r.n + 16, grid_blocks=gb)
    ms = []
    for lo, hi in batches(r.n, 1):
        if ctx.append(r.h[lo:hi], *r.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
            st = ctx.exploit()
            if lo > 1000:
                ms.append(st.device_ms)
    print(json.dumps({"workload": "cfg2", "grid_blocks": gb, "env": env, "replans": len(ms),
                      "median": round(statistics.median(ms), 4),
                      "p95": round(float(np.percentile(ms, 95)), 4),
                      "mean": round(statistics.mean(ms), 4)}), flush=True)


for gb in (0, 148, 74, 37, 16):
    for env in ({}, {"PIRRT_INC_IMPROVE": "0"}):
        run(gb, env)
for gb in (0, 148, 74, 37, 16, 4, 1):
    run_cfg2(gb, {})
