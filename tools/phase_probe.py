"""Phase timeline of the per-batch exploit (DevCtl::phase_ns through the
diagnostic export pirrt_debug_phases) at the bench workload (configs[2],
6-D 1M gamma_k, S = 4096) and at configs[1] (2-D 50k gamma*, S = 1).
    python tools/phase_probe.py > gpurun_out/phase_probe.json"""
import ctypes as C
import json
import os
import statistics
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import gen  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402
from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED, batches  # noqa: E402

NAMES = ["improve_discovery", "improve_scan", "eval_inc_E2", "eval_inc_E3", "eval_inc_validate",
         "eval_full", "n_inc_evals", "n_improves"]
lib = pirrt._lib
lib.pirrt_debug_phases.argtypes = [C.c_void_p, C.c_void_p, C.c_int]


def phases(ctx):
    out = (C.c_ulonglong * 8)()
    lib.pirrt_debug_phases(ctx._h, out, 8)
    return list(out)


def summarize(name, recs, ex):
    tot = [sum(r[i] for r in recs) for i in range(8)]
    k = len(recs)
    out = {"workload": name, "exploits": k,
           "exploit_us": round(1e3 * statistics.mean([s.device_ms for s in ex]), 2),
           "barriers": round(statistics.mean([s.barriers for s in ex]), 2),
           "iterations": round(statistics.mean([s.iterations for s in ex]), 2)}
    for i in range(6):
        out[NAMES[i] + "_us_per_exploit"] = round(tot[i] / k / 1e3, 2)
    out["us_per_inc_eval"] = {NAMES[i]: round(tot[i] / max(1, tot[6]) / 1e3, 2) for i in (2, 3, 4)}
    out["us_per_improve"] = {NAMES[i]: round(tot[i] / max(1, tot[7]) / 1e3, 2) for i in (0, 1)}
    print(json.dumps(out), flush=True)


a = types.SimpleNamespace(workload="cfg3", d=6, n=1_000_000, S=4096, gamma="k", boxes=20, seed=0,
                          warmup=0, steps=20, graph_cache="/tmp/g1m_bench.npz")
g, gm, _ = bench.make_graph(a, 0, 1)
S, K = a.S, 24
n0 = a.n - K * S
ctx = pirrt.Context(h_root=g.h_root(), vertex_capacity=g.n + 1024,
                    edge_capacity=int(2.4 * g.off[-1]) + 4096)
for lo, hi in batches(n0, S):
    if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        ctx.exploit()
recs, ex = [], []
for k in range(K):
    lo, hi = n0 + k * S, n0 + (k + 1) * S
    if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        st = ctx.exploit()
        if k >= 4:
            ex.append(st)
            recs.append(phases(ctx))
summarize("cfg3", recs, ex)
del ctx

r = gen.rrg(2, 50000, gen.gamma_star(2), n_boxes=30, seed=gen.seed_of("cfg2", 0))
ctx = pirrt.Context(h_root=r.h_root(), vertex_capacity=r.n + 16)
recs, ex = [], []
for lo, hi in batches(r.n, 1):
    if ctx.append(r.h[lo:hi], *r.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        st = ctx.exploit()
        if lo > 1000:
            ex.append(st)
            recs.append(phases(ctx))
summarize("cfg2", recs, ex)
