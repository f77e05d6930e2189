"""Host-side timing of the e2e legs at the bench workload (configs[2]): per
call (append, exploit / exploit_wait, best_path, exploit_async) in the
synchronous and the pipelined (NEXT-1) forms, inputs in pinned host memory.
    python tools/e2e_pipe_probe.py"""
import json
import os
import statistics
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402
from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED, batches  # noqa: E402

a = types.SimpleNamespace(workload="cfg3", d=6, n=1_000_000, S=4096, gamma="k", boxes=20, seed=0,
                          warmup=0, steps=20, graph_cache="/tmp/g1m_bench.npz")
g, gm, _ = bench.make_graph(a, 0, 1)
S, K = a.S, 20
n0 = a.n - 2 * K * S
stream = torch.cuda.current_stream()
ctx = pirrt.Context(h_root=g.h_root(), stream=stream, vertex_capacity=g.n + 1024,
                    edge_capacity=int(2.4 * g.off[-1]) + 4096)
for lo, hi in batches(n0, S):
    if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        ctx.exploit()
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
inp = []
for k in range(2 * K):
    lo, hi = n0 + k * S, n0 + (k + 1) * S
    s, d, c = g.batch(lo, hi, directed=False)
    inp.append((pin(g.h[lo:hi]), pin(s), pin(d), pin(c)))
torch.cuda.synchronize()
T = {}


def tick(key, t0):
    t = time.perf_counter()
    T.setdefault(key, []).append(1e3 * (t - t0))
    return t


t_all = time.perf_counter()
for i in range(K):
    t = time.perf_counter()
    np_ = ctx.append(*inp[i], flags=EDGES_UNDIRECTED)
    t = tick("sync.append", t)
    if np_ > 0:
        ctx.exploit()
        t = tick("sync.exploit", t)
    ctx.best_path()
    tick("sync.best_path", t)
torch.cuda.synchronize()
sync_ms = 1e3 * (time.perf_counter() - t_all) / K
inflight = False
t_all = time.perf_counter()
for i in range(K, 2 * K):
    t = time.perf_counter()
    np_ = ctx.append(*inp[i], flags=EDGES_UNDIRECTED)
    t = tick("pipe.append", t)
    if inflight:
        ctx.exploit_wait()
        t = tick("pipe.wait", t)
        inflight = False
    ctx.best_path()
    t = tick("pipe.best_path", t)
    if np_ > 0:
        ctx.exploit_async()
        inflight = True
        tick("pipe.async", t)
if inflight:
    ctx.exploit_wait()
torch.cuda.synchronize()
pipe_ms = 1e3 * (time.perf_counter() - t_all) / K
print(json.dumps({"sync_ms_per_step_wall": round(sync_ms, 4), "pipe_ms_per_step_wall": round(pipe_ms, 4),
                  "calls_ms_median": {k: round(statistics.median(v), 4) for k, v in T.items()}}))
