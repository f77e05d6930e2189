"""Where the e2e step time goes (bench workload, configs[2]): the H2D of one
batch from pinned host memory alone, the deferred step pipeline with device
and with host inputs, and the host time inside step_async / step_wait.
    python tools/step_probe.py"""
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
n0 = a.n - 3 * K * S
stream = torch.cuda.current_stream()
ctx = pirrt.Context(h_root=g.h_root(), stream=stream, vertex_capacity=g.n + 1024,
                    edge_capacity=int(2.4 * g.off[-1]) + 4096)
for lo, hi in batches(n0, S):
    if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        ctx.exploit()
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
inp = []
for k in range(3 * K):
    lo, hi = n0 + k * S, n0 + (k + 1) * S
    s, d, c = g.batch(lo, hi, directed=False)
    inp.append(tuple(pin(x) for x in (g.h[lo:hi], s, d, c)))
out = {}
# (1) H2D alone: the 4 arrays of one batch, torch non_blocking copies
dsts = [[torch.empty_like(x, device="cuda") for x in inp[k]] for k in range(K)]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for k in range(K):
    e0.record()
    for dd, x in zip(dsts[k], inp[k]):
        dd.copy_(x, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
nbytes = sum(x.numel() * x.element_size() for x in inp[0])
out["h2d_ms_median"] = round(statistics.median(ts), 4)
out["h2d_GBps"] = round(nbytes / (statistics.median(ts) * 1e-3) / 1e9, 2)
out["batch_bytes"] = nbytes
out["is_pinned"] = bool(inp[0][1].is_pinned())


def pipeline(items, dev):
    T_async, T_wait = [], []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for x in items:
        args = [y.cuda(non_blocking=False) for y in x] if dev else [y.numpy() for y in x]
        t = time.perf_counter()
        ctx.step_async(*args, flags=EDGES_UNDIRECTED)
        T_async.append(1e3 * (time.perf_counter() - t))
        if ctx.steps_outstanding >= 2:
            t = time.perf_counter()
            ctx.step_wait()
            T_wait.append(1e3 * (time.perf_counter() - t))
    while ctx.steps_outstanding:
        ctx.step_wait()
    e1.record()
    torch.cuda.synchronize()
    return {"ms_per_step_device": round(e0.elapsed_time(e1) / len(items), 4),
            "ms_per_step_wall": round(1e3 * (time.perf_counter() - t0) / len(items), 4),
            "step_async_host_ms_median": round(statistics.median(T_async), 4),
            "step_wait_host_ms_median": round(statistics.median(T_wait), 4)}


def sync_dev(items, flush):
    """bench.py's device leg: append (device pointers) + exploit + best_path."""
    fl = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ts, ex, tap, tbp = [], [], [], []
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for x in items:
        if flush:
            fl.zero_()
        e0.record()
        np_ = ctx.append(*x, flags=EDGES_UNDIRECTED)
        ea.record()
        if np_ > 0:
            ex.append(ctx.exploit().device_ms)
        eb.record()
        ctx.best_path()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        tap.append(e0.elapsed_time(ea))
        tbp.append(eb.elapsed_time(e1))
    return {"ms_per_step": round(statistics.mean(ts), 4), "exploit_ms_mean": round(statistics.mean(ex), 4),
            "append_ms_mean": round(statistics.mean(tap), 4), "best_path_ms_mean": round(statistics.mean(tbp), 4)}


def pipe_dev(items):
    torch.cuda.synchronize()
    e0.record()
    ex = []
    for x in items:
        ctx.step_async(*x, flags=EDGES_UNDIRECTED)
        if ctx.steps_outstanding >= 2:
            r = ctx.step_wait()
            if r.replanned:
                ex.append(r.stats.device_ms)
    while ctx.steps_outstanding:
        r = ctx.step_wait()
        if r.replanned:
            ex.append(r.stats.device_ms)
    e1.record()
    torch.cuda.synchronize()
    return {"ms_per_step": round(e0.elapsed_time(e1) / len(items), 4),
            "exploit_ms_mean": round(statistics.mean(ex), 4)}


out["pipeline_host_inputs_first"] = pipeline(inp[:K], dev=False)
if os.environ.get("PROBE_ONLY"):
    dev_b = [[y.cuda() for y in x] for x in inp[K:K + 10]]
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("B")
    print(json.dumps(sync_dev(dev_b, os.environ["PROBE_ONLY"] == "A")))
    torch.cuda.nvtx.range_pop()
    sys.exit(0)
for name, fn in (("A_sync_dev_flush", lambda it: sync_dev(it, True)),
                 ("B_sync_dev_noflush", lambda it: sync_dev(it, False)),
                 ("C_pipe_dev", pipe_dev)):
    items = [[y.cuda() for y in x] for x in inp[K:K + 10]] if False else None
    out[name] = None
K2 = 10
blocks = [inp[K + i * K2: K + (i + 1) * K2] for i in range(4)]
dev_blocks = [[[y.cuda() for y in x] for x in b] for b in blocks]
torch.cuda.synchronize()
out["A_sync_dev_flush"] = sync_dev(dev_blocks[0], True)
out["B_sync_dev_noflush"] = sync_dev(dev_blocks[1], False)
out["C_pipe_dev"] = pipe_dev(dev_blocks[2])
out["D_pipe_host"] = pipeline(blocks[3], dev=False)
print(json.dumps(out))
