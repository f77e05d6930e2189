"""Append phase timeline at the bench workload (configs[2], S = 4096, device
pointers): %globaltimer per phase of k_append_fused (DevCtl::app_ns, lead
thread, pirrt_debug_append_phases), averaged over K appends, plus the host
time per append call and the fold share.
    python tools/append_probe.py [K]"""
import ctypes as C
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

K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
a = types.SimpleNamespace(workload="cfg3", d=6, n=1_000_000, S=4096, gamma="k", boxes=20, seed=0,
                          warmup=0, steps=20, graph_cache="/tmp/g1m_bench.npz")
g, gm, _ = bench.make_graph(a, 0, 1)
S = a.S
n0 = a.n - K * S
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = pirrt.Context(h_root=g.h_root(), stream=s, vertex_capacity=g.n + 1024,
                    edge_capacity=int(2.4 * g.off[-1]) + 4096)
for lo, hi in batches(n0, S):
    if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        ctx.exploit()
lib = pirrt._lib
lib.pirrt_debug_append_phases.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 12)()


def phases():
    lib.pirrt_debug_append_phases(ctx._h, buf, 12)
    return np.array(list(buf), np.float64)


dev = []
for k in range(K):
    lo, hi = n0 + k * S, n0 + (k + 1) * S
    sb, db, cb = g.batch(lo, hi, directed=False)
    dev.append([torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (g.h[lo:hi], sb, db, cb)])
torch.cuda.synchronize()
p0 = phases()
host = []
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
dev_ms = []
for x in dev:
    t = time.perf_counter()
    ev[0].record()
    nprom = ctx.append(*x, flags=EDGES_UNDIRECTED)
    ev[1].record()
    host.append(1e3 * (time.perf_counter() - t))
    torch.cuda.synchronize()
    dev_ms.append(ev[0].elapsed_time(ev[1]))
    if nprom > 0:
        ctx.exploit()
p1 = phases()
d = (p1 - p0)
n_app = d[9]
names = ["validate", "old_lengths", "histogram", "scan_partials", "row_offsets", "old_delta_copy",
         "scatter_init", "local_relaxation", "promising"]
out = {"appends": int(n_app),
       "us_per_append": {nm: round(d[i] / n_app / 1e3, 2) for i, nm in enumerate(names)},
       "kernel_us_sum": round(d[:9].sum() / n_app / 1e3, 2),
       "block0_us": {"p4_chunk_copy": round(d[10] / n_app / 1e3, 2),
                     "p4_cursors": round(d[11] / n_app / 1e3, 2)},
       "append_call_ms": {"host_median": round(statistics.median(host), 4),
                          "device_event_mean": round(statistics.mean(dev_ms), 4),
                          "device_event_median": round(statistics.median(dev_ms), 4),
                          "device_event_max": round(max(dev_ms), 4)}}
print(json.dumps(out))
