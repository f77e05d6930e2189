"""Walk-up / traversal split of the incremental Evaluate at the bench
workload (needs a library built with -DPIRRT_WALK_TRACE=1; device printf).
    bash tools/build_variant.sh walk -DPIRRT_WALK_TRACE=1
    PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_walk.so python tools/walk_probe.py"""
import os
import sys
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
n0 = a.n - 6 * a.S
ctx = pirrt.Context(h_root=g.h_root(), vertex_capacity=g.n + 1024, edge_capacity=int(2.4 * g.off[-1]) + 4096)
for lo, hi in batches(n0, a.S):
    if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        ctx.exploit()
os.environ["PIRRT_DEBUG"] = "1"
for k in range(6):
    lo, hi = n0 + k * a.S, n0 + (k + 1) * a.S
    if ctx.append(g.h[lo:hi], *g.batch(lo, hi, directed=False), flags=EDGES_UNDIRECTED) > 0:
        st = ctx.exploit()
        print(f"exploit {k}: {st.device_ms:.3f} ms, {st.iterations} it, {st.evaluations} ev", flush=True)
    torch.cuda.synchronize()
