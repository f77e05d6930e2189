"""Per-level trace of exploits at the bench workload.

Run with a library built with -DPIRRT_LEVEL_TRACE=1 (PIRRT_LIB=...); the
kernel prints one line per BFS level when PIRRT_DEBUG=1.

    PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/level_probe.py
"""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402
from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED, replay  # noqa: E402

a = types.SimpleNamespace(d=6, n=1_000_000, S=4096, gamma="k", boxes=20, seed=0, warmup=3,
                          steps=10, graph_cache=os.environ.get("GRAPH_CACHE"))
g, gm, _ = bench.make_graph(a, 0, 1)
S = a.S
ctx = pirrt.Context(h_root=g.h_root(), vertex_capacity=g.n + 1024,
                    edge_capacity=int(2.4 * g.off[-1]) + 4096)
n0 = a.n - 4 * S
replay(ctx, g, S, n_stop=n0, final=False)
for k in range(4):
    lo, hi = n0 + k * S, n0 + (k + 1) * S
    s, d, c = g.batch(lo, hi, directed=False)
    nprom = ctx.append(g.h[lo:hi], s, d, c, flags=EDGES_UNDIRECTED)
    if k >= 2:
        os.environ["PIRRT_DEBUG"] = "1"
    print(f"== batch {k} n={hi} nprom={nprom}", flush=True)
    st = ctx.exploit()
    torch.cuda.synchronize()
    print(f"== stats it={st.iterations} ev={st.evaluations} prom={st.promising} "
          f"visits={st.eval_visits} scanned={st.eval_scanned} relax={st.relaxations} "
          f"device_ms={st.device_ms:.3f} improve_ms={st.improve_ms:.3f} "
          f"evaluate_ms={st.evaluate_ms:.3f} barriers={st.barriers} max_level={st.max_level}",
          flush=True)
    os.environ.pop("PIRRT_DEBUG", None)
