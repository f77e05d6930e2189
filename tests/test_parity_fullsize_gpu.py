"""Parity at BASELINE.json's full size, in the launch configuration bench.py
times: configs[2] = 6-D, 1M vertices, gamma_k, 20 boxes, BE-RRT# S=4096 (the
bench workload; same generator seed and the same Context settings).

The GPU replays the history to n0 = 1M - 4 S; its state (parent, g, b) is
handed to the oracle (all edges so far + set_policy, SURVEY.md 8(d) "state
hand-off"); then the next 4 batches run on both and every exploit is compared
element by element -- g bitwise, parent, pc, b, every counter -- plus the
best path.  Run on a B200: -m gpu (about a minute: the 1M-vertex graph)."""
import os
import sys
import types

import numpy as np
import pytest

import gen
from oracle import EDGES_UNDIRECTED, Oracle
from parity import assert_same_state, assert_same_stats

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_workload_full_size_parity():
    import torch
    sys.path.insert(0, ROOT)
    import bench
    from paper_2003_04920_b200 import pirrt
    from paper_2003_04920_b200.berrt import batches
    a = types.SimpleNamespace(workload="cfg3", d=6, n=1_000_000, S=4096, gamma="k", boxes=20, seed=0, warmup=0,
                              steps=2, graph_cache=os.environ.get("PIRRT_FULLSIZE_CACHE", ""))
    g, gm, _ = bench.make_graph(a, 0, 1)
    S = a.S
    n0 = a.n - 4 * S
    stream = torch.cuda.current_stream()
    gpu = pirrt.Context(h_root=g.h_root(), stream=stream, vertex_capacity=g.n + 1024,
                        edge_capacity=int(2.4 * g.off[-1]) + 4096)
    for lo, hi in batches(n0, S):
        s, d_, c = g.batch(lo, hi, directed=False)
        if gpu.append(g.h[lo:hi], s, d_, c, flags=EDGES_UNDIRECTED) > 0:
            gpu.exploit()
    # state hand-off to the oracle
    parent, gv, _, b = gpu.state()
    orc = Oracle(h_root=g.h_root())
    s, d_, c = g.batch(2, n0, directed=False)
    orc.append(g.h[2:n0], s, d_, c, flags=EDGES_UNDIRECTED)
    orc.set_policy(parent, gv, b)
    assert_same_state(gpu, orc, "after hand-off")
    # the next 4 batches on both, device-pointer appends as bench.py does
    for k in range(4):
        lo, hi = n0 + k * S, n0 + (k + 1) * S
        s, d_, c = g.batch(lo, hi, directed=False)
        dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (g.h[lo:hi], s, d_, c)]
        pg = gpu.append(*dev, flags=EDGES_UNDIRECTED)
        po = orc.append(g.h[lo:hi], s, d_, c, flags=EDGES_UNDIRECTED)
        assert pg == po
        if po > 0:
            assert_same_stats(gpu.exploit(), orc.exploit(), f"batch {k}")
        assert_same_state(gpu, orc, f"batch {k}")
    gp, gc, gg = gpu.best_path_goal()
    op, oc, og = orc.best_path_goal()
    assert np.array_equal(gp, op) and gc == oc and gg == og
