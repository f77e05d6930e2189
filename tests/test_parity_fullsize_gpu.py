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
from parity import RankGroup, assert_same_state, assert_same_stats

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nranks", [1, 2])
def test_bench_workload_full_size_parity(nranks):
    """nranks = 2: the same at P = 2 -- an in-process group (the sharded
    kernels, owner-partitioned in-edge store, record all-gather as device
    copies; tests/test_parity_group_gpu.py) on one GPU."""
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
    kw = dict(h_root=g.h_root(), stream=stream, vertex_capacity=g.n + 1024,
              edge_capacity=int(2.4 * g.off[-1]) + 4096)
    gpu = pirrt.Context(**kw) if nranks == 1 else RankGroup(pirrt, nranks, **kw)
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


@pytest.mark.parametrize("k0", [0, 180])
def test_gamma_star_7d_full_size_handoff_parity(k0):
    """configs[3] at its full size and the headline radius: 7-D, 200k
    vertices, gamma* (mean degree ~1,250, ~2.3e8 directed edges, 30 boxes),
    built on the GPU by the device Extend in BE-RRT# batches of 1000 with the
    Alg. 3 guard.  At batch k0 (180 = 20 batches before the end; 0 = from
    the empty graph, so the one Replan on this workload that changes the
    policy -- batch 0: 3 PI iterations, 2 Evaluates; the gamma* radius in
    7-D is ~0.8 at n = 1000 and the best path never improves after it, see
    tools/gstar7_probe.py -- is compared too), the stored graph
    (pirrt_get_in_edges) and the policy state are handed to the oracle
    (append + set_policy); then every remaining batch runs on both -- the
    oracle is fed the edges the device Extend stored for that batch -- and
    every Replan is compared bitwise: g, parent, pc, b, every counter, the
    best path at the end."""
    from paper_2003_04920_b200 import pirrt
    from paper_2003_04920_b200.berrt import batches
    d, n, S, boxes = 7, 200_000, 1000, 30
    gm = gen.gamma_star(d)
    pts, bx = gen.points(d, n, boxes, seed=gen.seed_of("fullsize-gstar", d, n))
    h_root = float(np.sqrt(((pts[0] - pts[1]) ** 2).sum()))
    # h as the device Extend computes it: squared differences summed in
    # coordinate order, IEEE sqrt
    s2 = np.zeros(n)
    for k in range(d):
        u = pts[:, k] - pts[1, k]
        s2 = s2 + u * u
    h = np.sqrt(s2)
    gpu = pirrt.Context(h_root=h_root, vertex_capacity=n + 1024, edge_capacity=int(2.2 * 700 * n))
    gpu.set_world(d, bx, pts[0], pts[1], gm)
    bl = list(batches(n, S))
    for lo, hi in bl[:k0]:
        if gpu.extend(pts[lo:hi])[0] > 0:
            gpu.exploit()
    # hand-off
    n0 = gpu.n
    parent, g, _, b = gpu.state()
    off, src, cost = gpu.in_edges()
    assert off[-1] == gpu.n_edges
    dst = np.repeat(np.arange(n0, dtype=np.int32), np.diff(off))
    orc = Oracle(h_root=h_root)
    if n0 > 2:
        orc.append(h[2:n0], src, dst, cost)
        orc.set_policy(parent, g, b)
    del src, dst, cost, off
    assert_same_state(gpu, orc, "after hand-off")
    # the remaining batches: the device Extend, then the oracle fed the
    # edges it stored (those touching the batch's new vertices)
    replans = evals = 0
    for k, (lo, hi) in enumerate(bl[k0:k0 + 20]):
        n_old = gpu.n
        pg = gpu.extend(pts[lo:hi])[0]
        n_new = gpu.n
        off, src, cost = gpu.in_edges()
        dst = np.repeat(np.arange(n_new, dtype=np.int32), np.diff(off))
        sel = (src >= n_old) | (dst >= n_old)
        po = orc.append(h[n_old:n_new], src[sel], dst[sel], cost[sel])
        del src, dst, cost, off, sel
        assert pg == po, f"batch {k0 + k}: promising {pg} vs {po}"
        if po > 0:
            st = orc.exploit()
            assert_same_stats(gpu.exploit(), st, f"batch {k0 + k}")
            replans += 1
            evals += st.evaluations
        assert_same_state(gpu, orc, f"batch {k0 + k}")
    gp, gc, gg = gpu.best_path_goal()
    op, oc, og = orc.best_path_goal()
    assert np.array_equal(gp, op) and gc == oc and gg == og
    print(f"gamma* 7-D: hand-off at n={n0}, {n_old} -> {n_new} vertices, {gpu.n_edges} directed edges, "
          f"{replans} Replans, {evals} Evaluates compared, path cost {gc:.6f}")
    assert replans > 0 and (k0 == 180) == (n_new == n)


def test_gamma_star_1m_cold_solve_full_size_parity():
    """The bench line's gamma* cold solve at its full size (bench.py
    gamma_star_record, same seed): configs[2]'s 6-D 1M samples, 20 boxes,
    radius gamma* (~1.1e9 directed edges), every vertex added by the device
    Extend with no Replan in between, then one Replan from that state.  The
    stored graph and the Extend-relaxed state are handed to the oracle, both
    run the cold Replan, and g, parent, pc, b, every counter and the best path
    are compared bitwise.  Host memory ~45 GB, a few minutes."""
    import time
    import torch
    from paper_2003_04920_b200 import pirrt
    d, n, boxes, seed = 6, 1_000_000, 20, 0
    gm = gen.gamma_star(d)
    pts, bx = gen.points(d, n, boxes, seed=gen.seed_of("cfg3_gstar", d, n, boxes, seed))
    h_root = float(np.sqrt(((pts[0] - pts[1]) ** 2).sum()))
    gpu = pirrt.Context(h_root=h_root, vertex_capacity=n + 1024, edge_capacity=int(2.2 * 600 * n))
    gpu.set_world(d, bx, pts[0], pts[1], gm)
    dpts = torch.from_numpy(pts).cuda()
    for lo in range(2, n, 131072):
        gpu.extend(dpts[lo:min(n, lo + 131072)])
    del dpts
    s2 = np.zeros(n)
    for k in range(d):
        u = pts[:, k] - pts[1, k]
        s2 = s2 + u * u
    h = np.sqrt(s2)
    t0 = time.perf_counter()
    parent, g, _, b = gpu.state()
    off, src, cost = gpu.in_edges()
    m = int(off[-1])
    assert m == gpu.n_edges and m > 1e9
    dst = np.repeat(np.arange(n, dtype=np.int32), np.diff(off))
    del off
    orc = Oracle(h_root=h_root)
    orc.append(h[2:], src, dst, cost)
    del src, dst, cost
    orc.set_policy(parent, g, b)
    assert_same_state(gpu, orc, "after hand-off")
    t1 = time.perf_counter()
    st = orc.exploit()
    t2 = time.perf_counter()
    sg = gpu.exploit()
    assert_same_stats(sg, st, "cold solve")
    assert_same_state(gpu, orc, "cold solve")
    gp, gc, gg = gpu.best_path_goal()
    op, oc, og = orc.best_path_goal()
    assert np.array_equal(gp, op) and gc == oc and gg == og
    print(f"gamma* 6-D 1M cold solve: {m} directed edges, iterations={st.iterations} "
          f"evaluations={st.evaluations} relaxations={st.relaxations}; GPU {sg.device_ms:.2f} ms, "
          f"oracle {t2 - t1:.1f} s (hand-off {t1 - t0:.1f} s); path cost {gc:.6f}")


def test_cfg4_10m_sharded_cold_solve_full_size_parity():
    """configs[4] at its full size: the 10M-vertex 6-D gamma_k RRG (20 boxes)
    built by the device Extend in S = 65536 batches, as bench.py's sharded
    leg builds it, then its cold solve (bench.py main_sharded's `cold`
    sub-record) three ways: the oracle (state and stored graph handed over
    from a one-rank context), that context, and the sharded kernels as
    an in-process group of P = 2 on this GPU (vertex v's Improve on rank v mod 2,
    record all-gather as device copies).  g, parent, pc, b, every counter and
    the best path compared bitwise; the group's per-rank relaxation shares
    sum to the oracle's count."""
    import time
    import torch
    from paper_2003_04920_b200 import pirrt
    d, n, S, boxes = 6, 10_000_000, 65536, 20
    gm = gen.gamma_k(d)
    pts, bx = gen.points(d, n, boxes, seed=gen.seed_of("fullsize-cfg4", d, n, boxes))
    h_root = float(np.sqrt(((pts[0] - pts[1]) ** 2).sum()))
    dpts = torch.from_numpy(pts).cuda()

    def build(c):
        c.set_world(d, bx, pts[0], pts[1], gm)
        for lo in range(2, n, S):
            c.extend(dpts[lo:min(n, lo + S)])
        return c

    one = build(pirrt.Context(h_root=h_root, vertex_capacity=n + 1024, edge_capacity=int(2.2 * 45 * n)))
    s2 = np.zeros(n)
    for k in range(d):
        u = pts[:, k] - pts[1, k]
        s2 = s2 + u * u
    h = np.sqrt(s2)
    t0 = time.perf_counter()
    parent, g, _, b = one.state()
    off, src, cost = one.in_edges()
    m = int(off[-1])
    assert m == one.n_edges
    dst = np.repeat(np.arange(n, dtype=np.int32), np.diff(off))
    del off
    orc = Oracle(h_root=h_root)
    orc.append(h[2:], src, dst, cost)
    del src, dst, cost
    orc.set_policy(parent, g, b)
    assert_same_state(one, orc, "after hand-off")
    t1 = time.perf_counter()
    st = orc.exploit()
    t2 = time.perf_counter()
    op, oc, og = orc.best_path_goal()

    def check(c, name):
        assert_same_stats(c.exploit(), st, f"cold solve, {name}")
        assert_same_state(c, orc, f"cold solve, {name}")
        cp, cc, cg = c.best_path_goal()
        assert np.array_equal(cp, op) and cc == oc and cg == og

    check(one, "one rank")
    one.close()
    del one
    # the group: P stores on this GPU, each sized for the graph just built (P
    # = 4 does not fit one GPU's memory at this size; tests/
    # test_parity_group_gpu.py covers P = 3, 4 at smaller sizes)
    for P in (2,):
        grp = build(RankGroup(pirrt, P, h_root=h_root, vertex_capacity=n + 1024, edge_capacity=int(1.3 * m)))
        check(grp, f"P = {P}")
        for c in grp.ranks:
            c.close()
        del grp
    print(f"configs[4] 10M cold solve: {m} directed edges, iterations={st.iterations} "
          f"evaluations={st.evaluations} relaxations={st.relaxations}; oracle {t2 - t1:.1f} s "
          f"(hand-off {t1 - t0:.1f} s)")
