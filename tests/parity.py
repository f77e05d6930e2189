"""Helpers for GPU-vs-oracle parity tests (test infrastructure).

The bar (BASELINE.json north_star): g within 1e-9 relative, parent bit-exact
where competing costs differ by more than that, promising set and best goal
bit-exact.  Under readings R2/R3/R6/R9 with one IEEE add per tree edge the
CUDA path reproduces the oracle bit for bit, so these helpers assert the
stronger bitwise equality of g, parent, pc and b and the equality of every
counter of the exploit statistics.
"""
import numpy as np

STAT_KEYS = ("iterations", "evaluations", "relaxations", "eval_visits", "max_level", "promising",
             "stalled")


def first_diff(a, b, n=5):
    idx = np.nonzero(a != b)[0][:n]
    return [(int(i), a[i], b[i]) for i in idx]


def assert_same_state(gpu, orc, where=""):
    gp, gg, gpc, gb = gpu.state()
    op, og, opc, ob = orc.state()
    assert gg.size == og.size, where
    gbits, obits = gg.view(np.uint64), og.view(np.uint64)
    assert np.array_equal(gbits, obits), f"{where} g differs at {first_diff(gg, og)}"
    assert np.array_equal(gp, op), f"{where} parent differs at {first_diff(gp, op)}"
    assert np.array_equal(gpc.view(np.uint64), opc.view(np.uint64)), \
        f"{where} pc differs at {first_diff(gpc, opc)}"
    assert np.array_equal(gb, ob), f"{where} b differs at {first_diff(gb, ob)}"


def assert_same_stats(gs, os_, where=""):
    for k in STAT_KEYS:
        assert getattr(gs, k) == getattr(os_, k), f"{where} stat {k}: gpu {getattr(gs, k)} " \
                                                  f"oracle {getattr(os_, k)}"
    assert np.float64(gs.last_delta_g).view(np.uint64) == \
        np.float64(os_.last_delta_g).view(np.uint64), where


def dual_replay(gpu, orc, graph, S, n_stop=None, undirected=True, check_every=1, final=True):
    """Replay BE-RRT# batches (Alg. 3) into both contexts; compare after each exploit."""
    from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED, batches
    n_stop = graph.n if n_stop is None else n_stop
    flags = EDGES_UNDIRECTED if undirected else 0
    k_ex = 0
    for k, (a, b) in enumerate(batches(n_stop, S)):
        src, dst, cost = graph.batch(a, b, directed=not undirected)
        pg = gpu.append(graph.h[a:b], src, dst, cost, flags=flags)
        po = orc.append(graph.h[a:b], src, dst, cost, flags=flags)
        assert pg == po, f"batch {k}: n_new_promising gpu {pg} oracle {po}"
        if po > 0:
            gs, os_ = gpu.exploit(), orc.exploit()
            assert_same_stats(gs, os_, f"batch {k} [{a},{b})")
            if k_ex % check_every == 0:
                assert_same_state(gpu, orc, f"batch {k} [{a},{b})")
            k_ex += 1
    if final:
        gs, os_ = gpu.exploit(), orc.exploit()
        assert_same_stats(gs, os_, "final")
    assert_same_state(gpu, orc, "final")
    gpath, gcost, ggoal = gpu.best_path_goal()
    opath, ocost, ogoal = orc.best_path_goal()
    assert np.array_equal(gpath, opath) and gcost == ocost and ggoal == ogoal
    return k_ex
