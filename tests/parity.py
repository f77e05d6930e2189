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


def sorted_edges(src, dst, cost):
    """(src, dst, cost bits) rows in lexicographic (dst, src, cost bits) order."""
    src, dst = np.asarray(src, np.int64), np.asarray(dst, np.int64)
    cb = np.asarray(cost, np.float64).view(np.uint64)
    order = np.lexsort((cb, src, dst))
    return src[order], dst[order], cb[order]


def assert_same_edge_set(gpu, src, dst, cost, where=""):
    """The library's stored in-edge store (pirrt_get_in_edges) equals the
    directed multiset (src, dst, cost) element by element (cost bitwise)."""
    off, gs, gc = gpu.in_edges()
    assert off[0] == 0 and np.all(np.diff(off) >= 0), where
    gd = np.repeat(np.arange(off.size - 1, dtype=np.int64), np.diff(off))
    a, b = sorted_edges(gs, gd, gc), sorted_edges(src, dst, cost)
    assert a[0].size == b[0].size, f"{where} {a[0].size} edges stored, expected {b[0].size}"
    for name, x, y in zip(("src", "dst", "cost"), a, b):
        bad = np.nonzero(x != y)[0][:5]
        assert bad.size == 0, f"{where} edge {name} differs at sorted rows {bad.tolist()}"


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


class RankGroup:
    """P contexts of one in-process group (PIRRT_F_LOCAL_GROUP) driven SPMD,
    with the Context interface dual_replay uses: every append goes to every
    rank; exploit() runs pirrt_group_exploit and returns rank 0's stats with
    the per-rank shares (relaxations, improve_set) summed -- after checking
    that every rank reports the same loop counters; state() checks that every
    rank holds the same bits and returns rank 0's."""

    LOOP_KEYS = ("iterations", "evaluations", "eval_visits", "max_level", "promising", "stalled")

    def __init__(self, P, nranks, stream=None, **kw):
        self.P = P
        flags = kw.pop("flags", 0) | P.PIRRT_F_LOCAL_GROUP
        self.ranks = [P.Context(nranks=nranks, rank=r, flags=flags, stream=stream, **kw)
                      for r in range(nranks)]

    @property
    def n(self):
        return self.ranks[0].n

    def append(self, *args, **kw):
        got = [c.append(*args, **kw) for c in self.ranks]
        assert len(set(got)) == 1, got
        return got[0]

    def set_world(self, *args):
        for c in self.ranks:
            c.set_world(*args)

    def extend(self, *args, **kw):
        got = [c.extend(*args, **kw) for c in self.ranks]
        assert len(set(got)) == 1, got
        return got[0]

    def exploit(self):
        import dataclasses
        sts = self.P.group_exploit(self.ranks)
        for k in self.LOOP_KEYS:
            vals = {getattr(s, k) for s in sts}
            assert len(vals) == 1, (k, vals)
        assert len({np.float64(s.last_delta_g).view(np.uint64) for s in sts}) == 1
        return dataclasses.replace(sts[0], relaxations=sum(s.relaxations for s in sts),
                                   improve_set=sum(s.improve_set for s in sts))

    def state(self):
        ref = self.ranks[0].state()
        for c in self.ranks[1:]:
            for name, x, y in zip(("parent", "g", "pc", "b"), c.state(), ref):
                assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)), \
                    f"rank state {name} differs"
        return ref

    def best_path_goal(self):
        return self.ranks[0].best_path_goal()
