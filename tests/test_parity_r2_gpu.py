"""GPU parity for the loop-control cases and the incremental Evaluate.

* The hand-built R13 / epsilon states of tests/test_oracle_loop_pins.py
  (their expected values are derived by hand there) through the C ABI.
* epsilon > 0 on BE-RRT# replays (R5: the last Improve's changes are kept
  without re-evaluation, and the next exploit starts from them -- the
  incremental Evaluate's dirty set carries over between exploits).
* Duplicate edges without VALIDATE (a child reached through two out-row
  entries is visited once).
* The incremental Evaluate against the full one and the oracle, with every
  counter (eval_visits, max_level are the full traversal's, computed from
  child counts and depths), and the share of Evaluates that ran incrementally.
Run on a B200: -m gpu.
"""
import numpy as np
import pytest

import gen
from oracle import EDGES_UNDIRECTED, PRUNE_OFF, Oracle
from parity import assert_same_edge_set, assert_same_state, assert_same_stats, dual_replay
from test_oracle_loop_pins import chain_oracle, eps_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2003_04920_b200 import pirrt
    return pirrt


def gpu_chain(P, h, edges, parent, g, b, eps=0.0):
    ctx = P.Context(h_root=h[0], h_goal=h[1], epsilon=eps)
    src = np.array([e[0] for e in edges], np.int32)
    dst = np.array([e[1] for e in edges], np.int32)
    cost = np.array([e[2] for e in edges], np.float64)
    ctx.append(np.array(h[2:], np.float64), src, dst, cost)
    ctx.set_policy(np.array(parent, np.int32), np.array(g, np.float64), np.array(b, np.uint8))
    return ctx


CASES = {
    "r13_g": ([0.0, 0.0, 0.0], [(0, 2, 1.0), (2, 1, 1.0)], [-1, 2, 0], [0.0, 10.0, 5.0], [0, 0, 1]),
    "r13_b": ([0.0, 0.0, 100.0, 0.0, 0.0], [(0, 2, 1.0), (2, 3, 1.0), (0, 4, 1.0), (0, 1, 10.0)],
              [-1, 0, 0, 2, 0], [0.0, 10.0, 1.0, 5.0, 1.0], [0, 0, 0, 1, 0]),
    "r13_stall": ([0.0, 0.0, 5.0], [(0, 2, 1.0), (2, 1, 1.0)], [-1, 2, 0], [0.0, 3.0, 1.0], [0, 0, 0]),
    "r13_parent": ([0.0, 0.0, 100.0], [(0, 2, 1.0), (2, 1, 1.0), (0, 1, 10.0)], [-1, 0, 0],
                   [0.0, 10.0, 1.0], [0, 0, 0]),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_r13_hand_cases(P, case):
    h, edges, parent, g, b = CASES[case]
    gpu = gpu_chain(P, h, edges, parent, g, b)
    orc = chain_oracle(h, edges, parent, g, b)
    for _ in range(2):                    # and once more from the converged state
        assert_same_stats(gpu.exploit(), orc.exploit(), case)
        assert_same_state(gpu, orc, case)


@pytest.mark.parametrize("eps", [8.0, 7.99, 0.0])
def test_epsilon_hand_case(P, eps):
    h = [0.0, 0.0, 0.0, 0.0]
    edges = [(0, 2, 1.0), (0, 3, 0.25), (3, 2, 0.25), (2, 1, 1.0), (0, 1, 10.0)]
    parent, g, b = [-1, 0, 0, 0], [0.0, 10.0, 1.0, 0.25], [0, 0, 1, 1]
    gpu = gpu_chain(P, h, edges, parent, g, b, eps=eps)
    orc = eps_oracle(eps)
    for _ in range(2):
        assert_same_stats(gpu.exploit(), orc.exploit(), f"eps {eps}")
        assert_same_state(gpu, orc)


@pytest.mark.parametrize("d,n,S,eps,inc", [(2, 4000, 40, 1e-3, None), (2, 4000, 40, 1e-2, "0"),
                                           (6, 12000, 500, 2e-3, None), (4, 8000, 1, 5e-3, None),
                                           (6, 12000, 500, 2e-3, "imp2")])
def test_epsilon_replay(P, monkeypatch, d, n, S, eps, inc):
    if inc == "imp2":
        monkeypatch.setenv("PIRRT_INC_IMPROVE", "2")
    elif inc:
        monkeypatch.setenv("PIRRT_INC_MAX", inc)
    r = gen.rrg(d, n, gen.gamma_star(d) if d == 2 else gen.gamma_k(d), n_boxes=10,
                seed=gen.seed_of("eps", d, S))
    gpu = P.Context(h_root=r.h_root(), epsilon=eps)
    orc = Oracle(h_root=r.h_root(), epsilon=eps)
    dual_replay(gpu, orc, r, S, n_stop=min(n, 2 + 300 * S))


@pytest.mark.parametrize("inc", [None, "0", "imp2"])
def test_duplicate_edges_without_validate(P, monkeypatch, inc):
    # every edge staged twice (and some three times): a child is reached
    # through several out-row entries of its parent and must be visited once
    if inc == "imp2":
        monkeypatch.setenv("PIRRT_INC_IMPROVE", "2")
    elif inc:
        monkeypatch.setenv("PIRRT_INC_MAX", inc)
    r = gen.rrg(3, 3000, gen.gamma_k(3), n_boxes=8, seed=gen.seed_of("dups"))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    from paper_2003_04920_b200.berrt import batches
    for k, (a, b) in enumerate(batches(r.n, 100)):
        s, t, c = r.batch(a, b, directed=False)
        rep = np.concatenate([np.arange(s.size)] * 2 + [np.arange(0, s.size, 3)])
        args = (r.h[a:b], s[rep], t[rep], c[rep])
        assert gpu.append(*args, flags=EDGES_UNDIRECTED) == orc.append(*args, flags=EDGES_UNDIRECTED)
        assert_same_stats(gpu.exploit(), orc.exploit(), f"batch {k}")
        assert_same_state(gpu, orc, f"batch {k}")
    # the stored multiset keeps every duplicate
    s, t, c = r.batch(2, r.n, directed=False)
    rows = []
    for a, b in batches(r.n, 100):
        lo, hi = np.searchsorted(t, a), np.searchsorted(t, b)
        rep = np.concatenate([np.arange(lo, hi)] * 2 + [np.arange(lo, hi)[0::3]])
        rows.append(rep)
    rep = np.concatenate(rows)
    assert_same_edge_set(gpu, np.concatenate([s[rep], t[rep]]), np.concatenate([t[rep], s[rep]]),
                         np.concatenate([c[rep], c[rep]]), "duplicates")


@pytest.mark.parametrize("d,n,S,gamma,flags", [(6, 20000, 256, "k", 0), (2, 8000, 1, "star", 0),
                                               (7, 10000, 1000, "k", 0), (3, 6000, 60, "k", PRUNE_OFF)])
def test_incremental_evaluate_is_used_and_exact(P, d, n, S, gamma, flags):
    """Default settings: most per-batch Evaluates run incrementally; results
    and every counter equal the oracle's (dual_replay), and eval_work (the
    visits actually made) is below eval_visits (the full traversal's)."""
    gm = gen.gamma_k(d) if gamma == "k" else gen.gamma_star(d)
    r = gen.rrg(d, n, gm, n_boxes=10, seed=gen.seed_of("inc", d, S))
    gpu = P.Context(h_root=r.h_root(), flags=flags)
    orc = Oracle(h_root=r.h_root(), flags=flags)
    stats = []

    class Spy:
        def __getattr__(self, k):
            return getattr(gpu, k)

        def exploit(self):
            st = gpu.exploit()
            stats.append(st)
            return st

    dual_replay(Spy(), orc, r, S, n_stop=min(n, 2 + 400 * S))
    inc = sum(s.inc_evaluations for s in stats)
    full = sum(s.full_evaluations for s in stats)
    assert inc + full == sum(s.evaluations for s in stats)
    assert inc > full, (inc, full)
    assert sum(s.eval_work for s in stats) < sum(s.eval_visits for s in stats)
    if not flags:
        # incremental Improves too (PRUNE_OFF always runs the full one)
        assert sum(s.inc_improves for s in stats) > 0
        assert sum(s.relax_work for s in stats) < sum(s.relaxations for s in stats)


@pytest.mark.parametrize("mode", ["0", "2"])
@pytest.mark.parametrize("d,n,S,gamma,goals", [(6, 20000, 256, "k", False), (2, 8000, 1, "star", False),
                                               (3, 8000, 100, "k", True), (7, 10000, 1000, "star", False)])
def test_incremental_improve_modes(P, monkeypatch, mode, d, n, S, gamma, goals):
    """PIRRT_INC_IMPROVE=0 (every Improve full) and 2 (incremental whenever
    its certificate is valid): identical results and counters to the oracle."""
    monkeypatch.setenv("PIRRT_INC_IMPROVE", mode)
    gm = gen.gamma_k(d) if gamma == "k" else gen.gamma_star(d)
    r = gen.rrg(d, n, gm, n_boxes=10, seed=gen.seed_of("inc-imp", d, S))
    kw = {}
    orc = Oracle(h_root=r.h_root())
    if goals:
        ids = (np.nonzero(r.h[2:] <= 0.15)[0] + 2).astype(np.int32)
        kw["goals"] = ids
        orc.set_goals(ids)
    gpu = P.Context(h_root=r.h_root(), **kw)
    dual_replay(gpu, orc, r, S, n_stop=min(n, 2 + 300 * S))


def test_incremental_after_set_policy_and_given_policy(P):
    """set_policy and an append with a given policy force the next Evaluate
    to be full; the following ones may be incremental again."""
    r = gen.rrg(4, 6000, gen.gamma_k(4), n_boxes=8, seed=gen.seed_of("inc-sp"))
    gpu, orc = P.Context(h_root=r.h_root()), Oracle(h_root=r.h_root())
    dual_replay(gpu, orc, r, 200, n_stop=3000, final=True)
    parent, g, pc, b = orc.state()
    gpu.set_policy(parent, g, b)
    orc.set_policy(parent, g, b)
    st = gpu.exploit()
    assert_same_stats(st, orc.exploit())
    # a batch with a given policy (the oracle's own local relaxation result)
    from paper_2003_04920_b200.berrt import batches
    for (a, bb) in batches(3600, 300, start=3000):
        s, t, c = r.batch(a, bb, directed=False)
        probe = Oracle(h_root=r.h_root())
        probe.append(r.h[2:bb], *r.batch(2, bb, directed=False), flags=EDGES_UNDIRECTED)
        pp, gg, _, _ = probe.state()
        for ctx in (gpu, orc):
            ctx.append(r.h[a:bb], s, t, c, parent_new=pp[a:bb], g_new=gg[a:bb], flags=EDGES_UNDIRECTED)
        gs = gpu.exploit()
        assert gs.full_evaluations >= (1 if gs.evaluations else 0)
        assert_same_stats(gs, orc.exploit())
        assert_same_state(gpu, orc)


@pytest.mark.parametrize("d,n,S,undirected", [(6, 20000, 256, True), (3, 6000, 1, False),
                                              (2, 30000, 4096, True)])
def test_stored_edge_set_after_appends_and_folds(P, d, n, S, undirected):
    """pirrt_get_in_edges after a BE-RRT# replay (many appends, delta folds):
    the stored graph equals the generator's directed edge multiset element by
    element (src, dst, cost bits)."""
    r = gen.rrg(d, n, gen.gamma_k(d), n_boxes=10, seed=gen.seed_of("edges", d, S))
    gpu = P.Context(h_root=r.h_root())
    from paper_2003_04920_b200.berrt import batches
    fl = EDGES_UNDIRECTED if undirected else 0
    for a, b in batches(r.n, S):
        gpu.append(r.h[a:b], *r.batch(a, b, directed=not undirected), flags=fl)
    assert gpu.n_edges == 2 * r.n_pairs
    assert_same_edge_set(gpu, *r.batch(2, r.n, directed=True), "replay")


@pytest.mark.parametrize("mode", ["1", "2"])
def test_edges_between_old_vertices(P, monkeypatch, mode):
    """Appends whose edges join two old vertices (an old vertex gains an
    in-edge without any new vertex next to it): the incremental Improve's
    sources do not cover it, so such an append forces the next Improve to be
    a full one.  Each batch adds its vertices with half of their edges; the
    other half follows as a batch with no new vertex, then an exploit."""
    monkeypatch.setenv("PIRRT_INC_IMPROVE", mode)
    r = gen.rrg(3, 6000, gen.gamma_k(3), n_boxes=6, seed=gen.seed_of("old-old"))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    from paper_2003_04920_b200.berrt import batches
    U = EDGES_UNDIRECTED
    for k, (a, b) in enumerate(batches(r.n, 200)):
        s, t, c = r.batch(a, b, directed=False)
        cut = int(np.searchsorted(t, (a + b) // 2))
        pg = gpu.append(r.h[a:b], s[:cut], t[:cut], c[:cut], flags=U)
        assert pg == orc.append(r.h[a:b], s[:cut], t[:cut], c[:cut], flags=U)
        if pg > 0:
            assert_same_stats(gpu.exploit(), orc.exploit(), f"batch {k}")
        z = np.zeros(0)
        assert gpu.append(z, s[cut:], t[cut:], c[cut:], flags=U) == 0
        orc.append(z, s[cut:], t[cut:], c[cut:], flags=U)
        assert_same_stats(gpu.exploit(), orc.exploit(), f"batch {k} (old-old edges)")
    assert_same_state(gpu, orc, "final")


@pytest.mark.parametrize("env", [{"PIRRT_SMALL_GRID": "0"}, {"PIRRT_SMALL_GRID": "7"},
                                 {"PIRRT_INC_VALIDATE": "1"},
                                 {"PIRRT_SMALL_GRID": "1", "PIRRT_INC_VALIDATE": "1"}])
@pytest.mark.parametrize("d,n,S", [(6, 12000, 500), (2, 8000, 1)])
def test_prebuilt_task_lists_and_small_grid(P, monkeypatch, env, d, n, S):
    """The incremental Evaluate builds the next Improve's task list (no
    discovery phase), also through the validation fixpoint's recount
    (PIRRT_INC_VALIDATE); small exploits run on the one-block-per-SM grid
    (default), on 7 or 1 blocks, or on the full grid (0): identical to the
    oracle, and the incremental Improve is used."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    gm = gen.gamma_k(d) if d > 2 else gen.gamma_star(d)
    r = gen.rrg(d, n, gm, n_boxes=10, seed=gen.seed_of("prebuilt", d, S))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    stats = []
    orig = gpu.exploit

    def rec():
        s = orig()
        stats.append(s)
        return s
    gpu.exploit = rec
    dual_replay(gpu, orc, r, S, n_stop=min(n, 2 + 300 * S))
    assert sum(s.inc_improves for s in stats) > 0


@pytest.mark.parametrize("d,n,S,gamma,pmax", [(6, 30000, 2048, "k", "1000000"), (2, 6000, 1, "star", "0"),
                                              (3, 8000, 300, "k", "1000000"), (2, 6000, 7, "star", "1000000")])
def test_append_prebuilt_first_improve(P, monkeypatch, d, n, S, gamma, pmax):
    """The next exploit's first Improve listed by the append (P8) -- forced on
    for large batches, off for S = 1 -- against the oracle: every counter
    (relaxations = the full Improve's) and the state, bit for bit."""
    monkeypatch.setenv("PIRRT_PREBUILD_MAX", pmax)
    gm = gen.gamma_k(d) if gamma == "k" else gen.gamma_star(d)
    r = gen.rrg(d, n, gm, n_boxes=12, seed=gen.seed_of("prebuild", d, S))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    dual_replay(gpu, orc, r, S, n_stop=min(n, 2 + 400 * S))
