"""GPU parity: the CUDA path (through the C ABI) against the serial oracle,
element by element, on identical seeded inputs.  Run on a B200: -m gpu."""
import math

import numpy as np
import pytest

import gen
from oracle import PRUNE_OFF, Oracle
from parity import assert_same_state, assert_same_stats, dual_replay

pytestmark = pytest.mark.gpu
INF = math.inf


@pytest.fixture(scope="module")
def P():
    from paper_2003_04920_b200 import pirrt
    return pirrt


def pair(P, h_root=0.0, flags=0, **kw):
    return P.Context(h_root=h_root, flags=flags, **kw), Oracle(h_root=h_root, flags=flags)


# ------------------------------------------------------------------ worked examples

def test_spec_triangle(P):
    # SPEC S:230/S:239/S:248/S:267 with SPEC vertex 2 as our goal (id 1)
    src = np.array([0, 2, 2, 1, 0, 1], np.int32)
    dst = np.array([2, 0, 1, 2, 1, 0], np.int32)
    cost = np.array([5, 5, 7, 7, 6, 6], np.float64)
    gpu, orc = P.Context(), Oracle()
    for ctx in (gpu, orc):
        ctx.append(np.zeros(1), src, dst, cost)
        ctx.set_policy(np.array([-1, 2, 0], np.int32), np.array([0, 12.0, 5.0]),
                       np.array([0, 1, 0], np.uint8))
    assert_same_state(gpu, orc, "after set_policy")
    gs = gpu.exploit()
    os_ = orc.exploit()
    assert gs.iterations == 2
    assert_same_stats(gs, os_)
    assert_same_state(gpu, orc)
    path, c = gpu.best_path()
    assert path.tolist() == [0, 1] and c == 6.0


@pytest.mark.parametrize("k", [5, 12, 40])
@pytest.mark.parametrize("flags", [0, PRUNE_OFF])
def test_lattice(P, k, flags):
    cells, _, src, dst, cost, h = gen.lattice(k)
    gpu, orc = pair(P, h_root=h[0], flags=flags)
    assert gpu.append(h[2:], src, dst, cost) == orc.append(h[2:], src, dst, cost)
    assert_same_state(gpu, orc, "after append")
    gs, os_ = gpu.exploit(), orc.exploit()
    assert_same_stats(gs, os_)
    assert_same_state(gpu, orc)
    assert gpu.costs()[1] == 2 * (k - 1)


# ------------------------------------------------------------------ random graphs

@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("flags", [0, PRUNE_OFF])
def test_random_graph_single_solve(P, seed, flags):
    n, m = 300 + 97 * seed, 3000 + 500 * seed
    src, dst, cost = gen.random_graph(n, m, seed, max_cost=2.0, integer_costs=(seed % 2 == 1))
    h = np.zeros(n)
    gpu, orc = pair(P, flags=flags)
    assert gpu.append(h[2:], src, dst, cost) == orc.append(h[2:], src, dst, cost)
    assert_same_state(gpu, orc, "after append")
    gs, os_ = gpu.exploit(), orc.exploit()
    assert_same_stats(gs, os_)
    assert_same_state(gpu, orc)


def test_zero_cost_and_ties(P):
    # massive exact ties (integer costs incl. zeros): lowest-id tie-break (R6)
    src, dst, cost = gen.random_graph(500, 8000, 3, integer_costs=True, zero_cost_frac=0.2)
    for flags in (0, PRUNE_OFF):
        gpu, orc = pair(P, flags=flags)
        gpu.append(np.zeros(498), src, dst, cost)
        orc.append(np.zeros(498), src, dst, cost)
        assert_same_stats(gpu.exploit(), orc.exploit())
        assert_same_state(gpu, orc)


# ------------------------------------------------------------------ RRG replays

@pytest.mark.parametrize("S", [1, 7, 100, 998])
def test_config1_2d_1k(P, S):
    # configs[0]: 2-D unit square, no obstacles, 1,000-vertex RRG
    r = gen.rrg(2, 1000, gen.gamma_star(2), seed=gen.seed_of("cfg1", S))
    gpu, orc = pair(P, h_root=r.h_root())
    dual_replay(gpu, orc, r, S)


@pytest.mark.parametrize("S", [1, 64])
def test_config2_shape_clutter(P, S):
    # configs[1] shape (2-D, box clutter, per-sample extension) at 6k vertices
    r = gen.rrg(2, 6000, gen.gamma_star(2), n_boxes=30, seed=gen.seed_of("cfg2", S))
    gpu, orc = pair(P, h_root=r.h_root())
    dual_replay(gpu, orc, r, S, check_every=7 if S == 1 else 1)


@pytest.mark.parametrize("gamma", ["k", "star"])
def test_config3_shape_6d(P, gamma):
    # configs[2] shape: 6-D, BE-RRT# batches, boxes
    gm = gen.gamma_k(6) if gamma == "k" else gen.gamma_star(6)
    r = gen.rrg(6, 20000, gm, n_boxes=20, seed=gen.seed_of("cfg3", gamma))
    gpu, orc = pair(P, h_root=r.h_root())
    dual_replay(gpu, orc, r, 1000)


def test_config4_shape_7d(P):
    r = gen.rrg(7, 8000, gen.gamma_k(7), n_boxes=30, seed=gen.seed_of("cfg4"))
    gpu, orc = pair(P, h_root=r.h_root())
    dual_replay(gpu, orc, r, 500)


def test_cold_solve_prune_off_6d(P):
    r = gen.rrg(6, 30000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("cold"))
    gpu, orc = pair(P, h_root=r.h_root(), flags=PRUNE_OFF)
    dual_replay(gpu, orc, r, r.n)


def test_directed_and_undirected_inputs_agree(P):
    r = gen.rrg(2, 3000, gen.gamma_star(2), n_boxes=10, seed=77)
    g1 = P.Context(h_root=r.h_root())
    g2 = P.Context(h_root=r.h_root())
    from paper_2003_04920_b200.berrt import replay
    replay(g1, r, 250, undirected=True)
    replay(g2, r, 250, undirected=False)
    for x, y in zip(g1.state(), g2.state()):
        assert np.array_equal(x, y)


# ------------------------------------------------------------------ edge cases

def test_empty_append_and_unreachable_goal(P):
    gpu, orc = pair(P)
    for c in (gpu, orc):
        assert c.append(np.zeros(0), np.zeros(0, np.int32), np.zeros(0, np.int32),
                        np.zeros(0)) == 0
        c.append(np.zeros(3), np.array([0, 2], np.int32), np.array([2, 3], np.int32),
                 np.ones(2))
    assert_same_stats(gpu.exploit(), orc.exploit())
    assert_same_state(gpu, orc)
    path, c = gpu.best_path()
    assert path.size == 0 and c == INF


@pytest.mark.parametrize("bad", ["range", "selfloop", "nan", "neg", "h", "negid"])
def test_malformed_append_rejected_state_unchanged(P, bad):
    gpu = P.Context()
    gpu.append(np.zeros(2), np.array([0, 2], np.int32), np.array([2, 3], np.int32), np.ones(2))
    gpu.exploit()
    before = gpu.state()
    src = np.array([0, 3], np.int32); dst = np.array([4, 4], np.int32); cost = np.ones(2)
    h = np.zeros(1)
    if bad == "range":
        dst = np.array([4, 9], np.int32)
    elif bad == "selfloop":
        src = np.array([4, 4], np.int32)
    elif bad == "nan":
        cost = np.array([1.0, np.nan])
    elif bad == "neg":
        cost = np.array([1.0, -1.0])
    elif bad == "negid":
        src = np.array([-3, 0], np.int32)
    else:
        h = np.array([np.inf])
    with pytest.raises(P.PirrtError):
        gpu.append(h, src, dst, cost)
    assert gpu.n == 4
    for x, y in zip(before, gpu.state()):
        assert np.array_equal(x, y)
    # still usable
    gpu.append(np.zeros(1), np.array([0], np.int32), np.array([4], np.int32), np.ones(1))
    assert gpu.n == 5


def test_given_policy_append_and_set_policy(P):
    r = gen.rrg(2, 800, gen.gamma_star(2), seed=12)
    gpu, orc = pair(P, h_root=r.h_root())
    src, dst, cost = r.batch(2, 400)
    orc.append(r.h[2:400], src, dst, cost)
    gpu.append(r.h[2:400], src, dst, cost)
    orc.exploit(); gpu.exploit()
    # next batch with a caller-given policy (the oracle's own local relaxation)
    src, dst, cost = r.batch(400, 800)
    orc2 = Oracle(h_root=r.h_root())
    s0, d0, c0 = r.batch(2, 400)
    orc2.append(r.h[2:400], s0, d0, c0); orc2.exploit()
    orc2.append(r.h[400:800], src, dst, cost)
    p2, g2, _, _ = orc2.state()
    orc.append(r.h[400:800], src, dst, cost, parent_new=p2[400:800], g_new=g2[400:800])
    gpu.append(r.h[400:800], src, dst, cost, parent_new=p2[400:800], g_new=g2[400:800])
    assert_same_state(gpu, orc, "given policy")
    assert_same_stats(gpu.exploit(), orc.exploit())
    assert_same_state(gpu, orc)
    # set_policy round trip
    st = orc.state()
    gpu.set_policy(st[0], st[1], st[3])
    assert_same_state(gpu, orc, "set_policy")


def test_device_pointer_append(P):
    import torch
    r = gen.rrg(2, 2000, gen.gamma_star(2), n_boxes=5, seed=21)
    g1 = P.Context(h_root=r.h_root())
    g2 = P.Context(h_root=r.h_root(), stream=torch.cuda.current_stream())
    from paper_2003_04920_b200.berrt import batches
    for a, b in batches(r.n, 300):
        src, dst, cost = r.batch(a, b, directed=False)
        g1.append(r.h[a:b], src, dst, cost, flags=P.PIRRT_F_EDGES_UNDIRECTED)
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
        g2.append(t(r.h[a:b]), t(src), t(dst), t(cost), flags=P.PIRRT_F_EDGES_UNDIRECTED)
        g1.exploit(); g2.exploit()
    for x, y in zip(g1.state(), g2.state()):
        assert np.array_equal(x, y)


def test_grid_sizes_agree(P):
    # the result must not depend on the persistent grid (1 CTA .. full chip)
    r = gen.rrg(2, 4000, gen.gamma_star(2), n_boxes=15, seed=31)
    states = []
    for gb in (1, 3, 0):
        c = P.Context(h_root=r.h_root(), grid_blocks=gb)
        from paper_2003_04920_b200.berrt import replay
        replay(c, r, 333)
        states.append(c.state())
    for s in states[1:]:
        for x, y in zip(states[0], s):
            assert np.array_equal(x, y)


def test_determinism_rerun(P):
    r = gen.rrg(4, 6000, gen.gamma_k(4), n_boxes=10, seed=41)
    from paper_2003_04920_b200.berrt import replay
    outs = []
    for _ in range(2):
        c = P.Context(h_root=r.h_root())
        replay(c, r, 500)
        outs.append(c.state())
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


def test_noconv_cap(P):
    r = gen.rrg(2, 2000, gen.gamma_star(2), seed=5)
    gpu = P.Context(h_root=r.h_root(), max_iterations=1)
    src, dst, cost = r.batch(2, r.n)
    gpu.append(r.h[2:], src, dst, cost)
    with pytest.raises(P.PirrtError) as ei:
        gpu.exploit()
    assert ei.value.code == P.PIRRT_E_NOCONV


# ------------------------------------------------------------------ sharded / Evaluate variants

@pytest.mark.parametrize("flags", [0, PRUNE_OFF])
def test_sharded_loop_single_rank_parity(P, flags):
    # the multi-GPU code path (vertex-split Improve -> ncclAllGather of the
    # records -> replicated Evaluate) with one rank: bit-identical to the oracle
    r = gen.rrg(2, 3000, gen.gamma_star(2), n_boxes=20, seed=gen.seed_of("shard", flags))
    gpu = P.Context(h_root=r.h_root(), flags=flags | P.PIRRT_F_SHARDED)
    orc = Oracle(h_root=r.h_root(), flags=flags)
    dual_replay(gpu, orc, r, 97)


def test_sharded_loop_6d(P):
    r = gen.rrg(6, 15000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("shard6"))
    gpu = P.Context(h_root=r.h_root(), flags=P.PIRRT_F_SHARDED)
    orc = Oracle(h_root=r.h_root())
    dual_replay(gpu, orc, r, 1000)


@pytest.mark.parametrize("inc,keep,tail,wide", [
    ("0", None, "0", "0"), ("0", "2", "100000", "0"), ("0", None, None, "5"),
    ("0", "3", "0", "40"), (None, "1", None, None), (None, "7", None, None),
    ("100000", "64", None, None), ("3", None, None, None)])
def test_evaluate_variants_parity(P, monkeypatch, inc, keep, tail, wide):
    # the Evaluate forms must agree with the oracle: full traversal
    # (PIRRT_INC_MAX=0; level-synchronous, with or without handing the
    # shrinking tail or a wide frontier to the work queue) and incremental
    # (default, or every Evaluate whose start set allows it; a tiny start-set
    # limit mixes both forms); the work queue's local frontier size wq_keep
    # decides how much goes through the global queue
    if inc:
        monkeypatch.setenv("PIRRT_INC_MAX", inc)
    if keep:
        monkeypatch.setenv("PIRRT_WQ_KEEP", keep)
    if tail:
        monkeypatch.setenv("PIRRT_WQ_TAIL", tail)
    if wide:
        monkeypatch.setenv("PIRRT_WQ_WIDE", wide)
    r = gen.rrg(2, 4000, gen.gamma_star(2), n_boxes=25, seed=gen.seed_of("async"))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    dual_replay(gpu, orc, r, 50)


@pytest.mark.parametrize("gb", [1, 2, 5])
@pytest.mark.parametrize("inc", ["100000", "0"])
def test_work_queue_small_grids_6d(P, monkeypatch, gb, inc):
    # few blocks: claims run far ahead of publication, staging overflows;
    # the incremental Evaluate's roots overflow the local frontiers
    monkeypatch.setenv("PIRRT_INC_MAX", inc)
    monkeypatch.setenv("PIRRT_WQ_KEEP", "3")
    r = gen.rrg(6, 8000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("wq-small", gb))
    gpu = P.Context(h_root=r.h_root(), grid_blocks=gb)
    orc = Oracle(h_root=r.h_root())
    dual_replay(gpu, orc, r, 700)


@pytest.mark.parametrize("gb", [1, 3])
def test_level_to_work_queue_handover_6d(P, monkeypatch, gb):
    # level-synchronous start, hand-over to the work queue at a wide or a
    # shrinking frontier, with few blocks and small local frontiers
    monkeypatch.setenv("PIRRT_WQ_WIDE", "20")
    monkeypatch.setenv("PIRRT_WQ_TAIL", "50")
    monkeypatch.setenv("PIRRT_WQ_KEEP", "4")
    r = gen.rrg(6, 8000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("handover", gb))
    gpu = P.Context(h_root=r.h_root(), grid_blocks=gb)
    orc = Oracle(h_root=r.h_root())
    dual_replay(gpu, orc, r, 700)


@pytest.mark.parametrize("lpv", ["16", "32"])
@pytest.mark.parametrize("wide", ["1", "300"])
@pytest.mark.parametrize("flags", [0, PRUNE_OFF])
def test_wide_improve_handoff_parity(P, monkeypatch, wide, flags, lpv):
    # every Improve with |I| >= PIRRT_WIDE_TASKS runs as the full-occupancy
    # launch (hand-off and resume of the persistent loop), with 16 or 32
    # lanes per vertex: same bits, same counters as the oracle
    monkeypatch.setenv("PIRRT_WIDE_TASKS", wide)
    monkeypatch.setenv("PIRRT_WIDE_LPV", lpv)
    r = gen.rrg(6, 12000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("wide", wide, flags))
    gpu = P.Context(h_root=r.h_root(), flags=flags)
    orc = Oracle(h_root=r.h_root(), flags=flags)
    dual_replay(gpu, orc, r, 1500)


def test_wide_improve_cold_solve_and_goal_set(P, monkeypatch):
    monkeypatch.setenv("PIRRT_WIDE_TASKS", "1000")
    r = gen.rrg(2, 20000, gen.gamma_star(2), n_boxes=30, seed=gen.seed_of("wide-cold"))
    ids = np.nonzero(r.h[2:] <= 0.05)[0].astype(np.int32) + 2
    gpu = P.Context(h_root=r.h_root(), goals=ids)
    orc = Oracle(h_root=r.h_root())
    orc.set_goals(ids)
    dual_replay(gpu, orc, r, r.n)


@pytest.mark.parametrize("env", [{}, {"PIRRT_INC_MAX": "0", "PIRRT_WQ_KEEP": "3"},
                                 {"PIRRT_WQ_TAIL": "0", "PIRRT_WQ_WIDE": "0"},
                                 {"PIRRT_WIDE_TASKS": "500"}])
@pytest.mark.parametrize("flags", [0, PRUNE_OFF])
def test_children_index_evaluate_parity(P, monkeypatch, env, flags):
    # every Evaluate builds the children index (PIRRT_KIDS_MIN=1) instead of
    # scanning out-rows: same bits and counters as the oracle
    monkeypatch.setenv("PIRRT_KIDS_MIN", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    r = gen.rrg(6, 12000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("kids", flags))
    gpu = P.Context(h_root=r.h_root(), flags=flags)
    orc = Oracle(h_root=r.h_root(), flags=flags)
    dual_replay(gpu, orc, r, 900)


@pytest.mark.parametrize("gb", [1, 7])
def test_children_index_small_grids_and_sharded(P, monkeypatch, gb):
    monkeypatch.setenv("PIRRT_KIDS_MIN", "100")
    r = gen.rrg(2, 6000, gen.gamma_star(2), n_boxes=20, seed=gen.seed_of("kids-gb", gb))
    for extra in (0, P.PIRRT_F_SHARDED):
        gpu = P.Context(h_root=r.h_root(), grid_blocks=gb, flags=extra)
        orc = Oracle(h_root=r.h_root())
        dual_replay(gpu, orc, r, 600)


def test_sharded_loop_wide_improve(P, monkeypatch):
    # the sharded loop's Improve as the full-occupancy launch (records path)
    monkeypatch.setenv("PIRRT_WIDE_TASKS", "200")
    r = gen.rrg(6, 12000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("shard-wide"))
    for flags in (0, PRUNE_OFF):
        gpu = P.Context(h_root=r.h_root(), flags=flags | P.PIRRT_F_SHARDED)
        orc = Oracle(h_root=r.h_root(), flags=flags)
        dual_replay(gpu, orc, r, 2000)


@pytest.mark.parametrize("gb", [1, 2])
@pytest.mark.parametrize("flags", [0, PRUNE_OFF])
def test_children_index_wide_levels_few_blocks(P, monkeypatch, gb, flags):
    # few blocks: every block's share of a level exceeds its thread count
    # (one item per thread over the children index) and its push staging
    # overflows into the queue (warp-aggregated reservations)
    monkeypatch.setenv("PIRRT_KIDS_MIN", "1")
    r = gen.rrg(6, 15000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("kids-wide", gb, flags))
    gpu = P.Context(h_root=r.h_root(), flags=flags, grid_blocks=gb)
    orc = Oracle(h_root=r.h_root(), flags=flags)
    dual_replay(gpu, orc, r, r.n // 2)


@pytest.mark.parametrize("gb", [1, 3, 0])
def test_fused_root_levels_parity(P, monkeypatch, gb):
    # full Evaluates: levels 0 and 1 without a barrier (every block owns the
    # root's children at its row positions); with 1 or 3 blocks the root's
    # row may exceed the owned capacity (fallback to the plain level)
    monkeypatch.setenv("PIRRT_INC_MAX", "0")
    r = gen.rrg(6, 12000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("fuse-root", gb))
    gpu = P.Context(h_root=r.h_root(), grid_blocks=gb)
    orc = Oracle(h_root=r.h_root())
    dual_replay(gpu, orc, r, 700)
