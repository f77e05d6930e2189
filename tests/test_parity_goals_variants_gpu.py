"""GPU parity (through the C ABI) of the goal-set form of R4 and of the
literal parent-form promising test (NEXT-4) against the oracle,
element by element, bit for bit, on seeded inputs.  Run on a B200: -m gpu."""
import numpy as np
import pytest

import gen
import oracle
from oracle import Oracle
from parity import assert_same_state, assert_same_stats, dual_replay
from test_oracle_goals_variants import goal_region, hand_tree, with_h

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2003_04920_b200 import pirrt
    return pirrt


def pair(P, h_root=0.0, prune_off=False, parent_form=False, goals=None, **kw):
    gf = (P.PIRRT_F_PRUNE_OFF if prune_off else 0) | (P.PIRRT_F_PARENT_FORM if parent_form else 0)
    of = (oracle.PRUNE_OFF if prune_off else 0) | (oracle.PARENT_FORM if parent_form else 0)
    gpu = P.Context(h_root=h_root, flags=gf | kw.pop("extra_flags", 0), goals=goals, **kw)
    orc = Oracle(h_root=h_root, flags=of)
    if goals is not None:
        orc.set_goals(goals)
    return gpu, orc


@pytest.mark.parametrize("S", [1, 37, 500])
@pytest.mark.parametrize("prune_off", [False, True])
def test_goal_region_replay_2d(P, S, prune_off):
    r = gen.rrg(2, 3000, gen.gamma_star(2), n_boxes=20, seed=gen.seed_of("gpu-goalset", S))
    ids, h = goal_region(r, 0.08)
    assert ids.size > 5
    gpu, orc = pair(P, h_root=h[0], prune_off=prune_off, goals=ids)
    dual_replay(gpu, orc, with_h(r, h), S)


def test_goal_region_replay_6d(P):
    r = gen.rrg(6, 20000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("gpu-goalset6"))
    ids, h = goal_region(r, 0.3)
    assert ids.size > 5
    gpu, orc = pair(P, h_root=h[0], goals=ids)
    dual_replay(gpu, orc, with_h(r, h), 1500)


@pytest.mark.parametrize("k", [5, 30])
@pytest.mark.parametrize("prune_off", [False, True])
def test_lattice_goal_row(P, k, prune_off):
    cells, id_of, src, dst, cost, _ = gen.lattice(k)
    h = (k - 1 - cells[:, 0]).astype(np.float64)
    gpu, orc = pair(P, h_root=h[0], prune_off=prune_off, goals=id_of[k - 1, :])
    assert gpu.append(h[2:], src, dst, cost) == orc.append(h[2:], src, dst, cost)
    gs, os_ = gpu.exploit(), orc.exploit()
    assert_same_stats(gs, os_)
    assert_same_state(gpu, orc)
    path, c, goal = gpu.best_path_goal()
    assert c == k - 1 and goal == id_of[k - 1, 0]
    assert path.tolist() == [int(id_of[r_, 0]) for r_ in range(k)]


def test_goal_ids_beyond_n_join_later(P):
    r = gen.rrg(2, 2000, gen.gamma_star(2), n_boxes=10, seed=gen.seed_of("gpu-future"))
    ids, h = goal_region(r, 0.1)
    gpu, orc = pair(P, h_root=h[0], goals=np.concatenate([ids, [5000, 1 << 20]]))
    assert gpu.best_path_goal()[2] == -1
    dual_replay(gpu, orc, with_h(r, h), 211)


def test_bad_goal_id_rejected(P):
    with pytest.raises(P.PirrtError) as ei:
        P.Context(goals=[0])
    assert ei.value.code == P.PIRRT_E_RANGE


def test_parent_form_hand_example(P):
    # the hand-derived Evaluate of tests/test_oracle_goals_variants.py,
    # through the full exploit on both sides
    gpu = P.Context(flags=P.PIRRT_F_PARENT_FORM)
    orc = hand_tree(oracle.PARENT_FORM)
    src = np.array([0, 2, 3, 3, 0], np.int32)
    dst = np.array([2, 3, 1, 4, 1], np.int32)
    gpu.append(np.zeros(3), src, dst, np.array([1, 1, 1, 5, 10], np.float64))
    gpu.set_policy(np.array([-1, 3, 0, 2, 3], np.int32), np.array([0, 3, 1, 2, 9.0]),
                   np.zeros(5, np.uint8))
    assert_same_state(gpu, orc, "after set_policy")
    gs, os_ = gpu.exploit(), orc.exploit()
    assert_same_stats(gs, os_)
    assert_same_state(gpu, orc)


@pytest.mark.parametrize("d,n,S,boxes", [(2, 3000, 1, 20), (2, 4000, 50, 25), (6, 20000, 1000, 10),
                                         (7, 8000, 400, 30)])
def test_parent_form_replay(P, d, n, S, boxes):
    gamma = gen.gamma_star(d) if d == 2 else gen.gamma_k(d)
    r = gen.rrg(d, n, gamma, n_boxes=boxes, seed=gen.seed_of("gpu-parent-form", d, S))
    gpu, orc = pair(P, h_root=r.h_root(), parent_form=True)
    dual_replay(gpu, orc, r, S)


def test_parent_form_with_goal_set_and_sharded_loop(P):
    r = gen.rrg(2, 3000, gen.gamma_star(2), n_boxes=15, seed=gen.seed_of("gpu-pf-shard"))
    ids, h = goal_region(r, 0.1)
    gpu, orc = pair(P, h_root=h[0], parent_form=True, goals=ids, extra_flags=P.PIRRT_F_SHARDED)
    dual_replay(gpu, orc, with_h(r, h), 97)


@pytest.mark.parametrize("env", [{"PIRRT_INC_MAX": "0", "PIRRT_WQ_KEEP": "3"},
                                 {"PIRRT_WQ_TAIL": "0", "PIRRT_WQ_WIDE": "0"},
                                 {"PIRRT_INC_MAX": "100000", "PIRRT_WQ_KEEP": "1"},
                                 {"PIRRT_INC_VALIDATE": "1"}])
def test_goal_set_parent_form_variants(P, monkeypatch, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    r = gen.rrg(6, 8000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("gpu-gs-var"))
    ids, h = goal_region(r, 0.3)
    for pf in (False, True):
        gpu, orc = pair(P, h_root=h[0], parent_form=pf, goals=ids, grid_blocks=3)
        dual_replay(gpu, orc, with_h(r, h), 700)


# ------------------------------------------------ VALIDATE: duplicates, cycles

def _states_equal(a, b):
    return all(np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
               for x, y in zip(a, b))


@pytest.mark.parametrize("undirected", [False, True])
def test_validate_duplicates_rejected_like_oracle(P, undirected):
    fl = P.PIRRT_F_EDGES_UNDIRECTED if undirected else 0
    ofl = oracle.EDGES_UNDIRECTED if undirected else 0
    gpu = P.Context(flags=P.PIRRT_F_VALIDATE)
    orc = Oracle(flags=oracle.VALIDATE)
    for ctx, f in ((gpu, fl), (orc, ofl)):
        ctx.append(np.zeros(3), np.array([0, 2, 3], np.int32), np.array([2, 3, 4], np.int32),
                   np.ones(3), flags=f)
    before = gpu.state()
    cases = [([0], [2]), ([4, 4], [1, 1]), ([2], [3])]
    if undirected:
        cases.append(([3], [2]))          # the reverse of a stored undirected pair
    for src, dst in cases:
        args = (np.zeros(0), np.array(src, np.int32), np.array(dst, np.int32), np.ones(len(src)))
        with pytest.raises(P.PirrtError) as eg:
            gpu.append(*args, flags=fl)
        with pytest.raises(oracle.OracleError) as eo:
            orc.append(*args, flags=ofl)
        assert eg.value.code == eo.value.code == P.PIRRT_E_INVAL
        assert _states_equal(gpu.state(), before)
    # a fresh pair is still accepted, then both agree
    for ctx, f in ((gpu, fl), (orc, ofl)):
        ctx.append(np.zeros(0), np.array([4], np.int32), np.array([1], np.int32), np.ones(1), flags=f)
    assert_same_stats(gpu.exploit(), orc.exploit())
    assert_same_state(gpu, orc)


def test_validate_cycles_rejected_like_oracle(P):
    src = np.array([0, 2, 3, 4], np.int32)
    dst = np.array([2, 3, 4, 2], np.int32)
    parent = np.array([-1, -1, 4, 2, 3], np.int32)
    g = np.array([0, np.inf, 1, 1, 1])
    gpu = P.Context(flags=P.PIRRT_F_VALIDATE)
    orc = Oracle(flags=oracle.VALIDATE)
    for ctx in (gpu, orc):
        ctx.append(np.zeros(3), src, dst, np.ones(4))
    before = gpu.state()
    with pytest.raises(P.PirrtError) as eg:
        gpu.set_policy(parent, g)
    assert eg.value.code == P.PIRRT_E_CORRUPT and _states_equal(gpu.state(), before)
    # given policy of a batch closing a zero-cost 2-cycle
    g3 = P.Context(flags=P.PIRRT_F_VALIDATE)
    with pytest.raises(P.PirrtError) as eg:
        g3.append(np.zeros(2), np.array([3, 2], np.int32), np.array([2, 3], np.int32), np.zeros(2),
                  parent_new=np.array([3, 2], np.int32), g_new=np.array([1.0, 1.0]))
    assert eg.value.code == P.PIRRT_E_CORRUPT and g3.n == 2
    # a long acyclic chain 0 -> 2 -> 3 -> ... -> n-1 -> 1 passes (many
    # pointer-jumping rounds), both on the given-policy append and set_policy
    n = 5000
    chain = np.concatenate([[0], np.arange(2, n), [1]]).astype(np.int32)
    src, dst = chain[:-1], chain[1:]
    parent = np.full(n, -1, np.int32); parent[dst] = src
    g = np.full(n, np.inf); g[0] = 0.0
    g[chain[1:]] = np.arange(1, n, dtype=np.float64)
    gl = P.Context(flags=P.PIRRT_F_VALIDATE)
    ol = Oracle(flags=oracle.VALIDATE)
    for ctx in (gl, ol):
        ctx.append(np.zeros(n - 2), src, dst, np.ones(n - 1), parent_new=parent[2:], g_new=g[2:])
        ctx.set_policy(parent, g)
    assert_same_stats(gl.exploit(), ol.exploit())
    assert_same_state(gl, ol)


# ------------------------------------- asynchronous exploit (NEXT-1)

@pytest.mark.parametrize("d,n,S", [(2, 4000, 37), (6, 20000, 1500)])
def test_async_exploit_pipelined_replay(P, d, n, S):
    # Alg. 3 with the exploit of batch k running while batch k+1 is staged
    # (its H2D on the side stream): same bits and counters as the oracle
    from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED, batches
    gamma = gen.gamma_star(d) if d == 2 else gen.gamma_k(d)
    r = gen.rrg(d, n, gamma, n_boxes=15, seed=gen.seed_of("async-exploit", d))
    gpu, orc = P.Context(h_root=r.h_root()), Oracle(h_root=r.h_root())
    started = False
    for k, (a, b) in enumerate(batches(r.n, S)):
        src, dst, cost = r.batch(a, b, directed=False)
        h = np.ascontiguousarray(r.h[a:b])
        pg = gpu.append(h, src, dst, cost, flags=EDGES_UNDIRECTED)   # overlaps the running exploit
        if started:
            assert_same_stats(gpu.exploit_wait(), orc_stats, f"batch {k}")
            started = False
        po = orc.append(h, src, dst, cost, flags=EDGES_UNDIRECTED)
        assert pg == po
        if po > 0:
            orc_stats = orc.exploit()
            gpu.exploit_async()
            started = True
            if k % 7 == 0:                 # a read-out completes the pending exploit
                assert_same_state(gpu, orc, f"batch {k}")
    if started:
        assert_same_stats(gpu.exploit_wait(), orc_stats, "last")
    gpu.exploit_async()
    assert_same_stats(gpu.exploit_wait(), orc.exploit(), "final")
    assert_same_state(gpu, orc, "final")


def test_async_exploit_wait_without_start(P):
    gpu = P.Context()
    with pytest.raises(P.PirrtError) as ei:
        gpu.exploit_wait()
    assert ei.value.code == P.PIRRT_E_STATE
    gpu.exploit_async()
    gpu.exploit_wait()
    with pytest.raises(P.PirrtError):
        gpu.exploit_wait()


# ------------------------------------------------------------ combinations

@pytest.mark.parametrize("env", [{"PIRRT_KIDS_MIN": "1"}, {"PIRRT_KIDS_MIN": "1", "PIRRT_INC_MAX": "0"},
                                 {"PIRRT_WIDE_TASKS": "1"}])
def test_parent_form_goal_set_with_index_and_wide_improve(P, monkeypatch, env):
    # the KIDS and parent-form instantiations together, and every Improve
    # through the full-occupancy launch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    r = gen.rrg(6, 10000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("combo", len(env)))
    ids, h = goal_region(r, 0.3)
    gpu, orc = pair(P, h_root=h[0], parent_form=True, goals=ids)
    dual_replay(gpu, orc, with_h(r, h), 1200)


def test_extend_with_goal_set_parent_form_and_async(P):
    # device-side Extend + goal set + parent form + the asynchronous exploit
    from oracle import EDGES_UNDIRECTED
    from paper_2003_04920_b200.berrt import batches
    r = gen.rrg(4, 8000, gen.gamma_k(4), n_boxes=12, seed=gen.seed_of("combo-extend"))
    ids, _ = goal_region(r, 0.15)
    # the device computes h = |x - x_goal| itself, as the generator does (r.h)
    gpu, orc = pair(P, h_root=r.h_root(), parent_form=True, goals=ids)
    gpu.set_world(4, r.boxes, r.points[0], r.points[1], gen.gamma_k(4))
    started = False
    for k, (a, b) in enumerate(batches(r.n, 300)):
        pg, ne = gpu.extend(r.points[a:b])
        if started:
            assert_same_stats(gpu.exploit_wait(), ost, f"batch {k}")
            started = False
        s, d_, c = r.batch(a, b, directed=False)
        po = orc.append(r.h[a:b], s, d_, c, flags=EDGES_UNDIRECTED)
        assert pg == po and ne == s.size
        if po > 0:
            ost = orc.exploit()
            gpu.exploit_async()
            started = True
    if started:
        assert_same_stats(gpu.exploit_wait(), ost, "last")
    assert_same_state(gpu, orc, "final")
