"""GPU parity of the deferred BE-RRT# step (pirrt_step_async / pirrt_step_wait,
SURVEY.md 8(f) NEXT-1) against the oracle driven step by
step through the synchronous form of Alg. 3 (append; Replan iff a new
promising vertex, P:461 / R10; best path).

Each step's n_new_promising, the Replan decision, every exploit counter, the
best path, its cost and goal must equal the oracle's; the whole vertex state
is compared bitwise whenever no step is outstanding.  Steps are kept two deep
(step k+1 enqueued before step k is waited), so the append of k+1 reads the
B-list state k's exploit left on the device.
Run on a B200: -m gpu.
"""
import numpy as np
import pytest

import gen
import oracle
from oracle import EDGES_UNDIRECTED, Oracle
from parity import assert_same_state, assert_same_stats

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2003_04920_b200 import pirrt
    return pirrt


def pinned(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()


def oracle_step(orc, h, s, t, c):
    nprom = orc.append(h, s, t, c, flags=EDGES_UNDIRECTED)
    st = orc.exploit() if nprom > 0 else None
    path, cost, goal = orc.best_path_goal()
    return nprom, st, path, cost, goal


def check_result(r, ref, where):
    nprom, st, path, cost, goal = ref
    assert r.n_new_promising == nprom, f"{where}: n_new_promising {r.n_new_promising} vs {nprom}"
    assert r.replanned == (st is not None), where
    if st is not None:
        assert_same_stats(r.stats, st, where)
    assert np.array_equal(r.path, path), f"{where}: best path differs"
    assert np.float64(r.cost).view(np.uint64) == np.float64(cost).view(np.uint64), where
    assert r.goal == goal, where


def run_pipelined(P, gpu, orc, r, batches, depth=2, device=False, check_state_every=4, where=""):
    """Enqueue up to `depth` steps ahead; compare each result as it is waited."""
    import torch
    pend = []
    k_done = 0
    for k, (a, b) in enumerate(batches):
        s, t, c = r.batch(a, b, directed=False)
        h = r.h[a:b]
        if device:
            args = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (h, s, t, c)]
        else:
            args = [pinned(x) for x in (h, s, t, c)]
        gpu.step_async(*args, flags=EDGES_UNDIRECTED)
        pend.append((k, oracle_step(orc, h, s, t, c)))
        if len(pend) >= depth:
            kk, ref = pend.pop(0)
            check_result(gpu.step_wait(), ref, f"{where} step {kk}")
            k_done += 1
            if k_done % check_state_every == 0 and not pend:
                assert_same_state(gpu, orc, f"{where} step {kk}")
    while pend:
        kk, ref = pend.pop(0)
        check_result(gpu.step_wait(), ref, f"{where} step {kk}")
    assert gpu.steps_outstanding == 0
    assert_same_state(gpu, orc, f"{where} end")


@pytest.mark.parametrize("d,n,S,gamma,boxes", [(2, 6000, 1, "star", 10), (2, 20000, 50, "star", 20),
                                               (6, 30000, 1024, "k", 20), (7, 12000, 1000, "star", 30),
                                               (3, 5000, 4999, "k", 5)])
def test_step_pipeline_matches_oracle(P, d, n, S, gamma, boxes):
    from paper_2003_04920_b200.berrt import batches
    gm = gen.gamma_k(d) if gamma == "k" else gen.gamma_star(d)
    r = gen.rrg(d, n, gm, n_boxes=boxes, seed=gen.seed_of("step", d, n, S))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    bl = list(batches(r.n, S))
    if S == 1:
        bl = bl[:1500]
    run_pipelined(P, gpu, orc, r, bl, where=f"{d}-D S={S}")


def test_step_mixed_with_synchronous_calls(P):
    """Steps, then synchronous appends / exploits, then steps again: each
    hand-over between the host's mirror and the device's B-list state."""
    from paper_2003_04920_b200.berrt import batches
    r = gen.rrg(4, 12000, gen.gamma_k(4), n_boxes=15, seed=gen.seed_of("step-mixed"))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    bl = list(batches(r.n, 400))
    run_pipelined(P, gpu, orc, r, bl[:8], where="part 1")
    for k, (a, b) in enumerate(bl[8:14]):
        s, t, c = r.batch(a, b, directed=False)
        pg = gpu.append(r.h[a:b], s, t, c, flags=EDGES_UNDIRECTED)
        po = orc.append(r.h[a:b], s, t, c, flags=EDGES_UNDIRECTED)
        assert pg == po
        if k % 2 == 0:                          # also an exploit without new members
            assert_same_stats(gpu.exploit(), orc.exploit(), f"sync {k}")
    assert_same_state(gpu, orc, "after sync part")
    run_pipelined(P, gpu, orc, r, bl[14:], depth=2, where="part 2")
    # a step that brings no vertex and no edge: the Replan is skipped on the device
    gpu.step_async(np.zeros(0), np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))
    res = gpu.step_wait()
    assert res.n_new_promising == 0 and not res.replanned
    path, cost, goal = orc.best_path_goal()
    assert np.array_equal(res.path, path) and res.cost == cost and res.goal == goal


def test_step_growth_with_steps_outstanding(P):
    """Tiny initial capacities: vertex, edge and staging buffers grow while a
    step is outstanding (the host mirror is refreshed from the device first)."""
    from paper_2003_04920_b200.berrt import batches
    r = gen.rrg(3, 20000, gen.gamma_k(3), n_boxes=10, seed=gen.seed_of("step-grow"))
    gpu = P.Context(h_root=r.h_root(), vertex_capacity=1024, edge_capacity=4096)
    orc = Oracle(h_root=r.h_root())
    run_pipelined(P, gpu, orc, r, list(batches(r.n, 700)), check_state_every=3, where="grow")


def test_step_device_pointers(P):
    from paper_2003_04920_b200.berrt import batches
    r = gen.rrg(6, 20000, gen.gamma_k(6), n_boxes=20, seed=gen.seed_of("step-dev"))
    gpu = P.Context(h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    run_pipelined(P, gpu, orc, r, list(batches(r.n, 2048)), device=True, where="device ptrs")


def test_step_goal_set_and_parent_form(P):
    from paper_2003_04920_b200.berrt import batches
    r = gen.rrg(2, 8000, gen.gamma_star(2), n_boxes=10, seed=gen.seed_of("step-goals"))
    goals = [5, 77, 300, 4000]
    gpu = P.Context(h_root=r.h_root(), goals=goals, flags=P.PIRRT_F_PARENT_FORM)
    orc = Oracle(h_root=r.h_root(), flags=oracle.PARENT_FORM)
    orc.set_goals(goals)
    run_pipelined(P, gpu, orc, r, list(batches(r.n, 37))[:120], where="goals+parent form")


def test_step_errors(P):
    r = gen.rrg(2, 2000, gen.gamma_star(2), n_boxes=0, seed=gen.seed_of("step-err"))
    gpu = P.Context(h_root=r.h_root())
    s, t, c = r.batch(2, 500, directed=False)
    with pytest.raises(P.PirrtError) as e:
        gpu.step_wait()
    assert e.value.code == P.PIRRT_E_STATE
    with pytest.raises(P.PirrtError) as e:
        gpu.step_async(r.h[2:500], s, t, c, flags=EDGES_UNDIRECTED | P.PIRRT_F_VALIDATE)
    assert e.value.code == P.PIRRT_E_INVAL
    gpu.step_async(r.h[2:500], s, t, c, flags=EDGES_UNDIRECTED)
    s2, t2, c2 = r.batch(500, 600, directed=False)
    gpu.step_async(r.h[500:600], s2, t2, c2, flags=EDGES_UNDIRECTED)
    s3, t3, c3 = r.batch(600, 700, directed=False)
    with pytest.raises(P.PirrtError) as e:      # two outstanding
        gpu.step_async(r.h[600:700], s3, t3, c3, flags=EDGES_UNDIRECTED)
    assert e.value.code == P.PIRRT_E_STATE
    for call in (gpu.exploit, gpu.best_path, gpu.policy,
                 lambda: gpu.append(r.h[600:700], s3, t3, c3, flags=EDGES_UNDIRECTED)):
        with pytest.raises(P.PirrtError) as e:
            call()
        assert e.value.code == P.PIRRT_E_STATE
    gpu.step_wait()
    gpu.step_wait()
    gpu.best_path()                              # usable again
    # a batch the device rejects (an endpoint beyond the new vertices)
    bad = t3.copy()
    bad[0] = 10 ** 6
    gpu.step_async(r.h[600:700], s3, bad, c3, flags=EDGES_UNDIRECTED)
    with pytest.raises(P.PirrtError) as e:
        gpu.step_wait()
    assert e.value.code == P.PIRRT_E_RANGE
    with pytest.raises(P.PirrtError) as e:      # unusable afterwards
        gpu.best_path()
    assert e.value.code == P.PIRRT_E_STATE


@pytest.mark.parametrize("variant", ["prune_off", "neighbours", "eps"])
def test_step_variants(P, variant):
    """Deferred steps under the configuration variants (classical PI, the
    NEIGHBOURS Improve set, epsilon > 0) against the oracle's synchronous step."""
    from paper_2003_04920_b200.berrt import batches
    r = gen.rrg(3, 6000, gen.gamma_k(3), n_boxes=8, seed=gen.seed_of("step-var", variant))
    kw, okw = {}, {}
    if variant == "prune_off":
        kw["flags"], okw["flags"] = P.PIRRT_F_PRUNE_OFF, oracle.PRUNE_OFF
    elif variant == "neighbours":
        kw["flags"], okw["flags"] = P.PIRRT_F_NEIGHBOURS, oracle.NEIGHBOURS
    else:
        kw["epsilon"] = okw["epsilon"] = 1e-3
    gpu = P.Context(h_root=r.h_root(), **kw)
    orc = Oracle(h_root=r.h_root(), **okw)
    run_pipelined(P, gpu, orc, r, list(batches(r.n, 211)), where=variant)
