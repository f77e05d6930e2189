"""Multi-rank sharded exploitation with P > 1 ranks on ONE
GPU: an in-process group of P contexts (PIRRT_F_LOCAL_GROUP) runs the same
kernels and the same chunked, device-driven loop as one process per GPU, with
the record all-gather done as device copies (pirrt_group_exploit).  Vertex
v's Improve runs on rank v mod P; every rank applies every record and runs
the replicated Evaluate.  Checked bit for bit against the oracle after every
exploit, every rank's state identical, the per-rank relaxation shares summing
to the oracle's count.  Run on a B200: -m gpu."""
import numpy as np
import pytest

import gen
from oracle import PRUNE_OFF, Oracle
from parity import RankGroup, dual_replay

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2003_04920_b200 import pirrt
    return pirrt


@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
def test_group_replay_2d(P, nranks):
    r = gen.rrg(2, 4000, gen.gamma_star(2), n_boxes=20, seed=gen.seed_of("group2d", nranks))
    grp = RankGroup(P, nranks, h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    dual_replay(grp, orc, r, 97)


@pytest.mark.parametrize("nranks,flags", [(2, 0), (3, PRUNE_OFF), (2, PRUNE_OFF)])
def test_group_replay_6d(P, nranks, flags):
    r = gen.rrg(6, 15000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("group6d", nranks, flags))
    grp = RankGroup(P, nranks, h_root=r.h_root(), flags=flags)
    orc = Oracle(h_root=r.h_root(), flags=flags)
    dual_replay(grp, orc, r, 1000)


def test_group_shared_stream_and_wide_improve(P, monkeypatch):
    # all ranks on one stream; large improve sets through the full-occupancy
    # Improve launch (the device picks it per iteration)
    import torch
    monkeypatch.setenv("PIRRT_WIDE_TASKS", "200")
    r = gen.rrg(6, 12000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("group-wide"))
    grp = RankGroup(P, 2, stream=torch.cuda.current_stream(), h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    dual_replay(grp, orc, r, 2000)


def test_group_goal_set_and_parent_form(P):
    import oracle
    r = gen.rrg(2, 5000, gen.gamma_star(2), n_boxes=15, seed=gen.seed_of("group-goals"))
    ids = (np.nonzero(r.h[2:] <= 0.1)[0] + 2).astype(np.int32)
    grp = RankGroup(P, 3, h_root=r.h_root(), goals=ids, flags=P.PIRRT_F_PARENT_FORM)
    orc = Oracle(h_root=r.h_root(), flags=oracle.PARENT_FORM)
    orc.set_goals(ids)
    dual_replay(grp, orc, r, 50)


def test_group_record_overflow_regather(P):
    # a cold solve (S = N): the first Improves emit far more records than
    # the initial per-rank stride K -- the loop stops before applying any,
    # re-gathers with a larger K and goes on, bit-exact
    r = gen.rrg(3, 20000, gen.gamma_k(3), n_boxes=8, seed=gen.seed_of("group-over"))
    grp = RankGroup(P, 2, h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    dual_replay(grp, orc, r, r.n)


def test_group_iteration_cap(P):
    # R11 cap inside the chunked loop: E_NOCONV on every rank, state as the
    # oracle leaves it after the same number of Improves
    r = gen.rrg(2, 3000, gen.gamma_star(2), n_boxes=10, seed=gen.seed_of("group-cap"))
    grp = RankGroup(P, 2, h_root=r.h_root(), max_iterations=2)
    orc = Oracle(h_root=r.h_root(), max_iterations=2)
    from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED
    s, t, c = r.batch(2, r.n, directed=False)
    assert grp.append(r.h[2:], s, t, c, flags=EDGES_UNDIRECTED) == \
        orc.append(r.h[2:], s, t, c, flags=EDGES_UNDIRECTED)
    with pytest.raises(P.PirrtError) as ei:
        grp.exploit()
    assert ei.value.code == P.PIRRT_E_NOCONV
    orc.exploit(allow_noconv=True)
    from parity import assert_same_state
    assert_same_state(grp, orc, "cap")


def test_group_misuse(P):
    a = P.Context(nranks=2, rank=0, flags=P.PIRRT_F_LOCAL_GROUP)
    b = P.Context(nranks=2, rank=1, flags=P.PIRRT_F_LOCAL_GROUP)
    with pytest.raises(P.PirrtError) as ei:
        a.exploit()                                    # only through pirrt_group_exploit
    assert ei.value.code == P.PIRRT_E_STATE
    with pytest.raises(P.PirrtError) as ei:
        P.group_exploit([b, a])                        # ranks out of order
    assert ei.value.code == P.PIRRT_E_STATE
    P.group_exploit([a, b])


def test_group_partitioned_store(P):
    """nranks > 1: a fold keeps only the in-edge rows of the vertices a rank
    owns (v mod P == rank).  After a replay with many folds each rank's owned
    rows hold exactly the generator's in-edges (element by element), the
    rank stores fewer edges than the graph has, the results stay bit-exact
    (dual_replay), and set_policy -- which needs every policy edge's cost --
    is refused."""
    from parity import sorted_edges
    r = gen.rrg(6, 20000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("group-part"))
    grp = RankGroup(P, 2, h_root=r.h_root())
    orc = Oracle(h_root=r.h_root())
    dual_replay(grp, orc, r, 256)
    src, dst, cost = r.batch(2, r.n, directed=True)
    for rank, c in enumerate(grp.ranks):
        off, s_, c_ = c.in_edges()
        d_ = np.repeat(np.arange(off.size - 1), np.diff(off))
        assert off[-1] < src.size, "no row was dropped"
        mine = d_ % 2 == rank
        want = dst % 2 == rank
        a = sorted_edges(s_[mine], d_[mine], c_[mine])
        b = sorted_edges(src[want], dst[want], cost[want])
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        assert c.n_edges == src.size                     # the graph's count, not the rank's
        with pytest.raises(P.PirrtError) as ei:
            c.set_policy(*orc.state()[:2])
        assert ei.value.code == P.PIRRT_E_STATE
