"""GPU parity of the NEIGHBOURS variant (PIRRT_F_NEIGHBOURS; SURVEY.md 8(f)
NEXT-4, reading R16: I = B u N+(B u {root}) u G \\ {root})
against the oracle's ORC_F_NEIGHBOURS, which tests/test_oracle_neighbours.py
pins to hand-derived cases, Dijkstra and the Bellman certificate.  Bit-exact
state and equal counters after every exploit.  Run on a B200: -m gpu."""
import numpy as np
import pytest

import gen
from oracle import NEIGHBOURS, PARENT_FORM, PRUNE_OFF, Oracle
from parity import assert_same_state, assert_same_stats, dual_replay
from test_oracle_neighbours import CASE_A, CASE_B, build_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2003_04920_b200 import pirrt
    return pirrt


@pytest.mark.parametrize("case", [CASE_A, CASE_B], ids=["A", "B"])
@pytest.mark.parametrize("nb", [False, True])
def test_hand_cases(P, case, nb):
    gpu = P.Context(flags=P.PIRRT_F_NEIGHBOURS if nb else 0)
    orc = Oracle(flags=NEIGHBOURS if nb else 0)
    build_case(gpu, case)
    build_case(orc, case)
    gs, os_ = gpu.exploit(), orc.exploit()
    assert_same_stats(gs, os_)
    want = case["neighbours" if nb else "default"]
    assert gs.relaxations == want["relaxations"] and gs.iterations == want["iterations"]
    assert_same_state(gpu, orc)
    path, c = gpu.best_path()
    assert c == want["g_goal"] and path.tolist() == want["path"]


@pytest.mark.parametrize("d,n,S,gamma,extra", [
    (2, 4000, 1, "star", 0), (2, 6000, 40, "k", 0), (3, 8000, 300, "k", 0),
    (6, 12000, 1000, "k", 0), (7, 6000, 6000, "star", 0),            # S = N: one cold solve
    (2, 3000, 20, "star", PARENT_FORM), (3, 3000, 50, "k", PRUNE_OFF)])
def test_replay(P, d, n, S, gamma, extra):
    gm = gen.gamma_star(d) if gamma == "star" else gen.gamma_k(d)
    r = gen.rrg(d, n, gm, n_boxes=10, seed=gen.seed_of("nbr-gpu", d, n, S))
    gfl = P.PIRRT_F_NEIGHBOURS | {0: 0, PARENT_FORM: P.PIRRT_F_PARENT_FORM,
                                  PRUNE_OFF: P.PIRRT_F_PRUNE_OFF}[extra]
    gpu = P.Context(h_root=r.h_root(), flags=gfl)
    orc = Oracle(h_root=r.h_root(), flags=NEIGHBOURS | extra)
    dual_replay(gpu, orc, r, S, n_stop=min(n, 2 + 200 * S))


def test_goal_set(P):
    r = gen.rrg(2, 5000, gen.gamma_star(2), n_boxes=12, seed=gen.seed_of("nbr-goals"))
    ids = (np.nonzero(r.h[2:] <= 0.12)[0] + 2).astype(np.int32)
    gpu = P.Context(h_root=r.h_root(), flags=P.PIRRT_F_NEIGHBOURS, goals=ids)
    orc = Oracle(h_root=r.h_root(), flags=NEIGHBOURS)
    orc.set_goals(ids)
    dual_replay(gpu, orc, r, 25)


def test_rejected_with_sharding(P):
    with pytest.raises(P.PirrtError) as ei:
        P.Context(flags=P.PIRRT_F_NEIGHBOURS | P.PIRRT_F_SHARDED)
    assert ei.value.code == P.PIRRT_E_INVAL
