"""Pins of the oracle's goal-set form of R4 and of the literal parent-form
promising test (NEXT-4), against things other than the oracle:
scipy Dijkstra, closed forms on the unit lattice, a hand-derived Evaluate of
PAPER.md:255-270, the Bellman certificate and the definition of B.

Goal set (R4): G = {x_goal} u extra ids; the threshold is the
minimum of g over the goals that exist; every existing goal is improved; the
best goal is the lowest id at that minimum.
"""
import math

import numpy as np
import pytest

import gen
from oracle import PARENT_FORM, PRUNE_OFF, Oracle
from paper_2003_04920_b200.berrt import replay
from test_oracle_pins import bits, certificate, scipy_sssp

INF = math.inf


def goal_region(r, radius):
    """Goal set = x_goal plus every sample within `radius` of it; h = distance
    to that ball (admissible and consistent for the region)."""
    ids = np.nonzero(r.h[2:] <= radius)[0].astype(np.int32) + 2
    h = np.maximum(r.h - radius, 0.0)
    return ids, h


def with_h(r, h):
    import copy
    r2 = copy.copy(r)
    r2.h = h
    return r2


# ---------------------------------------------- goal set, PRUNE_OFF = Dijkstra

@pytest.mark.parametrize("seed", range(4))
def test_goal_set_prune_off_equals_dijkstra(seed):
    r = gen.rrg(2, 800, gen.gamma_star(2), n_boxes=5, seed=gen.seed_of("goalset", seed))
    ids, h = goal_region(r, 0.12)
    assert ids.size >= 2
    o = Oracle(h_root=h[0], flags=PRUNE_OFF)
    o.set_goals(ids)
    replay(o, with_h(r, h), r.n)
    src, dst, cost = r.batch(2, r.n)
    dist, _ = scipy_sssp(r.n, src, dst, cost)
    _, g, _, _ = o.state()
    reach = np.isfinite(dist)
    assert np.array_equal(bits(g[reach]), bits(dist[reach])) and np.isinf(g[~reach]).all()
    goals = np.concatenate([[1], ids])
    best = dist[goals].min()
    path, c, goal = o.best_path_goal()
    assert c == best and goal == goals[dist[goals] == best].min()
    assert path[0] == 0 and path[-1] == goal


@pytest.mark.parametrize("seed,S", [(0, 1), (1, 20), (2, 200)])
def test_goal_set_certificate(seed, S):
    # north-star mode: Bellman certificate on S = B u G (every existing goal
    # is improved, R4); best goal = lowest id at the minimum of g over G
    r = gen.rrg(2, 600, gen.gamma_star(2), n_boxes=8, seed=gen.seed_of("goalcert", seed))
    ids, h = goal_region(r, 0.1)
    o = Oracle(h_root=h[0])
    o.set_goals(ids)
    replay(o, with_h(r, h), S)
    src, dst, cost = r.batch(2, r.n)
    _, g, _, b = o.state()
    certificate(o, src, dst, cost, goals=np.concatenate([[1], ids]))
    goals = np.concatenate([[1], ids])
    path, c, goal = o.best_path_goal()
    m = g[goals].min()
    assert c == m and goal == goals[g[goals] == m].min()


@pytest.mark.parametrize("k", [5, 9])
@pytest.mark.parametrize("flags", [0, PRUNE_OFF])
def test_lattice_goal_row(k, flags):
    # goals = the whole far row r = k-1 (x_goal = (k-1, k-1) is in it);
    # h = k-1-r is the exact distance to that row.  The nearest goal is
    # (k-1, 0), straight up from the root along column 0: g = k-1, a unique
    # shortest path.
    cells, id_of, src, dst, cost, _ = gen.lattice(k)
    h = (k - 1 - cells[:, 0]).astype(np.float64)
    o = Oracle(h_root=h[0], flags=flags)
    o.set_goals(id_of[k - 1, :])
    o.append(h[2:], src, dst, cost)
    o.exploit()
    path, c, goal = o.best_path_goal()
    assert c == k - 1 and goal == id_of[k - 1, 0]
    assert path.tolist() == [int(id_of[r, 0]) for r in range(k)]


def test_future_goal_ids_join_when_appended():
    # a goal id beyond |V| is inactive until its vertex exists
    cells, id_of, src, dst, cost, h = gen.lattice(4)
    o = Oracle(h_root=h[0])
    o.set_goals([15])                      # the last vertex of the lattice
    assert o.best_path_goal()[2] == -1
    o.append(h[2:], src, dst, cost)
    o.exploit()
    _, g, _, _ = o.state()
    path, c, goal = o.best_path_goal()
    assert c == min(g[1], g[15])


# ------------------------------------------- parent-form test (P:263 literal)

def hand_tree(flags):
    """Root 0 -> 2 (c=1) -> 3 (c=1) -> {goal 1 (c=1), 4 (c=5)}, plus 0 -> 1
    (c=10); h = 0.  Policy = that tree with g(goal) = 3 (so thr = 3) and a
    stale g(4) = 9."""
    o = Oracle(flags=flags)
    src = np.array([0, 2, 3, 3, 0], np.int32)
    dst = np.array([2, 3, 1, 4, 1], np.int32)
    cost = np.array([1, 1, 1, 5, 10], np.float64)
    o.append(np.zeros(3), src, dst, cost)
    o.set_policy(np.array([-1, 3, 0, 2, 3], np.int32), np.array([0, 3, 1, 2, 9.0]),
                 np.zeros(5, np.uint8))
    return o


def test_evaluate_child_vs_parent_form_hand_example():
    # P:255-270 by hand with thr = g(goal) = 3:
    #   child form (R2): 2 (f=1), 3 (f=2) pass; the goal (f=3) and 4 (f=7)
    #     are visited (g written) but not expanded  -> B = {2, 3}
    #   parent form (P:263 as printed): the children of 0 (f=0), 2 (f=1) and
    #     3 (f=2) are all pushed                    -> B = {1, 2, 3, 4}
    # g after the step is [0, 3, 1, 2, 7] in both.
    for flags, want in ((0, [0, 0, 1, 1, 0]), (PARENT_FORM, [0, 1, 1, 1, 1])):
        o = hand_tree(flags)
        o.evaluate_step()
        _, g, _, b = o.state()
        assert g.tolist() == [0, 3, 1, 2, 7] and b.tolist() == want


def goal_cost(g, goals):
    return min(g[t] for t in goals if t < g.size)


@pytest.mark.parametrize("form", [0, PARENT_FORM])
@pytest.mark.parametrize("seed", range(3))
def test_B_definition_after_every_evaluate(form, seed):
    # the set Evaluate builds is the least fixed point of its definition
    # (P:255-270): with E = {root} u B (the expanded vertices) and thr the
    # goal cost at entry, for every vertex n with parent p:
    #   p in E  =>  g(n) == g(p) + pc(n)  and  (n in B  <=>  test passes),
    #   p not in E  =>  n not in B,
    # test = g(n)+h(n) < thr (child form) or g(p)+h(p) < thr (parent form),
    # and every member of B is reached from the root through E.
    r = gen.rrg(2, 400, gen.gamma_k(2), n_boxes=6, seed=gen.seed_of("bdef", seed))
    o = Oracle(h_root=r.h_root(), flags=form)
    checked = 0
    for a, b_ in [(2, 150), (150, 151), (151, 260), (260, 400)]:
        src, dst, cost = r.batch(a, b_)
        o.append(r.h[a:b_], src, dst, cost)
        for _ in range(50):
            dg, _, _ = o.improve_step()
            if dg <= 0:
                break
            _, g0, _, _ = o.state()
            thr = goal_cost(g0, [1])
            o.evaluate_step()
            parent, g, pc, b = o.state()
            E = b.astype(bool).copy()
            E[0] = True
            for n_ in range(1, g.size):
                p = parent[n_]
                if p >= 0 and E[p]:
                    assert bits(g[p] + pc[n_]) == bits(g[n_])
                    f = g[n_] + r.h[n_] if form == 0 else g[p] + r.h[p]
                    assert bool(b[n_]) == (f < thr)
                else:
                    assert b[n_] == 0
            for n_ in np.nonzero(b)[0]:          # reached from the root through E
                v, hops = int(n_), 0
                while v != 0:
                    v = int(parent[v]); hops += 1
                    assert v == 0 or b[v]
                    assert hops <= g.size
            checked += 1
    assert checked >= 3


def test_parent_form_prune_off_equals_dijkstra():
    # thr = +inf: both forms expand everything, PI = Dijkstra (P1)
    r = gen.rrg(2, 500, gen.gamma_star(2), n_boxes=4, seed=gen.seed_of("pf-dij"))
    o = Oracle(h_root=r.h_root(), flags=PRUNE_OFF | PARENT_FORM)
    replay(o, r, 50)
    src, dst, cost = r.batch(2, r.n)
    dist, _ = scipy_sssp(r.n, src, dst, cost)
    _, g, _, _ = o.state()
    reach = np.isfinite(dist)
    assert np.array_equal(bits(g[reach]), bits(dist[reach]))


# --------------------------------------- VALIDATE: duplicates and parent cycles

from oracle import VALIDATE, OracleError  # noqa: E402


def test_validate_duplicate_edge_rejected():
    # a (src,dst) pair stored twice is rejected under
    # VALIDATE, against the stored graph and inside one batch; state unchanged
    o = Oracle(flags=VALIDATE)
    o.append(np.zeros(2), np.array([0, 2], np.int32), np.array([2, 3], np.int32), np.ones(2))
    before = o.state()
    for src, dst in (([0], [2]), ([3, 3], [1, 1])):
        with pytest.raises(OracleError) as ei:
            o.append(np.zeros(0), np.array(src, np.int32), np.array(dst, np.int32),
                     np.ones(len(src)))
        assert ei.value.code == -1
        for x, y in zip(o.state(), before):
            assert np.array_equal(x, y)
    Oracle().append(np.zeros(1), np.array([0, 0], np.int32), np.array([2, 2], np.int32),
                    np.ones(2))   # accepted without VALIDATE (caller's responsibility)


def test_validate_parent_cycle_rejected():
    # the policy is a tree.  A 3-cycle 2 -> 3 -> 4 -> 2 among
    # stored edges is rejected by set_policy under VALIDATE (E_CORRUPT)
    src = np.array([0, 2, 3, 4], np.int32)
    dst = np.array([2, 3, 4, 2], np.int32)
    parent = np.array([-1, -1, 4, 2, 3], np.int32)
    g = np.array([0, np.inf, 1, 1, 1])
    o = Oracle(flags=VALIDATE)
    o.append(np.zeros(3), src, dst, np.ones(4))
    with pytest.raises(OracleError) as ei:
        o.set_policy(parent, g)
    assert ei.value.code == -8
    o2 = Oracle()
    o2.append(np.zeros(3), src, dst, np.ones(4))
    o2.set_policy(parent, g)                  # not checked without VALIDATE
    # a given policy closing a zero-cost 2-cycle passes the g check but not
    # the cycle check
    o3 = Oracle(flags=VALIDATE)
    with pytest.raises(OracleError) as ei:
        o3.append(np.zeros(2), np.array([3, 2], np.int32), np.array([2, 3], np.int32),
                  np.zeros(2), parent_new=np.array([3, 2], np.int32), g_new=np.array([1.0, 1.0]))
    assert ei.value.code == -8 and o3.n == 2
