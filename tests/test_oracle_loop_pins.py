"""Pins of the oracle's loop control and counters (CPU only).

* R13 stall guard: "stop when an iteration changes no
  parent value AND the following Evaluate changes no g bit and no b bit".
  Hand-built states (loaded with set_policy) where Improve changes no parent
  but Evaluate changes g (or only b): the loop must go on; and one where
  nothing changes: the loop must stop with stalled = 1.  Expected values are
  derived by hand from Alg. 2 in the docstrings.
* Counters against brute force from the edge list: relaxations of one
  Improve = sum over v in I of indeg(v); visits of
  one Evaluate = #{v : parent(v) in {root} u B_new} (every child of
  an expanded vertex is visited once); levels = depth of the deepest such v.
* epsilon > 0 (R5): the loop stops when Delta g <= eps and keeps the
  final Improve's parent changes without re-evaluating them.
"""
import math

import numpy as np
import pytest

import gen
from oracle import EDGES_UNDIRECTED, Oracle
from paper_2003_04920_b200.berrt import replay

INF = math.inf


def chain_oracle(h, edges, parent, g, b, eps=0.0):
    """Oracle with vertices 0..len(h)-1 (h[0], h[1] = root, goal), the given
    directed edges (u, v, c), and the policy snapshot (parent, g, b)."""
    n = len(h)
    o = Oracle(h_root=h[0], h_goal=h[1], epsilon=eps)
    src = np.array([e[0] for e in edges], np.int32)
    dst = np.array([e[1] for e in edges], np.int32)
    cost = np.array([e[2] for e in edges], np.float64)
    o.append(np.array(h[2:], np.float64), src, dst, cost)
    o.set_policy(np.array(parent, np.int32), np.array(g, np.float64), np.array(b, np.uint8))
    assert o.n == n
    return o


def test_r13_goes_on_when_evaluate_changes_g():
    """Root 0 -> a=2 (c 1), a -> goal 1 (c 1); h = 0.  Snapshot: parent(a)=0,
    g(a)=5 (stale), parent(goal)=a, g(goal)=10, B={a}.
    it 1: Improve over I={a, goal}: a: 0+1=1 < 5 (parent 0 again), goal:
    5+1=6 < 10 (parent a again) -> Delta g = 4, NO parent value changed.
    Evaluate (thr=10): a: g=1 in B; goal: g=2 in B -> g changed -> go on.
    it 2: a: 1 = g, goal: 1+1 = 2 = g -> Delta g = 0 -> stop.
    So: iterations 2, evaluations 1, stalled 0, g = (0, 2, 1)."""
    o = chain_oracle([0.0, 0.0, 0.0], [(0, 2, 1.0), (2, 1, 1.0)],
                     parent=[-1, 2, 0], g=[0.0, 10.0, 5.0], b=[0, 0, 1])
    st = o.exploit()
    assert (st.iterations, st.evaluations, st.stalled) == (2, 1, 0)
    parent, g, pc, b = o.state()
    assert g.tolist() == [0.0, 2.0, 1.0]
    assert parent.tolist() == [-1, 2, 0] and b.tolist() == [0, 1, 1]
    assert st.last_delta_g == 0.0


def test_r13_goes_on_when_evaluate_changes_only_b():
    """Root 0; a=2 (0->a c 1, h(a)=100: never expanded), x=3 (a->x c 1,
    h 0), y=4 (0->y c 1, h 0), goal 1 (0->goal c 10).  Snapshot: parent(a)=0
    g 1, parent(x)=a g 5 (stale), parent(y)=0 g 1, parent(goal)=0 g 10;
    B = {x}.
    it 1: I = {x, goal}: x: 1+1 = 2 < 5 (parent a again) -> Delta g 3; goal:
    10 = g.  No parent change.  Evaluate (thr 10): a: g 1, f 101 -> out;
    y: g 1, f 1 < 10 -> in B (b flips 0 -> 1); goal: g 10, f 10 not < 10;
    x is not visited (a not expanded) -> leaves B (b flips 1 -> 0).  No g
    bit changed, but b did -> go on.
    it 2: I = {y, goal}: y 1 = g, goal 10 = g -> Delta g 0 -> stop."""
    o = chain_oracle([0.0, 0.0, 100.0, 0.0, 0.0],
                     [(0, 2, 1.0), (2, 3, 1.0), (0, 4, 1.0), (0, 1, 10.0)],
                     parent=[-1, 0, 0, 2, 0], g=[0.0, 10.0, 1.0, 5.0, 1.0], b=[0, 0, 0, 1, 0])
    st = o.exploit()
    assert (st.iterations, st.evaluations, st.stalled) == (2, 1, 0)
    parent, g, pc, b = o.state()
    assert g.tolist() == [0.0, 10.0, 1.0, 5.0, 1.0]
    assert b.tolist() == [0, 0, 0, 0, 1]


def test_r13_stalls_when_nothing_changes():
    """Root 0 -> a=2 (c 1, h(a)=5: f(a) = 6 >= thr 3, never expanded),
    a -> goal 1 (c 1).  Snapshot: parent(a)=0 g 1, parent(goal)=a g 3
    (stale: g(a)+1 = 2), B = {}.
    it 1: I = {goal}: 1+1 = 2 < 3 with parent a again -> Delta g 1, no
    parent change.  Evaluate (thr 3): a: g 1 (same bits), f 6 -> not
    expanded, b 0 (same); goal not visited -> nothing changed -> R13 stop:
    iterations 1, evaluations 1, stalled 1 (without R13: E_NOCONV)."""
    o = chain_oracle([0.0, 0.0, 5.0], [(0, 2, 1.0), (2, 1, 1.0)],
                     parent=[-1, 2, 0], g=[0.0, 3.0, 1.0], b=[0, 0, 0])
    st = o.exploit()
    assert (st.iterations, st.evaluations, st.stalled) == (1, 1, 1)
    assert st.last_delta_g == 1.0
    assert o.state()[1].tolist() == [0.0, 3.0, 1.0]


def test_r13_goes_on_after_a_parent_change_that_changes_nothing_else():
    """Root 0 -> a=2 (c 1, h(a)=100: never expanded), a -> goal 1 (c 1),
    0 -> goal (c 10).  Snapshot: parent(a)=0 g 1, parent(goal)=0 g 10, B={}.
    it 1: I = {goal}: min(1+1 via a, 0+10 via 0) = 2 < 10 -> parent(goal)
    0 -> a (a parent value CHANGED), Delta g 8.  Evaluate (thr 10): a: g 1
    (same), f 101 -> not expanded; goal (child of a now) not visited ->
    no g or b bit changed, but the parent did -> go on (R13 needs both).
    it 2: goal: 2 < 10 via a again -> Delta g 8, no parent change; Evaluate
    changes nothing -> R13 stop: iterations 2, evaluations 2, stalled 1."""
    o = chain_oracle([0.0, 0.0, 100.0], [(0, 2, 1.0), (2, 1, 1.0), (0, 1, 10.0)],
                     parent=[-1, 0, 0], g=[0.0, 10.0, 1.0], b=[0, 0, 0])
    st = o.exploit()
    assert (st.iterations, st.evaluations, st.stalled) == (2, 2, 1)
    assert st.last_delta_g == 8.0
    parent, g, pc, b = o.state()
    assert parent.tolist() == [-1, 2, 0] and g.tolist() == [0.0, 10.0, 1.0]


def eps_oracle(eps):
    """Root 0, goal 1, a=2, c=3, h = 0.  Edges 0->a 1, 0->c 0.25, c->a 0.25,
    a->goal 1, 0->goal 10.  Snapshot: parent(a)=0 g 1, parent(c)=0 g 0.25,
    parent(goal)=0 g 10, B = {a, c}.
    it 1: a: min(0+1, 0.25+0.25) = 0.5 via c (Delta 0.5); c: 0.25 = g;
    goal: min(1+1, 0+10) = 2 via a (Delta 8) -> Delta g = 8.
    eps >= 8: stop now (R5), parents kept, g not re-evaluated.
    eps < 8: Evaluate (thr 10): c 0.25, a 0.5, goal 1.5 (all in B); it 2:
    a 0.5 = g, c, goal 0.5+1 = 1.5 = g -> Delta g 0 -> stop."""
    return chain_oracle([0.0, 0.0, 0.0, 0.0],
                        [(0, 2, 1.0), (0, 3, 0.25), (3, 2, 0.25), (2, 1, 1.0), (0, 1, 10.0)],
                        parent=[-1, 0, 0, 0], g=[0.0, 10.0, 1.0, 0.25], b=[0, 0, 1, 1], eps=eps)


def test_epsilon_stops_and_keeps_the_last_improve():
    o = eps_oracle(8.0)
    st = o.exploit()
    assert (st.iterations, st.evaluations, st.last_delta_g) == (1, 0, 8.0)
    parent, g, pc, b = o.state()
    assert parent.tolist() == [-1, 2, 3, 0]          # Improve's changes kept (R5)
    assert pc.tolist() == [0.0, 1.0, 0.25, 0.25]
    assert g.tolist() == [0.0, 10.0, 1.0, 0.25]      # not re-evaluated
    assert b.tolist() == [0, 0, 1, 1]


@pytest.mark.parametrize("eps", [0.0, 7.99])
def test_epsilon_below_delta_runs_to_the_fixed_point(eps):
    o = eps_oracle(eps)
    st = o.exploit()
    assert (st.iterations, st.evaluations, st.last_delta_g) == (2, 1, 0.0)
    parent, g, pc, b = o.state()
    assert parent.tolist() == [-1, 2, 3, 0]
    assert g.tolist() == [0.0, 1.5, 0.5, 0.25]
    assert b.tolist() == [0, 1, 1, 1]


def test_epsilon_large_then_exploit_again():
    """With eps = 8 the first exploit leaves Improve's changes unevaluated.  A
    second exploit's first Improve sees the same stale g: a 0.5 < 1 (Delta
    0.5), goal 1 + 1 = 2 < 10 (Delta 8) -> Delta g 8 <= eps -> stops at once,
    still unevaluated: the literal R5 reading never re-evaluates below eps."""
    o = eps_oracle(8.0)
    o.exploit()
    st = o.exploit()
    assert (st.iterations, st.evaluations) == (1, 0)
    assert st.last_delta_g == 8.0                     # goal: 10 - (1 + 1)
    assert o.state()[1].tolist() == [0.0, 10.0, 1.0, 0.25]


# ------------------------------------------------------------ counters

def brute_counters(src, dst, n, parent_after_eval, b_before_improve, b_after_eval, goals=(1,)):
    """(relaxations of the Improve on the state with b_before_improve,
    visits and levels of the Evaluate that produced b_after_eval) by brute
    force from the edge list and the policy tree."""
    indeg = np.bincount(dst, minlength=n)
    I = b_before_improve.astype(bool).copy()
    for t in goals:
        if t < n:
            I[t] = True
    I[0] = False
    relax = int(indeg[I].sum())
    X = b_after_eval.astype(bool).copy()
    X[0] = True                                       # the root is always expanded
    p = parent_after_eval
    vis = (p >= 0) & X[np.maximum(p, 0)]
    visits = int(vis.sum())
    # depth of every vertex by repeated parent steps (the policy is a forest)
    depth = np.full(n, -1, np.int64)
    depth[0] = 0
    for _ in range(n):
        pd = np.where(p >= 0, depth[np.maximum(p, 0)], -1)
        new = np.where((depth < 0) & (pd >= 0), pd + 1, depth)
        if np.array_equal(new, depth):
            break
        depth = new
    levels = int(depth[vis].max()) if visits else 0
    return relax, visits, levels


@pytest.mark.parametrize("d,n,S,boxes,seed", [(2, 800, 50, 5, 1), (3, 1500, 200, 8, 2),
                                              (6, 2500, 500, 4, 3)])
def test_counters_equal_brute_force(d, n, S, boxes, seed):
    r = gen.rrg(d, n, gen.gamma_k(d), n_boxes=boxes, seed=gen.seed_of("counters", d, seed))
    src_all, dst_all, _ = r.batch(2, n, directed=True)
    o = Oracle(h_root=r.h_root())
    ref = Oracle(h_root=r.h_root())
    checked = 0
    for a, b in [(lo, min(n, lo + S)) for lo in range(2, n, S)]:
        s, t, c = r.batch(a, b, directed=False)
        for x in (o, ref):
            x.append(r.h[a:b], s, t, c, flags=EDGES_UNDIRECTED)
        m = o.n
        sel = (src_all < m) & (dst_all < m)
        src, dst = src_all[sel], dst_all[sel]
        # the whole exploit of `ref`, against per-step brute force on `o`
        st = ref.exploit()
        tot_r = tot_v = 0
        max_l = 0
        it = ev = 0
        while True:
            b0 = o.state()[3]
            dg, _, rx = o.improve_step()
            it += 1
            br, _, _ = brute_counters(src, dst, m, o.state()[0], b0, o.state()[3])
            assert rx == br
            tot_r += rx
            checked += 1
            if dg <= 0.0:
                break
            ch, vi, lv = o.evaluate_step()
            ev += 1
            parent, _, _, b1 = o.state()
            _, bv, bl = brute_counters(src, dst, m, parent, b0, b1)
            assert (vi, lv) == (bv, bl)
            tot_v += vi
            max_l = max(max_l, lv)
        assert (st.iterations, st.evaluations) == (it, ev)
        assert (st.relaxations, st.eval_visits, st.max_level) == (tot_r, tot_v, max_l)
    assert checked > 5
