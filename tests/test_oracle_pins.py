"""Pins of the serial oracle against things other than itself (CPU only).

Each test names the passage it follows (P:n = PAPER.md line n, S:n =
SPEC.md line n) and what fixes the expected value: a worked example printed
in SPEC, a library routine (scipy Dijkstra), a closed form, or an invariant.
"""
import heapq
import math

import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import dijkstra

import gen
from oracle import EDGES_UNDIRECTED, PRUNE_OFF, Oracle, OracleError
from paper_2003_04920_b200.berrt import replay

INF = math.inf


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def in_lists(n, src, dst, cost):
    lists = [[] for _ in range(n)]
    for u, v, c in zip(src.tolist(), dst.tolist(), cost.tolist()):
        lists[v].append((u, c))
    return lists


def scipy_sssp(n, src, dst, cost):
    A = csr_matrix((cost, (src, dst)), shape=(n, n))
    dist, pred = dijkstra(A, directed=True, indices=0, return_predecessors=True)
    return dist, pred


# ----------------------------------------------------------- SPEC worked examples

def spec_triangle(relabel_goal_last: bool):
    """SPEC S:230 example: vertices {0: g=0, a: g=5 parent 0, b: g=12 parent a},
    edges (0,a,5), (a,b,7), (0,b,6) and reverses.  Our goal is vertex 1, so the
    SPEC's vertex 2 (the one whose policy improves) is placed at id 1 when
    relabel_goal_last, else SPEC ids are kept (goal = SPEC vertex 1)."""
    a, b = (2, 1) if relabel_goal_last else (1, 2)
    o = Oracle()
    src = np.array([0, a, a, b, 0, b], np.int32)
    dst = np.array([a, 0, b, a, b, 0], np.int32)
    cost = np.array([5, 5, 7, 7, 6, 6], np.float64)
    o.append(np.zeros(1), src, dst, cost)
    parent = np.full(3, -1, np.int32); g = np.zeros(3)
    parent[a], g[a] = 0, 5.0
    parent[b], g[b] = a, 12.0
    bflag = np.zeros(3, np.uint8); bflag[b] = 1        # B = {b}
    o.set_policy(parent, g, bflag)
    return o, a, b


@pytest.mark.parametrize("relabel", [False, True])
def test_spec_improve_example(relabel):
    # B={2} -> parent(2)=0, delta_g=6; g is NOT written.
    o, a, b = spec_triangle(relabel)
    dg, changed, _ = o.improve_step()
    parent, g, pc, _ = o.state()
    assert dg == 6.0 and changed == 1
    assert parent[b] == 0 and pc[b] == 6.0
    assert g[b] == 12.0 and g[a] == 5.0


@pytest.mark.parametrize("relabel", [False, True])
def test_spec_evaluate_example(relabel):
    # after the Improve above, Evaluate gives g(1)=5, g(2)=6.
    o, a, b = spec_triangle(relabel)
    o.improve_step()
    o.evaluate_step()
    _, g, _, _ = o.state()
    assert g[a] == 5.0 and g[b] == 6.0


def test_spec_replan_and_path_example():
    # converges with g(2)=6 in <= 3 iterations (2 Improves under R4);
    # path [x_init, x_2], cost 6 (SPEC vertex 2 = our goal, id 1).
    o, a, b = spec_triangle(True)
    st = o.exploit()
    assert st.iterations == 2 and st.iterations <= 3
    _, g, _, _ = o.state()
    assert g[b] == 6.0
    path, cost = o.best_path()
    assert path.tolist() == [0, 1] and cost == 6.0


def test_spec_empty_B_no_change():
    # B = {} (and the goal already optimal) -> no change, delta_g = 0.
    o, a, b = spec_triangle(True)
    o.exploit()
    before = o.state()
    st = o.exploit()
    after = o.state()
    assert st.iterations == 1 and st.last_delta_g == 0.0
    for x, y in zip(before, after):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("seed", range(6))
def test_spec_dijkstra_tree_is_fixed_point(seed):
    # parents = a Dijkstra tree -> delta_g = 0 and no parent change.
    n, m = 60, 400
    src, dst, cost = gen.random_graph(n, m, seed, max_cost=2.0)
    cost += 0.01
    dist, pred = scipy_sssp(n, src, dst, cost)
    o = Oracle()
    o.append(np.zeros(n - 2), src, dst, cost)
    parent = np.where(pred < 0, -1, pred).astype(np.int32)
    parent[0] = -1
    o.set_policy(parent, dist, np.ones(n, np.uint8) * (np.isfinite(dist)).astype(np.uint8))
    dg, changed, _ = o.improve_step()
    assert dg == 0.0 and changed == 0
    assert np.array_equal(o.state()[0], parent)


# ----------------------------------------------------- P1: PRUNE_OFF == Dijkstra

def tree_height(parent, g):
    depth = {}
    def d(v):
        if v == 0:
            return 0
        if v in depth:
            return depth[v]
        depth[v] = d(int(parent[v])) + 1
        return depth[v]
    return max((d(v) for v in range(len(parent)) if np.isfinite(g[v])), default=0)


@pytest.mark.parametrize("seed", range(8))
def test_prune_off_equals_dijkstra_random(seed):
    # Special case that reduces to a textbook routine: with I = V\{root} and
    # thr = +inf the iteration is classical policy iteration for SSSP, whose
    # fixed point is the Dijkstra shortest-path tree.  g bit-exact (one add
    # per tree edge, root->leaf), unreachable <=> +inf.  Iterations <=
    # tree height + 2.
    n, m = 120 + 10 * seed, 700 + 40 * seed
    src, dst, cost = gen.random_graph(n, m, seed, max_cost=3.0)
    cost += 1e-3
    dist, _ = scipy_sssp(n, src, dst, cost)
    o = Oracle(flags=PRUNE_OFF)
    o.append(np.zeros(n - 2), src, dst, cost)
    st = o.exploit()
    parent, g, pc, b = o.state()
    assert np.array_equal(bits(g), bits(dist))
    fin = np.isfinite(g)
    for v in np.nonzero(fin)[0]:
        if v == 0:
            continue
        assert bits(g[parent[v]] + pc[v]) == bits(g[v])
    assert st.iterations <= tree_height(parent, g) + 2


@pytest.mark.parametrize("seed", range(4))
def test_prune_off_equals_dijkstra_rrg(seed):
    r = gen.rrg(2, 1000, gen.gamma_star(2), n_boxes=5 * seed, seed=gen.seed_of("p1", seed))
    src, dst, cost = r.batch(2, r.n)
    dist, _ = scipy_sssp(r.n, src, dst, cost)
    o = Oracle(h_root=r.h_root(), flags=PRUNE_OFF)
    o.append(r.h[2:], src, dst, cost)
    st = o.exploit()
    _, g, _, _ = o.state()
    assert np.array_equal(bits(g), bits(dist))
    assert st.iterations >= 1


def test_local_relaxation_on_id_dag_equals_dijkstra():
    # R14 pin: when every edge goes from a lower to a higher id,
    # relaxing new vertices in id order is exactly DAG shortest paths, which
    # equal Dijkstra's distances (library routine), bit for bit.
    rng = np.random.default_rng(5)
    n = 400
    src, dst = [], []
    for v in range(2, n):
        for u in rng.choice(v, size=min(v, 6), replace=False):
            src.append(u); dst.append(v)
    src = np.array(src, np.int32); dst = np.array(dst, np.int32)
    cost = rng.random(src.size) + 0.05
    dist, _ = scipy_sssp(n, src, dst, cost)
    o = Oracle()
    o.append(np.zeros(n - 2), src, dst, cost)
    parent, g, pc, _ = o.state()
    mask = np.arange(n) != 1       # the goal is an old vertex: not relaxed
    assert np.array_equal(bits(g[mask]), bits(dist[mask]))
    # lowest-id argmin among exactly equal candidates (R6)
    lists = in_lists(n, src, dst, cost)
    for v in range(2, n):
        if not np.isfinite(g[v]):
            assert parent[v] == -1
            continue
        ties = [u for u, c in lists[v] if u < v and g[u] + c == g[v]]
        assert parent[v] == min(ties)


# --------------------------------------------- P2: promising-subgraph certificate

def certificate(o, src, dst, cost, goals=(1,)):
    """Bellman certificate on S = B u G (north_star: 'PI's fixed point
    must equal the shortest-path tree on the promising subgraph')."""
    parent, g, pc, b = o.state()
    n = g.size
    lists = in_lists(n, src, dst, cost)
    S = set(np.nonzero(b)[0].tolist())
    for t in goals:
        t = int(t)
        if t >= n or b[t]:
            continue
        best = min(((g[u] + c, u) for u, c in lists[t]), default=(INF, -1))
        if best[0] < g[t]:
            # a goal outside B whose best parent is not expanded keeps a stale
            # g: Improve re-selects the SAME parent and the R13 stall guard
            # ends the loop (a single goal cannot be in this state: its best
            # parent beats thr = g(goal) and is expanded)
            assert best[1] == parent[t]
        else:
            S.add(t)
    for v in S:                                     # no strict improvement (R5)
        for u, c in lists[v]:
            assert not (g[u] + c < g[v])
    for v in np.nonzero(b)[0]:                      # consistent tree on B
        p = parent[v]
        assert p == 0 or b[p] == 1
        assert bits(g[p] + pc[v]) == bits(g[v])
    # multi-source Dijkstra relaxing only into S reproduces g on S bit-exactly
    label = {v: (0.0 if v == 0 else (INF if v in S else g[v])) for v in range(n)}
    heap = [(label[v], v) for v in range(n) if v not in S]
    heapq.heapify(heap)
    done = set()
    out_lists = [[] for _ in range(n)]
    for u, v, c in zip(src.tolist(), dst.tolist(), cost.tolist()):
        out_lists[u].append((v, c))
    while heap:
        d, u = heapq.heappop(heap)
        if u in done or d > label[u]:
            continue
        done.add(u)
        for v, c in out_lists[u]:
            if v in S and v != 0 and d + c < label[v]:
                label[v] = d + c
                heapq.heappush(heap, (label[v], v))
    for v in S:
        assert bits(label[v]) == bits(g[v]), v


@pytest.mark.parametrize("seed,S,boxes", [(1, 1, 0), (2, 10, 5), (3, 50, 10), (4, 998, 0), (5, 7, 20)])
def test_promising_certificate_rrg(seed, S, boxes):
    r = gen.rrg(2, 600, gen.gamma_star(2), n_boxes=boxes, seed=gen.seed_of("p2", seed))
    o = Oracle(h_root=r.h_root())
    replay(o, r, S, undirected=True)
    src, dst, cost = r.batch(2, r.n)
    certificate(o, src, dst, cost)


# ------------------------------------------------------- P6: closed forms

def test_straight_line_lower_bound_and_5_percent():
    # Obstacle-free: g(goal) >= |x_goal - x_init| (straight line is a lower
    # bound; allow 1 ulp per path edge); N=5000 within 5% on average.
    rels = []
    for seed in range(5):
        r = gen.rrg(2, 5000, gen.gamma_star(2), seed=gen.seed_of("p6", seed))
        o = Oracle(h_root=r.h_root())
        replay(o, r, 500)
        path, c = o.best_path()
        line = r.h_root()
        assert c >= line * (1 - 1e-15 * len(path))
        pts = r.points[path]
        seg = np.sqrt(((pts[1:] - pts[:-1]) ** 2).sum(1))
        assert abs(seg.sum() - c) <= 1e-12 * c
        rels.append(c / line - 1)
    assert np.mean(rels) < 0.05


def test_direct_edge_is_optimal():
    # If the direct root-goal edge exists in a complete Euclidean graph, it is
    # the shortest path (triangle inequality), so g(goal) == c(root, goal).
    rng = np.random.default_rng(3)
    pts = np.vstack([[0.1, 0.1], [0.9, 0.9], rng.random((30, 2))])
    n = len(pts)
    src, dst = np.nonzero(~np.eye(n, dtype=bool))
    cost = np.sqrt(((pts[src] - pts[dst]) ** 2).sum(1))
    h = np.sqrt(((pts - pts[1]) ** 2).sum(1))
    o = Oracle(h_root=h[0])
    o.append(h[2:], src.astype(np.int32), dst.astype(np.int32), cost)
    o.exploit()
    path, c = o.best_path()
    direct = cost[(src == 0) & (dst == 1)][0]
    assert path.tolist() == [0, 1] and c == direct


# ------------------------------------------------- P11: unit lattice closed form

@pytest.mark.parametrize("k", [5, 12])
def test_lattice_prune_off(k):
    cells, id_of, src, dst, cost, h = gen.lattice(k)
    o = Oracle(h_root=h[0], flags=PRUNE_OFF)
    o.append(h[2:], src, dst, cost)
    st = o.exploit()
    parent, g, _, _ = o.state()
    manhattan = cells.sum(1).astype(np.float64)
    assert np.array_equal(g, manhattan)
    lists = in_lists(k * k, src, dst, cost)
    for v in range(1, k * k):
        assert parent[v] == min(u for u, _ in lists[v] if g[u] == g[v] - 1)
    assert st.iterations == 2


@pytest.mark.parametrize("k", [5, 12])
def test_lattice_north_star_snapshot(k):
    # thr is the snapshot g(goal) = +inf at the only Evaluate (R3), so every
    # non-root vertex is promising; a live threshold would give a smaller B.
    cells, id_of, src, dst, cost, h = gen.lattice(k)
    o = Oracle(h_root=h[0])
    nprom = o.append(h[2:], src, dst, cost)
    assert nprom == k * k - 2
    st = o.exploit()
    _, g, _, b = o.state()
    assert g[1] == 2 * (k - 1) and st.iterations == 2
    assert b[0] == 0 and b[1:].all()


# ----------------------------------------------------- Evaluate = path sums

@pytest.mark.parametrize("seed", range(3))
def test_evaluate_equals_root_path_sums(seed):
    # g from Evaluate equals the root->vertex path sums (left fold
    # along the path, the definition of cost-to-come along the policy).
    rng = np.random.default_rng(seed)
    n = 1000
    parent = np.full(n, -1, np.int32)
    for v in range(1, n):
        parent[v] = rng.integers(0, v) if v > 1 else 0
    w = rng.random(n) + 0.1
    src = parent[1:].copy(); dst = np.arange(1, n, dtype=np.int32)
    o = Oracle(flags=PRUNE_OFF)
    o.append(np.zeros(n - 2), src, dst, w[1:])
    g0 = np.full(n, 1e9); g0[0] = 0.0
    o.set_policy(parent, g0)
    o.evaluate_step()
    _, g, _, _ = o.state()
    for v in range(1, n):
        chain = []
        x = v
        while x != 0:
            chain.append(x); x = parent[x]
        s = 0.0
        for x in reversed(chain):
            s = s + w[x]
        assert bits(s) == bits(g[v])


# ------------------------------------------------------------- P7 invariants

@pytest.mark.parametrize("d,S,boxes", [(2, 1, 5), (2, 25, 10), (4, 100, 5)])
def test_invariants_during_replay(d, S, boxes):
    n = 800 if d == 2 else 1500
    r = gen.rrg(d, n, gen.gamma_star(d), n_boxes=boxes, seed=gen.seed_of("p7", d, S))
    o = Oracle(h_root=r.h_root())
    prev = {"g": None, "goal": INF}

    def check(k, a, b, st):
        parent, g, pc, bf = o.state()
        assert st.last_delta_g >= 0.0 or st.iterations == 0
        if prev["g"] is not None:                      # g never increases
            m = prev["g"].size
            assert np.all(g[:m] <= prev["g"])
        assert g[1] <= prev["goal"]                    # anytime monotone
        # acyclic parents: every finite-g vertex reaches the root
        for v in range(g.size):
            x, hops = v, 0
            while x not in (-1, 0):
                x = parent[x]; hops += 1
                assert hops <= g.size
        for v in np.nonzero(bf)[0]:
            assert parent[v] == 0 or bf[parent[v]]
        prev["g"], prev["goal"] = g.copy(), g[1]

    replay(o, r, S, on_exploit=check)


# ------------------------------------------------------------- P12 degenerate

def test_empty_append_and_unreachable_goal():
    o = Oracle()
    assert o.append(np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0)) == 0
    o.append(np.zeros(3), np.array([0, 2], np.int32), np.array([2, 3], np.int32), np.ones(2))
    st = o.exploit()
    path, c = o.best_path()
    assert path.size == 0 and c == INF
    assert st.iterations == 1 and st.last_delta_g == 0.0


def test_zero_cost_edges_stay_acyclic():
    src, dst, cost = gen.random_graph(80, 600, 11, max_cost=1.0, zero_cost_frac=0.3)
    o = Oracle(flags=PRUNE_OFF)
    o.append(np.zeros(78), src, dst, cost)
    o.exploit()
    parent, g, _, _ = o.state()
    for v in range(80):
        x, hops = v, 0
        while x not in (-1, 0):
            x = parent[x]; hops += 1
            assert hops <= 80


@pytest.mark.parametrize("bad", ["range", "selfloop", "nan", "neg", "h"])
def test_malformed_append_leaves_state_unchanged(bad):
    o = Oracle()
    o.append(np.zeros(2), np.array([0, 2], np.int32), np.array([2, 3], np.int32), np.ones(2))
    before = o.state()
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
    else:
        h = np.array([np.inf])
    with pytest.raises(OracleError):
        o.append(h, src, dst, cost)
    after = o.state()
    assert o.n == 4
    for x, y in zip(before, after):
        assert np.array_equal(x, y)


def test_undirected_flag_equals_both_directions():
    r = gen.rrg(2, 400, gen.gamma_star(2), n_boxes=3, seed=9)
    o1 = Oracle(h_root=r.h_root()); o2 = Oracle(h_root=r.h_root())
    replay(o1, r, 37, undirected=True)
    replay(o2, r, 37, undirected=False)
    for x, y in zip(o1.state(), o2.state()):
        assert np.array_equal(x, y)


def test_S1_and_SN_batching():
    # S = N gives exactly one replan (plus the final one is a no-op).
    r = gen.rrg(2, 300, gen.gamma_star(2), seed=4)
    o = Oracle(h_root=r.h_root())
    log = replay(o, r, r.n)
    assert len(log) == 2 and log[-1][3].iterations == 1


@pytest.mark.parametrize("seed", range(3))
def test_B_members_beat_goal_cost(seed):
    # Definition of B: promising vertices are those whose g + h
    # lower bound beats the goal cost.  After each Evaluate every member of B
    # satisfies g + h < thr, thr = g(goal) at Evaluate entry (R3); a vertex
    # whose own bound fails is never in B even if its parent's passes (R2).
    r = gen.rrg(2, 1500, gen.gamma_star(2), n_boxes=10, seed=gen.seed_of("B", seed))
    o = Oracle(h_root=r.h_root())
    replay(o, r, 1000, n_stop=1002, final=False)   # a warm state, finite g(goal)
    src, dst, cost = r.batch(1002, r.n)
    o.append(r.h[1002:], src, dst, cost)
    checked = 0
    for _ in range(20):
        dg, _, _ = o.improve_step()
        if dg == 0.0:
            break
        thr = o.state()[1][1]
        o.evaluate_step()
        _, g, _, b = o.state()
        idx = np.nonzero(b)[0]
        assert np.all(g[idx] + r.h[idx] < thr)
        checked += idx.size
    assert checked > 0


def test_gen_points_equal_rrg_samples():
    # the sampling-only generator (for the device-side Extend) reproduces the
    # full generator's boxes and points bit for bit
    for d, nb in ((2, 0), (3, 5), (6, 20)):
        r = gen.rrg(d, 3000, gen.gamma_k(d), n_boxes=nb, seed=gen.seed_of("pts", d))
        p, b = gen.points(d, 3000, nb, seed=gen.seed_of("pts", d))
        assert np.array_equal(p, r.points) and np.array_equal(b, r.boxes)
