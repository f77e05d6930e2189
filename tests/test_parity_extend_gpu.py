"""Device-side Extend: pirrt_extend_batch builds the
batch's edges on the GPU from the sample points.  The edge set is pinned to
the CPU generator (gen/rrg.cpp, the recipe of DESIGN.md section 4) on the same
points, and the PI state after every batch to the oracle replaying the
generator's edges -- bit for bit.  Run on a B200: -m gpu."""
import numpy as np
import pytest

import gen
from oracle import EDGES_UNDIRECTED, Oracle
from parity import assert_same_edge_set, assert_same_state, assert_same_stats
from paper_2003_04920_b200.berrt import batches

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2003_04920_b200 import pirrt
    return pirrt


@pytest.mark.parametrize("d,n,S,boxes,gk", [
    (2, 300, 7, 0, "star"),        # brute force (few points: coarse grid)
    (2, 6000, 97, 25, "star"),     # 2-D grid, cluttered
    (2, 3000, 1, 10, "k"),         # S = 1 (PI-RRT#)
    (4, 8000, 500, 10, "k"),
    (6, 20000, 2000, 20, "k"),
    (7, 6000, 600, 30, "star"),
])
def test_extend_matches_generator_and_oracle(P, d, n, S, boxes, gk):
    gamma = gen.gamma_star(d) if gk == "star" else gen.gamma_k(d)
    r = gen.rrg(d, n, gamma, n_boxes=boxes, seed=gen.seed_of("extend", d, n, S))
    gpu = P.Context(h_root=r.h_root())
    gpu.set_world(d, r.boxes, r.points[0], r.points[1], gamma)
    orc = Oracle(h_root=r.h_root())
    for k, (a, b) in enumerate(batches(r.n, S)):
        pg, ne = gpu.extend(r.points[a:b])
        src, dst, cost = r.batch(a, b, directed=False)
        assert ne == src.size, f"batch {k}: {ne} edges on the GPU, generator {src.size}"
        po = orc.append(r.h[a:b], src, dst, cost, flags=EDGES_UNDIRECTED)
        assert pg == po, f"batch {k}: n_new_promising {pg} vs {po}"
        if po > 0:
            assert_same_stats(gpu.exploit(), orc.exploit(), f"batch {k}")
    assert_same_stats(gpu.exploit(), orc.exploit(), "final")
    assert_same_state(gpu, orc, "final")
    assert gpu.n_edges == 2 * r.n_pairs
    assert np.array_equal(gpu.points(), r.points)
    # the edge set itself, element by element: every directed (u, v, c(u, v))
    # of the generator, cost bitwise (not only the counts)
    src, dst, cost = r.batch(2, r.n, directed=True)
    assert_same_edge_set(gpu, src, dst, cost, "extend")


def test_extend_device_points_and_guards(P):
    import torch
    r = gen.rrg(3, 3000, gen.gamma_k(3), n_boxes=5, seed=gen.seed_of("extend-dev"))
    gpu = P.Context(h_root=r.h_root())
    with pytest.raises(P.PirrtError) as ei:
        gpu.extend(r.points[2:10])                     # no world yet
    assert ei.value.code == P.PIRRT_E_STATE
    gpu.set_world(3, r.boxes, r.points[0], r.points[1], gen.gamma_k(3))
    orc = Oracle(h_root=r.h_root())
    for a, b in batches(r.n, 400):
        pg, _ = gpu.extend(torch.from_numpy(np.ascontiguousarray(r.points[a:b])).cuda())
        s, d_, c = r.batch(a, b, directed=False)
        assert pg == orc.append(r.h[a:b], s, d_, c, flags=EDGES_UNDIRECTED)
        if pg > 0:
            assert_same_stats(gpu.exploit(), orc.exploit())
    assert_same_state(gpu, orc)
    with pytest.raises(P.PirrtError) as ei:                 # plain appends are refused now
        gpu.append(np.zeros(1), np.array([0], np.int32), np.array([r.n], np.int32), np.ones(1))
    assert ei.value.code == P.PIRRT_E_STATE
    with pytest.raises(P.PirrtError) as ei:                 # the world is set once, first
        gpu.set_world(3, r.boxes, r.points[0], r.points[1], 1.0)
    assert ei.value.code == P.PIRRT_E_STATE
