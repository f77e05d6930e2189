"""Seeded synthetic input generators (shared by the oracle side and the CUDA side).

Holds none of the method's arithmetic: only points, edge costs (Euclidean),
the heuristic h, and batch slicing.  See DESIGN.md section 4 for the recipe.

* :func:`rrg` -- random geometric graph with box obstacles and the incremental
  connection radius r(m) = gamma (ln m / m)^(1/d) (C++ in gen/rrg.cpp).
* :func:`gamma_star`, :func:`gamma_k` -- the two radius constants.
* :func:`random_graph`, :func:`lattice` -- tiny graphs for oracle pins.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built; run `make gen`")
        lib = C.CDLL(_LIB_PATH)
        lib.gen_rrg.restype = C.c_void_p
        lib.gen_rrg.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_int, C.c_double,
                                C.c_double, C.c_uint64, C.c_int]
        lib.gen_sizes.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        lib.gen_copy.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        lib.gen_free.argtypes = [C.c_void_p]
        lib.gen_points.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_double, C.c_double,
                                   C.c_uint64, C.c_void_p, C.c_void_p]
        _lib = lib
    return _lib


def seed_of(*parts) -> int:
    """Deterministic 64-bit seed from a tuple of config values (0x5EED-salted)."""
    h = hashlib.sha256(("0x5EED|" + "|".join(str(p) for p in parts)).encode()).digest()
    return int.from_bytes(h[:8], "little")


def unit_ball_volume(d: int) -> float:
    return math.pi ** (d / 2) / math.gamma(d / 2 + 1)


def gamma_star(d: int, mu_free: float = 1.0) -> float:
    """RRG/PRM* connectivity constant 2(1+1/d)^(1/d) (mu_free/zeta_d)^(1/d)."""
    return 2.0 * (1.0 + 1.0 / d) ** (1.0 / d) * (mu_free / unit_ball_volume(d)) ** (1.0 / d)


def gamma_k(d: int, mu_free: float = 1.0) -> float:
    """kPRM-equivalent constant (e (1+1/d) mu_free / zeta_d)^(1/d)."""
    return (math.e * (1.0 + 1.0 / d) * mu_free / unit_ball_volume(d)) ** (1.0 / d)


@dataclass
class RRG:
    d: int
    n: int
    gamma: float
    points: np.ndarray      # (n, d) f64
    boxes: np.ndarray       # (n_boxes, 2, d) f64
    h: np.ndarray           # (n,) f64, Euclidean distance to x_goal (h[1] = 0)
    off: np.ndarray         # (n+1,) i64: earlier-neighbour lists of vertex i
    nbr: np.ndarray         # (pairs,) i32: neighbour j < i
    cost: np.ndarray        # (pairs,) f64: |x_i - x_j|
    n_isolated: int
    n_candidates: int

    @property
    def n_pairs(self) -> int:
        return int(self.off[-1])

    @property
    def mean_degree(self) -> float:
        return 2.0 * self.n_pairs / self.n

    def h_root(self) -> float:
        return float(self.h[0])

    def batch(self, a: int, b: int, directed: bool = True):
        """Edges of new vertices [a, b) (a >= 2) to all earlier vertices.

        directed=True returns both directions (src, dst, cost) with j->i first
        then i->j per pair; directed=False returns each pair once (src=j,
        dst=i) for use with the EDGES_UNDIRECTED flag."""
        assert 2 <= a <= b <= self.n
        lo, hi = int(self.off[a]), int(self.off[b])
        j = self.nbr[lo:hi]
        i = np.repeat(np.arange(a, b, dtype=np.int32), np.diff(self.off[a:b + 1]).astype(np.int64))
        c = self.cost[lo:hi]
        if not directed:
            return j.copy(), i, c.copy()
        src = np.empty(2 * j.size, np.int32)
        dst = np.empty(2 * j.size, np.int32)
        cost = np.empty(2 * j.size, np.float64)
        src[0::2], dst[0::2], cost[0::2] = j, i, c
        src[1::2], dst[1::2], cost[1::2] = i, j, c
        return src, dst, cost


def rrg(d: int, n: int, gamma: float, n_boxes: int = 0, side=(0.05, 0.3), seed: int = 1,
        threads: int = 0) -> RRG:
    lib = _load()
    h = lib.gen_rrg(int(d), int(n), float(gamma), int(n_boxes), float(side[0]), float(side[1]),
                    C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(threads))
    if not h:
        raise ValueError("gen_rrg: bad arguments")
    try:
        sz = np.zeros(4, np.int64)
        lib.gen_sizes(h, sz[0:].ctypes.data, sz[1:].ctypes.data, sz[2:].ctypes.data,
                      sz[3:].ctypes.data)
        nn, pairs = int(sz[0]), int(sz[1])
        pts = np.empty((nn, d), np.float64)
        boxes = np.empty((n_boxes, 2, d), np.float64)
        hv = np.empty(nn, np.float64)
        off = np.empty(nn + 1, np.int64)
        nbr = np.empty(pairs, np.int32)
        cost = np.empty(pairs, np.float64)
        lib.gen_copy(h, pts.ctypes.data, boxes.ctypes.data if n_boxes else None, hv.ctypes.data,
                     off.ctypes.data, nbr.ctypes.data, cost.ctypes.data)
        return RRG(d, nn, gamma, pts, boxes, hv, off, nbr, cost, int(sz[2]), int(sz[3]))
    finally:
        lib.gen_free(h)


def points(d: int, n: int, n_boxes: int = 0, side=(0.05, 0.3), seed: int = 1):
    """Only the samples of rrg(...) with the same arguments: (points (n, d),
    boxes (n_boxes, 2, d)) -- for the device-side Extend, which builds the
    edges itself."""
    lib = _load()
    pts = np.empty((n, d), np.float64)
    boxes = np.empty((max(n_boxes, 0), 2, d), np.float64)
    rc = lib.gen_points(int(d), int(n), int(n_boxes), float(side[0]), float(side[1]),
                        C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), boxes.ctypes.data, pts.ctypes.data)
    if rc != 0:
        raise ValueError("gen_points: bad arguments")
    return pts, boxes


# ---------------------------------------------------------------- tiny graphs

def random_graph(n: int, m: int, seed: int, max_cost: float = 1.0, integer_costs: bool = False,
                 zero_cost_frac: float = 0.0):
    """Random directed simple graph on n vertices with m edges (no self loops,
    no duplicates), random costs, random admissible-looking h (h = 0)."""
    rng = np.random.default_rng(seed)
    pairs = set()
    src, dst = [], []
    limit = n * (n - 1)
    m = min(m, limit)
    while len(src) < m:
        u, v = rng.integers(0, n, size=2)
        if u == v or (u, v) in pairs:
            continue
        pairs.add((int(u), int(v)))
        src.append(int(u)); dst.append(int(v))
    if integer_costs:
        cost = rng.integers(1, 10, size=m).astype(np.float64)
    else:
        cost = rng.random(m) * max_cost
    if zero_cost_frac > 0:
        cost[rng.random(m) < zero_cost_frac] = 0.0
    return np.array(src, np.int32), np.array(dst, np.int32), cost


def lattice(k: int):
    """k x k 4-connected unit lattice.  Vertex 0 = corner (0,0) = x_init,
    vertex 1 = corner (k-1,k-1) = x_goal, vertices 2.. = the remaining cells in
    row-major order.  Returns (cell_of_id (k*k,2), id_of_cell (k,k), src, dst,
    cost (both directions, unit), h = Manhattan distance to the goal)."""
    order = [(0, 0), (k - 1, k - 1)] + [(r, c) for r in range(k) for c in range(k)
                                       if (r, c) not in ((0, 0), (k - 1, k - 1))]
    id_of = np.empty((k, k), np.int32)
    for i, (r, c) in enumerate(order):
        id_of[r, c] = i
    src, dst = [], []
    for r in range(k):
        for c in range(k):
            for dr, dc in ((0, 1), (1, 0)):
                r2, c2 = r + dr, c + dc
                if r2 < k and c2 < k:
                    a, b = int(id_of[r, c]), int(id_of[r2, c2])
                    src += [a, b]; dst += [b, a]
    cells = np.array(order, np.int64)
    h = ((k - 1 - cells[:, 0]) + (k - 1 - cells[:, 1])).astype(np.float64)
    return cells, id_of, np.array(src, np.int32), np.array(dst, np.int32), \
        np.ones(len(src), np.float64), h
