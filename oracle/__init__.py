"""ctypes binding of the serial CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE.  Only tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2003_04920_b200`` never imports it.
Argument marshalling only: all arithmetic is in oracle.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

PRUNE_OFF = 1
VALIDATE = 2
EDGES_UNDIRECTED = 4
PARENT_FORM = 8
NEIGHBOURS = 16


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class _Stats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("last_delta_g", C.c_double),
        ("relaxations", C.c_int64),
        ("eval_visits", C.c_int64),
        ("max_level", C.c_int32),
        ("promising", C.c_int32),
        ("stalled", C.c_int32),
        ("evaluations", C.c_int32),
    ]


@dataclass
class OracleStats:
    iterations: int
    last_delta_g: float
    relaxations: int
    eval_visits: int
    max_level: int
    promising: int
    stalled: int
    evaluations: int


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not built; run `make oracle` or __graft_entry__.build()")
    lib = C.CDLL(_LIB_PATH)
    P = C.c_void_p
    lib.orc_create.restype = P
    lib.orc_create.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int32, C.c_uint32]
    lib.orc_destroy.argtypes = [P]
    lib.orc_last_error.restype = C.c_char_p
    lib.orc_num_vertices.restype = C.c_int64
    lib.orc_num_vertices.argtypes = [P]
    lib.orc_append.argtypes = [P, C.c_int32, P, P, P, C.c_int64, P, P, P, C.c_uint32, P]
    lib.orc_exploit.argtypes = [P, C.POINTER(_Stats)]
    lib.orc_improve_step.argtypes = [P, P, P, P]
    lib.orc_evaluate_step.argtypes = [P, P, P, P]
    lib.orc_get_state.argtypes = [P, P, P, P, P, C.c_int64]
    lib.orc_set_policy.argtypes = [P, P, P, P]
    lib.orc_best_path.argtypes = [P, P, C.c_int64, P, P, P]
    lib.orc_set_goals.argtypes = [P, P, C.c_int32]
    _lib = lib
    return lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class Oracle:
    """One oracle context: vertices 0 (x_init) and 1 (x_goal) exist on creation."""

    def __init__(self, h_root=0.0, h_goal=0.0, epsilon=0.0, max_iterations=0, flags=0):
        self._lib = _load()
        self._c = self._lib.orc_create(float(h_root), float(h_goal), float(epsilon),
                                       int(max_iterations), int(flags))
        if not self._c:
            raise OracleError(-1, self._lib.orc_last_error().decode())

    def close(self):
        if self._c:
            self._lib.orc_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._lib.orc_last_error().decode())

    @property
    def n(self) -> int:
        return int(self._lib.orc_num_vertices(self._c))

    def append(self, h_new, src, dst, cost, parent_new=None, g_new=None, flags=0) -> int:
        h_new = np.ascontiguousarray(h_new, dtype=np.float64)
        src = np.ascontiguousarray(src, dtype=np.int32)
        dst = np.ascontiguousarray(dst, dtype=np.int32)
        cost = np.ascontiguousarray(cost, dtype=np.float64)
        if parent_new is not None:
            parent_new = np.ascontiguousarray(parent_new, dtype=np.int32)
            g_new = np.ascontiguousarray(g_new, dtype=np.float64)
        out = np.zeros(1, dtype=np.int32)
        self._check(self._lib.orc_append(self._c, int(h_new.size), _ptr(h_new), _ptr(parent_new),
                                         _ptr(g_new), int(src.size), _ptr(src), _ptr(dst),
                                         _ptr(cost), int(flags), _ptr(out)))
        return int(out[0])

    def exploit(self, allow_noconv=False) -> OracleStats:
        st = _Stats()
        rc = self._lib.orc_exploit(self._c, C.byref(st))
        if rc != 0 and not (allow_noconv and rc == -6):
            self._check(rc)
        return OracleStats(*(getattr(st, f[0]) for f in _Stats._fields_))

    def improve_step(self):
        dg = np.zeros(1, np.float64); ch = np.zeros(1, np.int32); rx = np.zeros(1, np.int64)
        self._check(self._lib.orc_improve_step(self._c, _ptr(dg), _ptr(ch), _ptr(rx)))
        return float(dg[0]), int(ch[0]), int(rx[0])

    def evaluate_step(self):
        ch = np.zeros(1, np.int32); vi = np.zeros(1, np.int64); lv = np.zeros(1, np.int32)
        self._check(self._lib.orc_evaluate_step(self._c, _ptr(ch), _ptr(vi), _ptr(lv)))
        return int(ch[0]), int(vi[0]), int(lv[0])

    def state(self):
        n = self.n
        parent = np.empty(n, np.int32); g = np.empty(n, np.float64)
        pc = np.empty(n, np.float64); b = np.empty(n, np.uint8)
        self._check(self._lib.orc_get_state(self._c, _ptr(parent), _ptr(g), _ptr(pc), _ptr(b), n))
        return parent, g, pc, b

    def set_policy(self, parent, g, b=None):
        parent = np.ascontiguousarray(parent, dtype=np.int32)
        g = np.ascontiguousarray(g, dtype=np.float64)
        if b is not None:
            b = np.ascontiguousarray(b, dtype=np.uint8)
        self._check(self._lib.orc_set_policy(self._c, _ptr(parent), _ptr(g), _ptr(b)))

    def set_goals(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        self._check(self._lib.orc_set_goals(self._c, _ptr(ids), int(ids.size)))

    def best_path_goal(self):
        """(path root..goal, cost, best goal id or -1)."""
        cap = self.n
        path = np.empty(max(cap, 1), np.int32)
        ln = np.zeros(1, np.int64); cost = np.zeros(1, np.float64); goal = np.zeros(1, np.int32)
        self._check(self._lib.orc_best_path(self._c, _ptr(path), cap, _ptr(ln), _ptr(cost),
                                            _ptr(goal)))
        return path[: int(ln[0])].copy(), float(cost[0]), int(goal[0])

    def best_path(self):
        path, cost, _ = self.best_path_goal()
        return path, cost
