"""Thin ctypes binding of the C ABI in include/pirrt.h (libpirrt.so).

Argument marshalling only: every step of the exploitation path runs in the
CUDA kernels of ``csrc/``.  Importing this module loads the in-tree
``lib/libpirrt.so`` and raises ImportError if it is missing -- there is no
CPU fallback.

Functions keep the ABI names (``pirrt_create``, ``pirrt_graph_append_batch``,
``pirrt_exploit``, ``pirrt_get_policy``, ``pirrt_get_costs``,
``pirrt_best_path`` ...); :class:`Context` wraps them for numpy arrays (host
pointers) and torch CUDA tensors (``PIRRT_F_DEVICE_PTRS``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIRRT_LIB") or os.path.join(_HERE, "lib", "libpirrt.so")

PIRRT_OK = 0
PIRRT_E_INVAL = -1
PIRRT_E_RANGE = -2
PIRRT_E_NOMEM = -3
PIRRT_E_CUDA = -4
PIRRT_E_NCCL = -5
PIRRT_E_NOCONV = -6
PIRRT_E_STATE = -7
PIRRT_E_CORRUPT = -8

PIRRT_F_PRUNE_OFF = 1
PIRRT_F_VALIDATE = 2
PIRRT_F_EDGES_UNDIRECTED = 4
PIRRT_F_DEVICE_PTRS = 8
PIRRT_F_SHARDED = 16
PIRRT_F_PARENT_FORM = 32
PIRRT_F_NEIGHBOURS = 64
PIRRT_F_LOCAL_GROUP = 128
NCCL_UNIQUE_ID_BYTES = 128
CUDA_STREAM_LEGACY = 1      # cudaStreamLegacy

# every symbol include/pirrt.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "pirrt_config_init", "pirrt_create", "pirrt_destroy", "pirrt_graph_append_batch",
    "pirrt_exploit", "pirrt_exploit_async", "pirrt_exploit_wait", "pirrt_get_policy",
    "pirrt_get_costs", "pirrt_get_promising", "pirrt_get_parent_costs", "pirrt_get_in_edges", "pirrt_best_path", "pirrt_set_policy", "pirrt_num_vertices",
    "pirrt_num_edges", "pirrt_kernel_launches", "pirrt_last_error", "pirrt_nccl_unique_id", "pirrt_group_exploit",
    "pirrt_set_world", "pirrt_extend_batch", "pirrt_get_points",
    "pirrt_step_async", "pirrt_step_wait", "pirrt_steps_outstanding",
    # include/pirrt_bench.h (measurement helpers)
    "pirrt_bench_rows", "pirrt_bench_relax", "pirrt_bench_gather", "pirrt_bench_relax_ctx",
)


class pirrt_config(C.Structure):
    _fields_ = [
        ("vertex_capacity", C.c_int64),
        ("edge_capacity", C.c_int64),
        ("h_root", C.c_double),
        ("h_goal", C.c_double),
        ("epsilon", C.c_double),
        ("max_iterations", C.c_int32),
        ("flags", C.c_uint32),
        ("device", C.c_int32),
        ("stream", C.c_void_p),
        ("grid_blocks", C.c_int32),
        ("nranks", C.c_int32),
        ("rank", C.c_int32),
        ("nccl_unique_id", C.c_void_p),
        ("goals", C.c_void_p),
        ("n_goals", C.c_int32),
        ("root", C.c_int32),
        ("goal", C.c_int32),
    ]


class pirrt_exploit_stats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("evaluations", C.c_int32),
        ("last_delta_g", C.c_double),
        ("relaxations", C.c_int64),
        ("eval_visits", C.c_int64),
        ("max_level", C.c_int32),
        ("promising", C.c_int32),
        ("stalled", C.c_int32),
        ("grid_blocks", C.c_int32),
        ("device_ms", C.c_float),
        ("improve_ms", C.c_float),
        ("evaluate_ms", C.c_float),
        ("barriers", C.c_int32),
        ("improve_set", C.c_int64),
        ("eval_scanned", C.c_int64),
        ("eval_work", C.c_int64),
        ("full_evaluations", C.c_int32),
        ("inc_evaluations", C.c_int32),
        ("relax_work", C.c_int64),
        ("improve_work", C.c_int64),
        ("inc_improves", C.c_int32),
        ("pad_", C.c_int32),
    ]


class pirrt_step_result(C.Structure):
    _fields_ = [
        ("n_new_promising", C.c_int32),
        ("replanned", C.c_int32),
        ("path_len", C.c_int64),
        ("path_cost", C.c_double),
        ("goal", C.c_int32),
        ("pad_", C.c_int32),
        ("stats", pirrt_exploit_stats),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make cuda` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    lib.pirrt_config_init.argtypes = [C.POINTER(pirrt_config)]
    lib.pirrt_config_init.restype = None
    lib.pirrt_create.argtypes = [C.POINTER(pirrt_config), C.POINTER(C.c_void_p)]
    lib.pirrt_destroy.argtypes = [P]
    lib.pirrt_graph_append_batch.argtypes = [P, C.c_int32, P, P, P, C.c_int64, P, P, P,
                                             C.c_uint32, P]
    lib.pirrt_exploit.argtypes = [P, C.POINTER(pirrt_exploit_stats)]
    lib.pirrt_exploit_async.argtypes = [P]
    lib.pirrt_set_world.argtypes = [P, C.c_int32, C.c_int32, P, P, P, C.c_double]
    lib.pirrt_extend_batch.argtypes = [P, C.c_int32, P, C.c_uint32, P, P]
    lib.pirrt_get_points.argtypes = [P, P, C.c_int64]
    lib.pirrt_exploit_wait.argtypes = [P, C.POINTER(pirrt_exploit_stats)]
    lib.pirrt_step_async.argtypes = [P, C.c_int32, P, C.c_int64, P, P, P, C.c_uint32]
    lib.pirrt_step_wait.argtypes = [P, C.POINTER(pirrt_step_result), P, C.c_int64]
    lib.pirrt_steps_outstanding.argtypes = [P]
    for f in ("pirrt_get_policy", "pirrt_get_costs", "pirrt_get_promising",
              "pirrt_get_parent_costs"):
        getattr(lib, f).argtypes = [P, P, C.c_int64]
    lib.pirrt_get_in_edges.argtypes = [P, P, C.c_int64, P, P, C.c_int64]
    lib.pirrt_best_path.argtypes = [P, P, C.c_int64, P, P, P]
    lib.pirrt_set_policy.argtypes = [P, P, P, P]
    lib.pirrt_num_vertices.argtypes = [P]
    lib.pirrt_num_vertices.restype = C.c_int64
    lib.pirrt_num_edges.argtypes = [P]
    lib.pirrt_num_edges.restype = C.c_int64
    lib.pirrt_kernel_launches.argtypes = [P]
    lib.pirrt_kernel_launches.restype = C.c_int64
    lib.pirrt_last_error.restype = C.c_char_p
    lib.pirrt_nccl_unique_id.argtypes = [P, C.c_int64]
    lib.pirrt_group_exploit.argtypes = [P, C.c_int32, P]
    lib.pirrt_bench_rows.argtypes = [P, P, P, P, C.c_int32, C.c_int32, P]
    lib.pirrt_bench_gather.argtypes = [P, P, C.c_int64, C.c_int32, P]
    lib.pirrt_bench_relax.argtypes = [P, P, P, P, P, C.c_int32, P, C.c_int32, P]
    lib.pirrt_bench_relax_ctx.argtypes = [P, C.c_int32, P, P]
    return lib


_lib = _load()

# ABI-named entry points (same names as include/pirrt.h)
pirrt_config_init = _lib.pirrt_config_init
pirrt_create = _lib.pirrt_create
pirrt_destroy = _lib.pirrt_destroy
pirrt_graph_append_batch = _lib.pirrt_graph_append_batch
pirrt_exploit = _lib.pirrt_exploit
pirrt_exploit_async = _lib.pirrt_exploit_async
pirrt_set_world = _lib.pirrt_set_world
pirrt_extend_batch = _lib.pirrt_extend_batch
pirrt_get_points = _lib.pirrt_get_points
pirrt_exploit_wait = _lib.pirrt_exploit_wait
pirrt_step_async = _lib.pirrt_step_async
pirrt_step_wait = _lib.pirrt_step_wait
pirrt_steps_outstanding = _lib.pirrt_steps_outstanding
pirrt_get_policy = _lib.pirrt_get_policy
pirrt_get_costs = _lib.pirrt_get_costs
pirrt_get_promising = _lib.pirrt_get_promising
pirrt_get_parent_costs = _lib.pirrt_get_parent_costs
pirrt_get_in_edges = _lib.pirrt_get_in_edges
pirrt_best_path = _lib.pirrt_best_path
pirrt_set_policy = _lib.pirrt_set_policy
pirrt_num_vertices = _lib.pirrt_num_vertices
pirrt_num_edges = _lib.pirrt_num_edges
pirrt_kernel_launches = _lib.pirrt_kernel_launches
pirrt_last_error = _lib.pirrt_last_error
pirrt_nccl_unique_id = _lib.pirrt_nccl_unique_id
pirrt_group_exploit = _lib.pirrt_group_exploit


def bench_rows(off, idx, cost, order, reps=5) -> float:
    """ms per pass streaming CSR rows in `order` (torch CUDA tensors)."""
    ms = C.c_float(0)
    _check(_lib.pirrt_bench_rows(off.data_ptr(), idx.data_ptr(), cost.data_ptr(), order.data_ptr(),
                                 int(order.numel()), int(reps), C.byref(ms)))
    return float(ms.value)


def bench_relax(off, idx, cost, g, order, out, reps=5) -> float:
    """ms per relaxation pass over the rows in `order` (torch CUDA tensors)."""
    ms = C.c_float(0)
    _check(_lib.pirrt_bench_relax(off.data_ptr(), idx.data_ptr(), cost.data_ptr(), g.data_ptr(),
                                  order.data_ptr(), int(order.numel()), out.data_ptr(), int(reps),
                                  C.byref(ms)))
    return float(ms.value)


def bench_relax_ctx(ctx, reps=5):
    """(ms per pass, entries per pass) of the relaxation microbenchmark over
    the context's own base CSR (pirrt_bench_relax_ctx)."""
    ms = C.c_float(0)
    ent = C.c_int64(0)
    _check(_lib.pirrt_bench_relax_ctx(ctx._h, int(reps), C.byref(ms), C.byref(ent)))
    return float(ms.value), int(ent.value)


def bench_gather(src, idx, reps=5) -> float:
    """ms per pass of idx.numel() random 8-byte gathers from src (torch CUDA tensors)."""
    ms = C.c_float(0)
    _check(_lib.pirrt_bench_gather(src.data_ptr(), idx.data_ptr(), int(idx.numel()), int(reps),
                                   C.byref(ms)))
    return float(ms.value)


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for a sharded context group."""
    buf = C.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    _check(pirrt_nccl_unique_id(buf, NCCL_UNIQUE_ID_BYTES))
    return buf.raw


class PirrtError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pirrt error {code}: {msg}")
        self.code = code


def _check(rc: int):
    if rc != PIRRT_OK:
        raise PirrtError(rc, (_lib.pirrt_last_error() or b"").decode())


@dataclass
class ExploitStats:
    iterations: int
    evaluations: int
    last_delta_g: float
    relaxations: int
    eval_visits: int
    max_level: int
    promising: int
    stalled: int
    grid_blocks: int
    device_ms: float
    improve_ms: float
    evaluate_ms: float
    barriers: int
    improve_set: int
    eval_scanned: int
    eval_work: int
    full_evaluations: int
    inc_evaluations: int
    relax_work: int
    improve_work: int
    inc_improves: int
    pad_: int


@dataclass
class StepResult:
    """pirrt_step_wait: one deferred BE-RRT# step's result."""
    n_new_promising: int
    replanned: bool
    stats: ExploitStats | None      # None when the Alg. 3 guard skipped the Replan
    path: np.ndarray
    cost: float
    goal: int


def _is_torch_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


# dtype each device-pointer argument must have (the C ABI reinterprets the
# memory: int32 ids, float64 costs / h / g / points)
_DEV_DTYPES = {"h_new": "float64", "src": "int32", "dst": "int32", "cost": "float64",
               "parent_new": "int32", "g_new": "float64", "points": "float64"}


def _check_device_tensors(device: int, sizes: dict, **tensors):
    """Device-pointer inputs: every tensor a contiguous torch CUDA tensor of
    the ABI's dtype on the context's device, with the stated element count."""
    for name, t in tensors.items():
        if t is None:
            continue
        if not _is_torch_cuda(t):
            raise PirrtError(PIRRT_E_INVAL, f"{name}: device-pointer append needs every input "
                                            "as a torch CUDA tensor")
        want = _DEV_DTYPES[name]
        if str(t.dtype) != f"torch.{want}":
            raise PirrtError(PIRRT_E_INVAL, f"{name}: dtype {t.dtype}, the ABI needs {want}")
        if not t.is_contiguous():
            raise PirrtError(PIRRT_E_INVAL, f"{name}: tensor is not contiguous")
        if t.device.index != device:
            raise PirrtError(PIRRT_E_INVAL, f"{name}: on {t.device}, the context is on cuda:{device}")
        if name in sizes and int(t.numel()) != sizes[name]:
            raise PirrtError(PIRRT_E_INVAL, f"{name}: {t.numel()} elements, expected {sizes[name]}")


def group_exploit(contexts) -> list:
    """pirrt_group_exploit over an in-process group (contexts[i] = rank i,
    created with nranks=len(contexts), rank=i, flags |= PIRRT_F_LOCAL_GROUP)."""
    n = len(contexts)
    hs = (C.c_void_p * n)(*[c._h for c in contexts])
    st = (pirrt_exploit_stats * n)()
    _check(pirrt_group_exploit(hs, n, st))
    return [ExploitStats(*(getattr(x, f[0]) for f in pirrt_exploit_stats._fields_)) for x in st]


class Context:
    """One exploitation context (vertices 0 = x_init and 1 = x_goal exist)."""

    def __init__(self, h_root=0.0, h_goal=0.0, epsilon=0.0, max_iterations=0, flags=0, device=0,
                 stream=None, vertex_capacity=0, edge_capacity=0, grid_blocks=0, nranks=1,
                 rank=0, nccl_id: bytes | None = None, goals=None):
        if (int(nranks) > 1 or int(flags) & PIRRT_F_SHARDED) and not int(flags) & PIRRT_F_LOCAL_GROUP:
            # libpirrt dlopens libnccl.so.2: let torch load its own build of
            # it first (same soname), so that a later `import torch` does not
            # bind to a different NCCL
            import torch  # noqa: F401
        cfg = pirrt_config()
        pirrt_config_init(C.byref(cfg))
        cfg.h_root, cfg.h_goal, cfg.epsilon = float(h_root), float(h_goal), float(epsilon)
        cfg.max_iterations, cfg.flags, cfg.device = int(max_iterations), int(flags), int(device)
        cfg.vertex_capacity, cfg.edge_capacity = int(vertex_capacity), int(edge_capacity)
        cfg.grid_blocks = int(grid_blocks)
        cfg.nranks, cfg.rank = int(nranks), int(rank)
        self._nccl_id = None
        if nccl_id is not None:
            self._nccl_id = C.create_string_buffer(bytes(nccl_id), NCCL_UNIQUE_ID_BYTES)
            cfg.nccl_unique_id = C.cast(self._nccl_id, C.c_void_p)
        if stream is not None:
            h = int(getattr(stream, "cuda_stream", stream))
            # torch's default stream is the legacy NULL stream (handle 0),
            # which the ABI reads as "create your own": pass cudaStreamLegacy
            # so that the work is ordered with the caller's default stream
            cfg.stream = h if h != 0 else CUDA_STREAM_LEGACY
        goal_arr = None
        if goals is not None and len(goals) > 0:
            goal_arr = np.ascontiguousarray(goals, dtype=np.int32)
            cfg.goals, cfg.n_goals = goal_arr.ctypes.data, int(goal_arr.size)
        h = C.c_void_p()
        _check(pirrt_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self.cfg = cfg

    def close(self):
        if getattr(self, "_h", None):
            pirrt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        return int(pirrt_num_vertices(self._h))

    @property
    def kernel_launches(self) -> int:
        return int(pirrt_kernel_launches(self._h))

    @property
    def n_edges(self) -> int:
        return int(pirrt_num_edges(self._h))

    def append(self, h_new, src, dst, cost, parent_new=None, g_new=None, flags=0) -> int:
        """pirrt_graph_append_batch.  numpy arrays -> host pointers; torch CUDA
        tensors (all of them) -> PIRRT_F_DEVICE_PTRS."""
        if any(_is_torch_cuda(x) for x in (h_new, src, dst, cost, parent_new, g_new)):
            flags |= PIRRT_F_DEVICE_PTRS
            ptr = lambda t: None if t is None else t.data_ptr()
            nn, m = int(h_new.numel()), int(src.numel())
            _check_device_tensors(int(self.cfg.device),
                                  {"dst": m, "cost": m, "parent_new": nn, "g_new": nn},
                                  h_new=h_new, src=src, dst=dst, cost=cost,
                                  parent_new=parent_new, g_new=g_new)
            keep = ()
        else:
            h_new = np.ascontiguousarray(h_new, np.float64)
            src = np.ascontiguousarray(src, np.int32)
            dst = np.ascontiguousarray(dst, np.int32)
            cost = np.ascontiguousarray(cost, np.float64)
            if parent_new is not None:
                parent_new = np.ascontiguousarray(parent_new, np.int32)
                g_new = np.ascontiguousarray(g_new, np.float64)
            ptr = lambda a: None if a is None else (a.ctypes.data if a.size else None)
            nn, m = int(h_new.size), int(src.size)
            keep = (h_new, src, dst, cost, parent_new, g_new)
        out = C.c_int32(0)
        _check(pirrt_graph_append_batch(self._h, nn, ptr(h_new), ptr(parent_new), ptr(g_new), m,
                                        ptr(src), ptr(dst), ptr(cost), int(flags), C.byref(out)))
        del keep
        return int(out.value)

    def exploit(self) -> ExploitStats:
        st = pirrt_exploit_stats()
        _check(pirrt_exploit(self._h, C.byref(st)))
        return ExploitStats(*(getattr(st, f[0]) for f in pirrt_exploit_stats._fields_))

    def set_world(self, d, boxes, x_init, x_goal, gamma):
        """pirrt_set_world: [0,1]^d, boxes (n_boxes, 2, d), x_init, x_goal, gamma."""
        boxes = np.ascontiguousarray(boxes, np.float64).reshape(-1)
        xi = np.ascontiguousarray(x_init, np.float64)
        xg = np.ascontiguousarray(x_goal, np.float64)
        nb = boxes.size // (2 * int(d))
        _check(pirrt_set_world(self._h, int(d), nb, boxes.ctypes.data if nb else None,
                               xi.ctypes.data, xg.ctypes.data, float(gamma)))
        self.d = int(d)

    def extend(self, points, flags=0):
        """pirrt_extend_batch: (n_new_promising, undirected pairs created)."""
        nprom, ne = C.c_int32(0), C.c_int64(0)
        if _is_torch_cuda(points):
            flags |= PIRRT_F_DEVICE_PTRS
            _check_device_tensors(int(self.cfg.device), {}, points=points)
            if points.dim() != 2 or int(points.shape[1]) != self.d:
                raise PirrtError(PIRRT_E_INVAL, f"points: shape {tuple(points.shape)}, "
                                                f"expected (n, {self.d})")
            n, ptr = int(points.shape[0]), points.data_ptr()
        else:
            points = np.ascontiguousarray(points, np.float64)
            n, ptr = int(points.shape[0]), (points.ctypes.data if points.size else None)
        _check(pirrt_extend_batch(self._h, n, ptr, int(flags), C.byref(nprom), C.byref(ne)))
        return int(nprom.value), int(ne.value)

    def points(self):
        out = np.empty((self.n, self.d), np.float64)
        _check(pirrt_get_points(self._h, out.ctypes.data, out.size))
        return out

    def exploit_async(self) -> None:
        """pirrt_exploit_async: start the exploit and return at once."""
        _check(pirrt_exploit_async(self._h))

    def exploit_wait(self) -> ExploitStats:
        """pirrt_exploit_wait: complete the started exploit."""
        st = pirrt_exploit_stats()
        _check(pirrt_exploit_wait(self._h, C.byref(st)))
        return ExploitStats(*(getattr(st, f[0]) for f in pirrt_exploit_stats._fields_))

    def step_async(self, h_new, src, dst, cost, flags=0) -> None:
        """pirrt_step_async: enqueue append + guarded exploit + best path of one
        BE-RRT# step and return at once.  numpy arrays (best: pinned, e.g.
        torch.pin_memory().numpy()) are referenced until the step's
        step_wait; torch CUDA tensors -> PIRRT_F_DEVICE_PTRS."""
        if any(_is_torch_cuda(x) for x in (h_new, src, dst, cost)):
            flags |= PIRRT_F_DEVICE_PTRS
            m = int(src.numel())
            _check_device_tensors(int(self.cfg.device), {"dst": m, "cost": m},
                                  h_new=h_new, src=src, dst=dst, cost=cost)
            keep = (h_new, src, dst, cost)
            ptrs = [t.data_ptr() for t in keep]
            nn = int(h_new.numel())
        else:
            keep = (np.ascontiguousarray(h_new, np.float64), np.ascontiguousarray(src, np.int32),
                    np.ascontiguousarray(dst, np.int32), np.ascontiguousarray(cost, np.float64))
            ptrs = [a.ctypes.data if a.size else None for a in keep]
            nn, m = int(keep[0].size), int(keep[1].size)
        _check(pirrt_step_async(self._h, nn, ptrs[0], m, ptrs[1], ptrs[2], ptrs[3], int(flags)))
        if not hasattr(self, "_step_keep"):
            self._step_keep = []
        self._step_keep.append(keep)        # the library reads them until the step completes

    def step_wait(self) -> StepResult:
        """pirrt_step_wait: complete the oldest outstanding step."""
        r = pirrt_step_result()
        cap = max(self.n, 1)
        path = np.empty(cap, np.int32)
        try:
            _check(pirrt_step_wait(self._h, C.byref(r), path.ctypes.data, cap))
        finally:
            if getattr(self, "_step_keep", None):
                self._step_keep.pop(0)
        st = ExploitStats(*(getattr(r.stats, f[0]) for f in pirrt_exploit_stats._fields_)) \
            if r.replanned else None
        return StepResult(int(r.n_new_promising), bool(r.replanned), st,
                          path[: r.path_len].copy(), float(r.path_cost), int(r.goal))

    @property
    def steps_outstanding(self) -> int:
        return int(pirrt_steps_outstanding(self._h))

    def _get(self, fn, dtype):
        n = self.n
        out = np.empty(n, dtype)
        _check(fn(self._h, out.ctypes.data, n))
        return out

    def policy(self):
        return self._get(pirrt_get_policy, np.int32)

    def costs(self):
        return self._get(pirrt_get_costs, np.float64)

    def promising(self):
        return self._get(pirrt_get_promising, np.uint8)

    def parent_costs(self):
        return self._get(pirrt_get_parent_costs, np.float64)

    def in_edges(self):
        """The stored graph as in-edge CSR (off[n + 1], src[E], cost[E]); row
        order as stored (pirrt_get_in_edges)."""
        n, E = self.n, self.n_edges
        off = np.empty(n + 1, np.int64)
        src = np.empty(max(E, 1), np.int32)
        cost = np.empty(max(E, 1), np.float64)
        _check(pirrt_get_in_edges(self._h, off.ctypes.data, n + 1, src.ctypes.data,
                                  cost.ctypes.data, E))
        k = int(off[-1])                # this rank's share on a partitioned sharded store
        return off, src[:k], cost[:k]

    def state(self):
        """(parent, g, pc, b) -- same order as the oracle's state()."""
        return self.policy(), self.costs(), self.parent_costs(), self.promising()

    def best_path_goal(self):
        """(path root..goal, cost, best goal id or -1)."""
        cap = max(self.n, 1)
        path = np.empty(cap, np.int32)
        ln = C.c_int64(0)
        cost = C.c_double(0)
        goal = C.c_int32(0)
        _check(pirrt_best_path(self._h, path.ctypes.data, cap, C.byref(ln), C.byref(cost),
                               C.byref(goal)))
        return path[: ln.value].copy(), float(cost.value), int(goal.value)

    def best_path(self):
        path, cost, _ = self.best_path_goal()
        return path, cost

    def set_policy(self, parent, g, b=None):
        parent = np.ascontiguousarray(parent, np.int32)
        g = np.ascontiguousarray(g, np.float64)
        bp = None
        if b is not None:
            b = np.ascontiguousarray(b, np.uint8)
            bp = b.ctypes.data
        _check(pirrt_set_policy(self._h, parent.ctypes.data, g.ctypes.data, bp))
