"""Debug: the goal-set S = 1 replay of tests/test_parity_goals_variants_gpu.py
(test_goal_region_replay_2d[False-1]); at the first exploit whose stats
differ, print the vertices whose state differs and their history.
    python tools/debug_goalset.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import gen  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402
from paper_2003_04920_b200.berrt import batches  # noqa: E402
from parity import STAT_KEYS  # noqa: E402
from test_oracle_goals_variants import goal_region, with_h  # noqa: E402

S = int(os.environ.get("DBG_S", "1"))
r = gen.rrg(2, 3000, gen.gamma_star(2), n_boxes=20, seed=gen.seed_of("gpu-goalset", S))
ids, h = goal_region(r, 0.08)
r = with_h(r, h)
gpu = pirrt.Context(h_root=h[0], goals=ids)
orc = Oracle(h_root=h[0])
orc.set_goals(ids)
goalset = set(int(x) for x in ids) | {1}
hist = []
import ctypes as C  # noqa: E402
lib = pirrt._lib
lib.pirrt_debug_inc.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]


def inc_state():
    out = (C.c_longlong * 12)()
    lst = np.zeros(4096, np.int32)
    lib.pirrt_debug_inc(gpu._h, out, lst.ctypes.data, 4096)
    o = list(out)
    names = ["imp_count", "app_pre_k", "pre0", "pre1", "c_buf", "c_n", "L_imp", "n_imp", "gc0", "gc1",
             "imp_full", "dirty_n"]
    d = dict(zip(names, o))
    d["list"] = sorted(lst[: o[2 + ((o[0] + 1) & 1)]].tolist())
    return d


for k, (a, b) in enumerate(batches(r.n, S)):
    s, t, c = r.batch(a, b, directed=False)
    pg = gpu.append(r.h[a:b], s, t, c, flags=4)
    po = orc.append(r.h[a:b], s, t, c, flags=4)
    assert pg == po
    if k >= 1014:
        print(k, "after append:", inc_state())
    if po == 0:
        hist.append((k, "no exploit"))
        continue
    g_before = gpu.costs()
    gs, os_ = gpu.exploit(), orc.exploit()
    bad = [x for x in STAT_KEYS if getattr(gs, x) != getattr(os_, x)]
    if k >= 1014:
        print(k, "after exploit:", inc_state(), "goal g:", {v: round(float(x), 6) for v, x in enumerate(gpu.costs()) if v in goalset and x < 1e9 and v < 40})
    hist.append((k, f"it={os_.iterations} ev={os_.evaluations} st={os_.stalled} dg={os_.last_delta_g:.3g}"))
    if bad:
        print("batch", k, "differs in", bad)
        print(" gpu", gs)
        print(" orc", os_)
        gp, gg, gpc, gb = gpu.state()
        op, og, opc, ob = orc.state()
        diff = np.nonzero((gp != op) | (gg.view(np.uint64) != og.view(np.uint64)))[0]
        for v in diff[:10]:
            print(f"  v={v} goal={v in goalset} gpu(p={gp[v]},g={gg[v]:.6f},b={gb[v]}) "
                  f"orc(p={op[v]},g={og[v]:.6f},b={ob[v]}) g_before={g_before[v]:.6f} "
                  f"g(parent)+pc={og[op[v]] + opc[v] if op[v] >= 0 else -1:.6f}")
        print(" history:", hist[-8:])
        break
else:
    print("no divergence")
