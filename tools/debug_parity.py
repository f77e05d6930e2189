"""Replay a BE-RRT# case on GPU and oracle, comparing after EVERY exploit;
print details at the first divergence (debug tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
from oracle import Oracle
from paper_2003_04920_b200 import pirrt
from paper_2003_04920_b200.berrt import batches
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity import STAT_KEYS

d, n, boxes, S, tag = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
gm = gen.gamma_star(d)
r = gen.rrg(d, n, gm, n_boxes=boxes, seed=gen.seed_of(tag, S))
gpu = pirrt.Context(h_root=r.h_root(), grid_blocks=int(os.environ.get("DBG_GRID", "0"))); orc = Oracle(h_root=r.h_root())
prev = None
for k, (a, b) in enumerate(batches(r.n, S)):
    src, dst, cost = r.batch(a, b, directed=False)
    pg = gpu.append(r.h[a:b], src, dst, cost, flags=4)
    po = orc.append(r.h[a:b], src, dst, cost, flags=4)
    if pg != po:
        print("nprom differs", k, pg, po); break
    if k % 250 == 0 or (os.environ.get("DBG_FROM") and k >= int(os.environ["DBG_FROM"])):
        print("batch", k, "edges", gpu.n_edges, flush=True)
    if po == 0:
        continue
    try:
        gs = gpu.exploit()
    except Exception as e:
        print("GPU exploit failed at batch", k, "verts", a, b, ":", e, flush=True)
        raise SystemExit(1)
    os_ = orc.exploit()
    gst, ost = gpu.state(), orc.state()
    import ctypes as C
    cap = gpu.n + 2
    lst = np.zeros(cap, np.int32); cnt = C.c_int32(0)
    pirrt._lib.pirrt_debug_blist.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    rc = pirrt._lib.pirrt_debug_blist(gpu._h, lst.ctypes.data, cap, C.byref(cnt))
    L = lst[1:1 + cnt.value]
    bset = set(np.nonzero(gst[3])[0].tolist())
    if rc != 0 or lst[0] != 0 or len(set(L.tolist())) != L.size or set(L.tolist()) != bset:
        print("BLIST INCONSISTENT at batch", k, "rc", rc, "root", lst[0], "count", cnt.value,
              "unique", len(set(L.tolist())), "|b|", len(bset),
              "missing", sorted(bset - set(L.tolist()))[:10], "extra", sorted(set(L.tolist()) - bset)[:10], flush=True)
        break
    bad = [kk for kk in STAT_KEYS if getattr(gs, kk) != getattr(os_, kk)]
    sdiff = [nm for nm, x, y in zip(("parent", "g", "pc", "b"), gst, ost) if not np.array_equal(x, y)]
    if bad or sdiff:
        print("DIVERGE at batch", k, "verts", a, b, "stats", bad, "state", sdiff)
        print(" gpu", gs); print(" orc", os_); print(" prev", prev)
        for nm, x, y in zip(("parent", "g", "pc", "b"), gst, ost):
            idx = np.nonzero(x != y)[0][:8]
            for i in idx:
                print(f"  {nm}[{i}] gpu={x[i]} orc={y[i]} | gpu p={gst[0][i]} g={gst[1][i]} b={gst[3][i]} ; orc p={ost[0][i]} g={ost[1][i]} b={ost[3][i]}")
        break
    prev = (gs, os_)
else:
    print("no divergence over", k + 1, "batches")
