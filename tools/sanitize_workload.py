"""Small workloads for compute-sanitizer runs (memcheck / racecheck /
synccheck), each checked against the oracle:
  configs[0] 2-D 1k gamma* (S = 1 and S = N), configs[1] shape at 6k (2-D
  clutter, S = 1), a 6-D 12k replay with wide-Improve hand-offs, a 2-rank
  in-process group, the NEIGHBOURS variant, deferred steps two deep.
    compute-sanitizer --tool memcheck python tools/sanitize_workload.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import gen  # noqa: E402
import oracle  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402
from parity import RankGroup, dual_replay  # noqa: E402

os.environ.setdefault("PIRRT_WQ_KEEP", "3")          # exercise the global work queue
cases = []
r1 = gen.rrg(2, 1000, gen.gamma_star(2), n_boxes=0, seed=gen.seed_of("san1"))
cases.append(("cfg1 S=1", lambda: (pirrt.Context(h_root=r1.h_root()), Oracle(h_root=r1.h_root()), r1, 1)))
cases.append(("cfg1 S=N", lambda: (pirrt.Context(h_root=r1.h_root()), Oracle(h_root=r1.h_root()), r1, r1.n)))
r2 = gen.rrg(2, 6000, gen.gamma_star(2), n_boxes=30, seed=gen.seed_of("san2"))
cases.append(("cfg2 shape S=1", lambda: (pirrt.Context(h_root=r2.h_root()), Oracle(h_root=r2.h_root()), r2, 1)))
r3 = gen.rrg(6, 12000, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("san3"))


def wide():
    os.environ["PIRRT_WIDE_TASKS"] = "300"
    c = pirrt.Context(h_root=r3.h_root())
    os.environ.pop("PIRRT_WIDE_TASKS")
    return c, Oracle(h_root=r3.h_root()), r3, 1500


cases.append(("6-D hand-offs", wide))
cases.append(("group P=2", lambda: (RankGroup(pirrt, 2, h_root=r3.h_root()), Oracle(h_root=r3.h_root()), r3, 1000)))
cases.append(("neighbours", lambda: (pirrt.Context(h_root=r2.h_root(), flags=pirrt.PIRRT_F_NEIGHBOURS),
                                     Oracle(h_root=r2.h_root(), flags=oracle.NEIGHBOURS), r2, 40)))


def step_pipeline(gpu, orc, r, S, n_stop):
    """Deferred steps (pirrt_step_async / pirrt_step_wait) two deep, each
    result against the oracle's synchronous Alg. 3 step."""
    import numpy as np
    from paper_2003_04920_b200.berrt import batches
    pend, k = [], 0
    for a, b in batches(n_stop, S):
        s, t, c = r.batch(a, b, directed=False)
        gpu.step_async(r.h[a:b], s, t, c, flags=oracle.EDGES_UNDIRECTED)
        nprom = orc.append(r.h[a:b], s, t, c, flags=oracle.EDGES_UNDIRECTED)
        if nprom > 0:
            orc.exploit()
        pend.append((nprom, orc.best_path()))
        while len(pend) >= 2 or (pend and b == n_stop):
            res = gpu.step_wait()
            nprom, (path, cost) = pend.pop(0)
            assert res.n_new_promising == nprom and np.array_equal(res.path, path) and res.cost == cost
            k += 1
    return k


cases.append(("steps 6-D", lambda: (pirrt.Context(h_root=r3.h_root()), Oracle(h_root=r3.h_root()), r3, 700)))
only = sys.argv[1:]
for name, make in cases:
    if only and not any(o in name for o in only):
        continue
    gpu, orc, r, S = make()
    n_stop = min(r.n, 2 + 60 * S) if S > 1 else min(r.n, 1500)
    if name.startswith("steps"):
        k = step_pipeline(gpu, orc, r, S, n_stop)
    else:
        k = dual_replay(gpu, orc, r, S, n_stop=n_stop)
    print(f"{name}: {k} exploits bit-exact", flush=True)
print("ok")
