"""Per-batch Extend/Replan trace of the gamma* 7-D 200k workload (configs[3]
sizes, tests/test_parity_fullsize_gpu.py seed): (batch, promising, PI
iterations, Evaluates, best-path cost) for every batch that Replans.
    python tools/gstar7_probe.py"""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, gen
from paper_2003_04920_b200 import pirrt
from paper_2003_04920_b200.berrt import batches
d, n, S = 7, 200_000, 1000
pts, bx = gen.points(d, n, 30, seed=gen.seed_of("fullsize-gstar", d, n))
h_root = float(np.sqrt(((pts[0] - pts[1]) ** 2).sum()))
gpu = pirrt.Context(h_root=h_root, vertex_capacity=n + 1024, edge_capacity=int(2.2 * 700 * n))
gpu.set_world(d, bx, pts[0], pts[1], gm := gen.gamma_star(d))
row = []
for k, (lo, hi) in enumerate(batches(n, S)):
    p = gpu.extend(pts[lo:hi])[0]
    if p > 0:
        st = gpu.exploit()
        row.append((k, p, st.iterations, st.evaluations, round(gpu.best_path_goal()[1], 5)))
print(row)
