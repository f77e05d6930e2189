"""Cold solve through the device-side Extend (bench.py's gamma* cold record)
at a configurable size -- a small reproducer for memcheck runs:
    compute-sanitizer --tool memcheck python tools/repro_cold.py --n 100000"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--d", type=int, default=6)
ap.add_argument("--chunk", type=int, default=131072)
ap.add_argument("--gamma", default="star")
a = ap.parse_args()
gm = gen.gamma_star(a.d) if a.gamma == "star" else gen.gamma_k(a.d)
pts, bx = gen.points(a.d, a.n, 20, seed=gen.seed_of("repro_cold", a.n))
h_root = float(np.sqrt(((pts[0] - pts[1]) ** 2).sum()))
ctx = pirrt.Context(h_root=h_root, vertex_capacity=a.n + 1024)
ctx.set_world(a.d, bx, pts[0], pts[1], gm)
for lo in range(2, a.n, a.chunk):
    ctx.extend(pts[lo:min(a.n, lo + a.chunk)])
st = ctx.exploit()
print("cold", st)
for lo in range(a.n, a.n, 1):
    pass
print("ok")
