"""Per-level trace of one exploit at the bench workload (PIRRT_DEBUG=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2003_04920_b200 import pirrt
from paper_2003_04920_b200.berrt import replay
S = 4096
z = np.load("/tmp/g1m.npz")
gm = gen.gamma_k(6)
g = gen.RRG(6, int(z["h"].size), gm, z["points"], z["boxes"], z["h"], z["off"], z["nbr"], z["cost"], 0, 0)
ctx = pirrt.Context(h_root=g.h_root(), vertex_capacity=g.n + 1024, edge_capacity=int(2.4 * g.off[-1]))
os.environ.pop("PIRRT_DEBUG", None)
replay(ctx, g, S, n_stop=1_000_000 - S, final=False)
a, b = 1_000_000 - S, 1_000_000
s, d, c = g.batch(a, b, directed=False)
ctx.append(g.h[a:b], s, d, c, flags=4)
os.environ["PIRRT_DEBUG"] = "1"
print("exploit...", flush=True)
st = ctx.exploit()
print(st, flush=True)
