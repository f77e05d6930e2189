"""One cold solve (S = N) of the 1M 6-D gamma_k graph (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gen, suite
g, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "x", "/tmp/g1m.npz")
ctx, rows = suite.gpu_replay(g, 1_000_000, 1_000_000)
st = rows[0][2]
print(st)
