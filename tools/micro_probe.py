import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gen, suite
g, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "x", "/tmp/g1m.npz")
print(json.dumps(suite.microbench(g), indent=1))
