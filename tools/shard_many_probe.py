import json, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import gen, suite
g6, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "cfg3_6d_1000k_berrt_S4096_gammak_20boxes|0", "/tmp/g1m.npz")
ctx, rows = suite.gpu_replay(g6, 4096, g6.n, time_from=g6.n - 60 * 4096, sharded=True)
out = [(round(app, 2), round(st.device_ms, 2)) for app, ex, st in rows if st is not None]
print(json.dumps(out))
