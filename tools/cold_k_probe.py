import json, os, sys, types
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tools'))
import suite, gen
g6, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "cfg3_6d_1000k_berrt_S4096_gammak_20boxes|0", "/tmp/g1m.npz")
for rep in range(2):
    ctx, rows = suite.gpu_replay(g6, g6.n, g6.n)
    st = rows[0][2]
    print(json.dumps({"device_ms": st.device_ms, "improve_ms": st.improve_ms, "evaluate_ms": st.evaluate_ms}))
    del ctx
_, rows = suite.gpu_replay(g6, 4096, g6.n, time_from=g6.n - 10 * 4096, sharded=True)
print(json.dumps(suite.exploit_summary(rows)))
print([round(r[2].device_ms, 3) for r in rows if r[2] is not None])
