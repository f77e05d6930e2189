"""Compare build variants (PIRRT_LIB) on the per-batch and cold-solve workloads."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import gen
import suite
g, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "x", "/tmp/g1m.npz")
n6 = 1_000_000
_, rows = suite.gpu_replay(g, 4096, n6, time_from=n6 - 20 * 4096)
pb = suite.exploit_summary(rows)
ctx, rows = suite.gpu_replay(g, n6, n6)
st = rows[0][2]
print(json.dumps({"lib": os.environ.get("PIRRT_LIB", "default"),
                  "per_batch_exploit_ms_mean": pb["exploit_ms_mean"], "per_batch_append_ms": pb["append_ms_mean"],
                  "cold_exploit_ms": st.device_ms, "cold_improve_ms": st.improve_ms,
                  "cold_improve_GBps": st.relaxations * 20 / (st.improve_ms * 1e-3) / 1e9,
                  "cold_evaluate_ms": st.evaluate_ms}), flush=True)
