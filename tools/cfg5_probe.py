"""configs[4] single-GPU point: 6-D 10M gamma_k graph -- cold solve (S=N) and
per-batch S=65536 exploits near n, on one B200 (the P=1 point of the scaling
study; the sharded loop runs the same graph over P ranks).

    python tools/cfg5_probe.py [N] [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import gen  # noqa: E402
import suite  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
t0 = time.perf_counter()
g = gen.rrg(6, N, gen.gamma_k(6), n_boxes=20, seed=gen.seed_of("cfg5", N))
tg = time.perf_counter() - t0
print("generated", N, "pairs", g.n_pairs, "mean degree", g.mean_degree, "in", tg, "s", flush=True)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import bench  # noqa: E402
peaks = {"hbm_gbs": bench.peaks()[0]}
rep = {"n": N, "gamma": gen.gamma_k(6), "mean_degree": g.mean_degree,
       "directed_edges": 2 * g.n_pairs, "generate_s": tg}
# cold solve
ctx, rows = suite.gpu_replay(g, N, N)
st = rows[0][2]
bytes_ = st.relaxations * 20 + st.improve_set * 40 + st.eval_scanned * 8 + st.eval_visits * 38
rep["cold"] = {"append_ms": rows[0][0], "exploit_ms": rows[0][1], "device_ms": st.device_ms,
               "iterations": st.iterations, "relaxations": st.relaxations,
               "improve_ms": st.improve_ms, "evaluate_ms": st.evaluate_ms,
               "improve_GBps": st.relaxations * 20 / (st.improve_ms * 1e-3) / 1e9,
               "exploit_GBps": bytes_ / (st.device_ms * 1e-3) / 1e9,
               "exploit_frac_hbm": bytes_ / (st.device_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
               "gteps": st.relaxations / (st.device_ms * 1e-3) / 1e9}
print(json.dumps(rep["cold"]), flush=True)
del ctx
# per-batch near n
S = 65536
_, rows = suite.gpu_replay(g, S, N, time_from=N - 8 * S)
rep["per_batch_S65536"] = suite.exploit_summary(rows)
print(json.dumps(rep["per_batch_S65536"]), flush=True)
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/cfg5_1gpu.json"
json.dump(rep, open(out, "w"), indent=1, default=float)
