"""Sharded loop (NCCL, one rank) on the bench workload's last batches: per
exploit the device time, the time inside Improve / Evaluate phases, and the
iteration and launch counts (host stall vs device work).
    python tools/shard_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import gen  # noqa: E402
import suite  # noqa: E402

g6, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "cfg3_6d_1000k_berrt_S4096_gammak_20boxes|0", "/tmp/g1m.npz")
ctx, rows = suite.gpu_replay(g6, 4096, g6.n, time_from=g6.n - 12 * 4096, sharded=True)
for app, ex, st in rows:
    if st is None:
        continue
    print(json.dumps({"append_ms": round(app, 3), "exploit_host_ms": round(ex, 3), "device_ms": round(st.device_ms, 3),
                      "improve_ms": round(st.improve_ms, 3), "evaluate_ms": round(st.evaluate_ms, 3),
                      "iterations": st.iterations, "barriers": st.barriers}))
