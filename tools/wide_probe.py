"""Cold solve (S = N) of the 1M 6-D gamma_k graph: exploit time and its
Improve / Evaluate split, for the library named by PIRRT_LIB (variants of the
wide Improve) and PIRRT_WIDE_TASKS."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gen  # noqa: E402
import suite  # noqa: E402

g, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "x", os.environ.get("GRAPH_CACHE", "/tmp/g1m.npz"))
res = []
for rep in range(3):
    ctx, rows = suite.gpu_replay(g, 1_000_000, 1_000_000)
    st = rows[0][2]
    res.append((st.device_ms, st.improve_ms, st.evaluate_ms))
    del ctx
lib = os.path.basename(os.environ.get("PIRRT_LIB", "libpirrt.so"))
best = min(res)
print(f"{lib} wide={os.environ.get('PIRRT_WIDE_TASKS', 'default')} it={st.iterations} "
      f"relax={st.relaxations} device_ms={best[0]:.3f} improve_ms={best[1]:.3f} "
      f"evaluate_ms={best[2]:.3f} all={[round(x[0], 3) for x in res]}", flush=True)
