"""Cold solve (S = N) of the 1M 6-D gamma_k graph with the per-iteration
Improve timeline (library built with -DPIRRT_LEVEL_TRACE=1, PIRRT_DEBUG=1):
    PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/cold_trace.py
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gen  # noqa: E402
import suite  # noqa: E402

g, _ = suite.graph(6, 1_000_000, gen.gamma_k(6), 20, "x", os.environ.get("GRAPH_CACHE", "/tmp/g1m.npz"))
for rep in range(2):
    if rep == 1:
        os.environ["PIRRT_DEBUG"] = "1"
    ctx, rows = suite.gpu_replay(g, 1_000_000, 1_000_000)
    st = rows[0][2]
    print(f"== rep {rep} it={st.iterations} relax={st.relaxations} improve_set={st.improve_set} "
          f"device_ms={st.device_ms:.3f} improve_ms={st.improve_ms:.3f} evaluate_ms={st.evaluate_ms:.3f}",
          flush=True)
    del ctx
