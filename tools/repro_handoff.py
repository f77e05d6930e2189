"""Small reproducer of tests/test_parity_gpu.py::test_wide_improve_handoff_parity
for compute-sanitizer runs:
    PIRRT_WIDE_TASKS=1 compute-sanitizer --tool memcheck python tools/repro_handoff.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity import dual_replay  # noqa: E402

n = int(os.environ.get("N", "12000"))
S = int(os.environ.get("S", "1500"))
flags = int(os.environ.get("FLAGS", "0"))
wide = os.environ.get("PIRRT_WIDE_TASKS", "1")
r = gen.rrg(6, n, gen.gamma_k(6), n_boxes=10, seed=gen.seed_of("wide", wide, flags))
gpu = pirrt.Context(h_root=r.h_root(), flags=flags)
orc = Oracle(h_root=r.h_root(), flags=flags)
print("exploits", dual_replay(gpu, orc, r, S), flush=True)
print("ok")
