"""Per-call host timing of append/exploit/best_path with device vs pinned-host inputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2003_04920_b200 import pirrt
from paper_2003_04920_b200.berrt import replay
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
S = 4096
r = gen.rrg(6, n + 20 * S, gen.gamma_k(6), n_boxes=20, seed=7)
stream = torch.cuda.current_stream()
ctx = pirrt.Context(h_root=r.h_root(), stream=stream, vertex_capacity=r.n + 1024,
                    edge_capacity=int(2.4 * r.off[-1]) + 4096)
replay(ctx, r, S, n_stop=n, final=False)
torch.cuda.synchronize()
def pin(x): return torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
def dev(x): return torch.from_numpy(np.ascontiguousarray(x)).cuda()
for mode in ("dev", "pin", "pageable"):
    for k in range(5):
        base = n + (["dev", "pin", "pageable"].index(mode) * 5 + k) * S
        s, d, c = r.batch(base, base + S, directed=False)
        args = [r.h[base:base + S], s, d, c]
        if mode == "dev": args = [dev(x) for x in args]
        elif mode == "pin": args = [pin(x) for x in args]
        torch.cuda.synchronize()
        t0 = time.perf_counter(); np_ = ctx.append(*args, flags=4); t1 = time.perf_counter()
        st = ctx.exploit(); t2 = time.perf_counter()
        ctx.best_path(); t3 = time.perf_counter()
        print(f"{mode:8s} append {1e3*(t1-t0):7.3f} ms  exploit {1e3*(t2-t1):7.3f} ms (dev {st.device_ms:.3f})  best_path {1e3*(t3-t2):6.3f} ms  edges {ctx.n_edges}", flush=True)
