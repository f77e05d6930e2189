"""configs[4] single-GPU point (10M-vertex 6-D gamma_k RRG, 20 boxes) built
with the device-side Extend instead of the CPU generator (which takes ~7 min
here).  Cold solve = extend every batch with no exploit in between, then one
exploit: bit-identical to append(S = N) + exploit (R14 is sequential in id
order either way, and thr = +inf until the first exploit).  Then 10 per-batch
exploits at S = 65536 beyond N.

    python tools/cfg5_extend_probe.py --n 10000000 --out gpurun_out/cfg5.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--S", type=int, default=65536)
    ap.add_argument("--batches", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/cfg5.json")
    ap.add_argument("--d", type=int, default=6)
    ap.add_argument("--gamma", default="k")
    ap.add_argument("--boxes", type=int, default=20)
    ap.add_argument("--seed-tag", default="", help="gen.seed_of tag (default: cfg5_extend)")
    a = ap.parse_args()
    d, boxes = a.d, a.boxes
    gamma = gen.gamma_k(d) if a.gamma == "k" else gen.gamma_star(d)
    n_all = a.n + a.batches * a.S
    t0 = time.perf_counter()
    seed = gen.seed_of(a.seed_tag) if a.seed_tag else gen.seed_of("cfg5_extend", a.n)
    pts, bx = gen.points(d, n_all, boxes, seed=seed)
    t_pts = time.perf_counter() - t0
    h_root = float(np.sqrt(((pts[0] - pts[1]) ** 2).sum()))
    # warm-up (first-call costs)
    w = pirrt.Context(h_root=h_root)
    w.set_world(d, bx, pts[0], pts[1], gamma)
    for lo in range(2, 20002, 5000):
        if w.extend(pts[lo:lo + 5000])[0] > 0:
            w.exploit()
    del w
    ctx = pirrt.Context(h_root=h_root, stream=torch.cuda.current_stream(),
                        vertex_capacity=n_all + 1024,
                        edge_capacity=int(2.2 * (40 if a.gamma == "k" else 600) * n_all))
    ctx.set_world(d, bx, pts[0], pts[1], gamma)
    dpts = torch.from_numpy(pts).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pairs = 0
    for lo in range(2, a.n, a.S):
        hi = min(a.n, lo + a.S)
        pairs += ctx.extend(dpts[lo:hi])[1]
    torch.cuda.synchronize()
    t_ext = time.perf_counter() - t0
    st = ctx.exploit()
    hbm = bench.peaks()[0]
    bytes_ = st.relaxations * 20 + st.improve_set * 40 + st.eval_scanned * 8 + st.eval_visits * 38
    rep = {"n": a.n, "d": d, "gamma": gamma, "boxes": boxes, "sampling_s": t_pts,
           "extend_s_total": t_ext, "extend_ms_per_batch": 1e3 * t_ext / ((a.n - 2 + a.S - 1) // a.S),
           "directed_edges": 2 * pairs, "mean_degree": 2 * pairs / a.n,
           "cold": {"device_ms": st.device_ms, "iterations": st.iterations, "relaxations": st.relaxations,
                    "improve_ms": st.improve_ms, "evaluate_ms": st.evaluate_ms,
                    "gteps": st.relaxations / (st.device_ms * 1e-3) / 1e9,
                    "exploit_GBps_algorithmic": bytes_ / (st.device_ms * 1e-3) / 1e9,
                    "exploit_frac_hbm": bytes_ / (st.device_ms * 1e-3) / 1e9 / hbm}}
    print(json.dumps(rep), flush=True)
    rows = []
    for k in range(a.batches):
        lo, hi = a.n + k * a.S, a.n + (k + 1) * a.S
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nprom, ne = ctx.extend(dpts[lo:hi])
        t1 = time.perf_counter()
        st = ctx.exploit() if nprom > 0 else None
        rows.append({"extend_ms": 1e3 * (t1 - t0), "exploit_device_ms": st.device_ms if st else 0.0,
                     "iterations": st.iterations if st else 0,
                     "relaxations": st.relaxations if st else 0})
    ex = [r for r in rows if r["iterations"]]
    ems = sorted(r["exploit_device_ms"] for r in ex)
    rep["per_batch"] = {"S": a.S, "rows": rows,
                        "exploit_ms_mean": float(np.mean(ems)) if ems else None,
                        "exploit_ms_median": ems[len(ems) // 2] if ems else None,
                        "extend_ms_mean": float(np.mean([r["extend_ms"] for r in rows]))}
    print(json.dumps(rep["per_batch"]), flush=True)
    json.dump(rep, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
