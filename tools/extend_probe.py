"""Device-side Extend (pirrt_extend_batch) end to end.

config 4 (7-D 200k gamma_k, 30 boxes, S = 1000): plan time with the CPU
generator building the edges (exploration on the host) vs sampling on the host
(gen.points) + edges built on the device, each followed by the same exploits.
config 3 (6-D, S = 4096) per-batch: extend (points over PCIe) vs append
(edge triples over PCIe) near n = 1M is in --n3 (default 0 = skip)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2003_04920_b200 import pirrt  # noqa: E402
from paper_2003_04920_b200.berrt import EDGES_UNDIRECTED, batches  # noqa: E402


def plan(d, n, gk, boxes, S, tag):
    gamma = gen.gamma_k(d) if gk == "k" else gen.gamma_star(d)
    seed = gen.seed_of(tag)
    # warm-up context (first-call costs)
    w = pirrt.Context(h_root=1.0)
    wp, wb = gen.points(d, 2000, 2, seed=3)
    w.set_world(d, wb, wp[0], wp[1], gamma)
    for a, b in batches(2000, 500):
        if w.extend(wp[a:b])[0] > 0:
            w.exploit()
    del w
    out = {"d": d, "n": n, "gamma": gk, "boxes": boxes, "S": S}
    # (a) host exploration: the CPU generator builds every edge, then append + exploit
    t0 = time.perf_counter()
    r = gen.rrg(d, n, gamma, n_boxes=boxes, seed=seed)
    t_gen = time.perf_counter() - t0
    ctx = pirrt.Context(h_root=r.h_root(), vertex_capacity=n + 16,
                        edge_capacity=int(2.4 * r.n_pairs) + 4096)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for a, b in batches(n, S):
        s_, d_, c_ = r.batch(a, b, directed=False)
        if ctx.append(r.h[a:b], s_, d_, c_, flags=EDGES_UNDIRECTED) > 0:
            ctx.exploit()
    ctx.exploit()
    t_a = time.perf_counter() - t0
    path_a, cost_a = ctx.best_path()
    del ctx
    # (b) host sampling only + device-side Extend
    t0 = time.perf_counter()
    pts, bx = gen.points(d, n, boxes, seed=seed)
    t_pts = time.perf_counter() - t0
    ctx = pirrt.Context(h_root=float(np.sqrt(((pts[0] - pts[1]) ** 2).sum())), vertex_capacity=n + 16,
                        edge_capacity=int(2.4 * r.n_pairs) + 4096)
    ctx.set_world(d, bx, pts[0], pts[1], gamma)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pairs = 0
    for a, b in batches(n, S):
        nprom, ne = ctx.extend(pts[a:b])
        pairs += ne
        if nprom > 0:
            ctx.exploit()
    ctx.exploit()
    t_b = time.perf_counter() - t0
    path_b, cost_b = ctx.best_path()
    assert pairs == r.n_pairs and cost_a == cost_b and np.array_equal(path_a, path_b)
    out.update({"pairs": int(pairs), "mean_degree": r.mean_degree,
                "host_exploration": {"generator_s": t_gen, "append_exploit_s": t_a, "plan_s": t_gen + t_a},
                "device_extend": {"sampling_s": t_pts, "extend_exploit_s": t_b, "plan_s": t_pts + t_b},
                "same_best_path": True, "best_cost": cost_b,
                "pcie_bytes_per_batch": {"points": S * d * 8, "edges": int(16 * r.n_pairs / max(1, n // S))}})
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/extend.json")
    a = ap.parse_args()
    rep = {"cfg4_7d_200k_gammak": plan(7, 200_000, "k", 30, 1000, "extend_cfg4"),
           "cfg3_6d_200k_gammak_S4096": plan(6, 200_000, "k", 20, 4096, "extend_cfg3")}
    json.dump(rep, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
