#!/usr/bin/env python
"""Measurement suite over SURVEY.md section 8(d)'s configurations (one B200).

Writes a JSON report (default profiles/suite.json) with, per configuration,
the GPU exploit times, the serial oracle on the same host (1 core), and the
"achievable gather bandwidth" microbenchmarks that serve as roofline
denominators next to MEASURED_PEAKS.json.  bench.py is the contract line;
this script fills the section 8(d) table.

    python tools/suite.py [--out profiles/suite.json] [--quick]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402


def pct(xs, q):
    return float(np.percentile(np.asarray(xs), q)) if xs else None


def graph(d, n, gamma, boxes, tag, cache=None):
    t = time.perf_counter()
    if cache and os.path.exists(cache):
        z = np.load(cache)
        g = gen.RRG(d, int(z["h"].size), gamma, z["points"], z["boxes"], z["h"], z["off"], z["nbr"],
                    z["cost"], 0, 0)
        if g.n >= n:
            return g, 0.0
    g = gen.rrg(d, n, gamma, n_boxes=boxes, seed=gen.seed_of(tag))
    return g, time.perf_counter() - t


def gpu_replay(g, S, n_stop, flags=0, time_from=None, sharded=False):
    """BE-RRT# replay on the GPU; returns per-batch (append_ms, exploit_ms, stats)."""
    import torch
    from paper_2003_04920_b200 import pirrt
    stream = torch.cuda.current_stream()
    kw = dict(flags=flags | (pirrt.PIRRT_F_SHARDED if sharded else 0))
    ctx = pirrt.Context(h_root=g.h_root(), stream=stream, vertex_capacity=g.n + 1024,
                        edge_capacity=int(2.4 * g.off[-1]) + 4096, **kw)
    out = []
    a = 2
    while a < n_stop:
        b = min(n_stop, a + S)
        s, dd, c = g.batch(a, b, directed=False)
        timed = time_from is None or a >= time_from
        if timed:
            args = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (g.h[a:b], s, dd, c)]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nprom = ctx.append(*args, flags=pirrt.PIRRT_F_EDGES_UNDIRECTED)
            t1 = time.perf_counter()
            st = ctx.exploit() if nprom > 0 else None
            t2 = time.perf_counter()
            out.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), st))
        else:
            nprom = ctx.append(g.h[a:b], s, dd, c, flags=pirrt.PIRRT_F_EDGES_UNDIRECTED)
            if nprom > 0:
                ctx.exploit()
        a = b
    return ctx, out


def oracle_replay(g, S, n_stop, budget_s=None, flags=0):
    from oracle import EDGES_UNDIRECTED, Oracle
    o = Oracle(h_root=g.h_root(), flags=flags)
    times = []
    t_start = time.perf_counter()
    a = 2
    while a < n_stop:
        b = min(n_stop, a + S)
        s, dd, c = g.batch(a, b, directed=False)
        t0 = time.perf_counter()
        nprom = o.append(g.h[a:b], s, dd, c, flags=EDGES_UNDIRECTED)
        t1 = time.perf_counter()
        st = o.exploit() if nprom > 0 else None
        t2 = time.perf_counter()
        times.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), st))
        a = b
        if budget_s and time.perf_counter() - t_start > budget_s:
            break
    return o, times


def exploit_summary(rows):
    ex = [r for r in rows if r[2] is not None]
    ems = [r[1] for r in ex]
    return {
        "batches": len(rows), "exploits": len(ex),
        "append_ms_mean": statistics.mean([r[0] for r in rows]) if rows else None,
        "exploit_ms_total": sum(ems), "exploit_ms_median": pct(ems, 50), "exploit_ms_p95": pct(ems, 95),
        "exploit_ms_mean": statistics.mean(ems) if ems else None,
        "iterations_mean": statistics.mean([r[2].iterations for r in ex]) if ex else None,
        "relaxations_total": sum(r[2].relaxations for r in ex),
        "device_ms_median": pct([r[2].device_ms for r in ex], 50) if ex and hasattr(ex[0][2], "device_ms") else None,
        "device_ms_p95": pct([r[2].device_ms for r in ex], 95) if ex and hasattr(ex[0][2], "device_ms") else None,
    }


def microbench(g):
    import torch
    from paper_2003_04920_b200 import pirrt
    n = g.n
    # in-edge CSR of the whole graph (both directions) on the device
    src, dst, cost = g.batch(2, n, directed=True)
    order = np.argsort(dst, kind="stable")
    dsts = dst[order]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, dsts + 1, 1)
    off = np.cumsum(off)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    t_off, t_idx, t_cost = dev(off), dev(src[order]), dev(cost[order])
    rng = np.random.default_rng(0)
    rows = dev(rng.permutation(n).astype(np.int32))
    E = int(off[-1])
    ms_rows = pirrt.bench_rows(t_off, t_idx, t_cost, rows, reps=10)
    res = {"rows_stream": {"edges": E, "ms": ms_rows, "GBps": 12 * E / (ms_rows * 1e-3) / 1e9}}
    gvec = torch.rand(n, dtype=torch.float64, device="cuda")
    outv = torch.empty(n, dtype=torch.float64, device="cuda")
    ms_rel = pirrt.bench_relax(t_off, t_idx, t_cost, gvec, rows, outv, reps=10)
    res["relax_pass"] = {"edges": E, "ms": ms_rel, "GBps_algorithmic": 20 * E / (ms_rel * 1e-3) / 1e9,
                         "G_relax_per_s": E / (ms_rel * 1e-3) / 1e9}
    for name, arr_n in (("gather_L2_8MB", 1_000_000), ("gather_HBM_2GB", 256_000_000)):
        src_arr = torch.rand(arr_n, dtype=torch.float64, device="cuda")
        idx = torch.randint(0, arr_n, (64_000_000,), dtype=torch.int32, device="cuda")
        ms = pirrt.bench_gather(src_arr, idx, reps=5)
        nn = idx.numel()
        res[name] = {"gathers": nn, "ms": ms, "G_per_s": nn / (ms * 1e-3) / 1e9,
                     "algorithmic_GBps": 12 * nn / (ms * 1e-3) / 1e9,
                     "sector_GBps": (4 + 32) * nn / (ms * 1e-3) / 1e9}
        del src_arr, idx
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "suite.json"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--cache", default="/tmp/g1m.npz")
    args = ap.parse_args()
    import torch
    rep = {"host": {"cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": "),
                    "cores": os.cpu_count()},
           "gpu": torch.cuda.get_device_name(0)}
    import bench
    hbm, src = bench.peaks()
    peaks = {"hbm_gbs": hbm}
    rep["peaks"] = {"hbm_gbs": hbm, "source": src}

    # ---- configs[2]: 6-D 1M gamma_k
    g6, tgen = graph(6, 1_000_000 if not args.quick else 200_000, gen.gamma_k(6), 20,
                     "cfg3_6d_1000k_berrt_S4096_gammak_20boxes|0", args.cache)
    n6 = 1_000_000 if not args.quick else 200_000
    rep["microbench"] = microbench(g6)
    rep["microbench"]["note"] = ("rows: random row order over the full in-edge CSR (12 B/entry); "
                                 "gathers: 64M random 8-B reads of an L2-resident 8 MB array and an "
                                 "HBM-resident 2 GB array (4 B index + 8 B value algorithmic, 36 B sectors)")
    per_batch = {}
    for S in ([1024, 4096, 16384, 65536] if not args.quick else [4096]):
        _, rows = gpu_replay(g6, S, n6, time_from=n6 - 10 * S)
        per_batch[f"S{S}"] = exploit_summary(rows)
    rep["cfg3_6d_1M_gammak_per_batch"] = per_batch
    # cold solve (S = N): one append of everything, one exploit
    ctx, rows = gpu_replay(g6, n6, n6)
    st = rows[0][2]
    bytes_ = bench.algo_bytes(st)                         # SURVEY.md 8(d) units over the work done
    rep["cfg3_6d_1M_gammak_cold_solve"] = {
        "append_ms": rows[0][0], "exploit_ms": rows[0][1], "device_ms": st.device_ms,
        "iterations": st.iterations, "evaluations": st.evaluations,
        "relaxations": st.relaxations, "improve_ms": st.improve_ms, "evaluate_ms": st.evaluate_ms,
        "improve_GBps_algorithmic": st.relaxations * 20 / (st.improve_ms * 1e-3) / 1e9,
        "exploit_GBps_algorithmic": bytes_ / (st.device_ms * 1e-3) / 1e9,
        "exploit_frac_of_hbm": bytes_ / (st.device_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
        "promising": st.promising, "max_level": st.max_level,
    }
    del ctx
    # oracle on the cold solve (same graph, 1 core)
    from oracle import EDGES_UNDIRECTED, Oracle
    o = Oracle(h_root=g6.h_root())
    s, dd, c = g6.batch(2, n6, directed=False)
    t0 = time.perf_counter(); o.append(g6.h[2:n6], s, dd, c, flags=EDGES_UNDIRECTED)
    t1 = time.perf_counter(); ost = o.exploit(); t2 = time.perf_counter()
    rep["cfg3_6d_1M_gammak_cold_solve"]["oracle_append_ms"] = 1e3 * (t1 - t0)
    rep["cfg3_6d_1M_gammak_cold_solve"]["oracle_exploit_ms"] = 1e3 * (t2 - t1)
    rep["cfg3_6d_1M_gammak_cold_solve"]["oracle_iterations"] = ost.iterations
    del o
    # sharded loop (NCCL, one rank) on the per-batch workload
    _, rows = gpu_replay(g6, 4096, n6, time_from=n6 - 10 * 4096, sharded=True)
    rep["cfg3_sharded_loop_1rank_S4096"] = exploit_summary(rows)

    # ---- configs[1]: 2-D 50k clutter, S = 1
    g2, _ = graph(2, 50_000 if not args.quick else 10_000, gen.gamma_star(2), 30, "suite_cfg2")
    _, rows = gpu_replay(g2, 1, g2.n)
    gsum = exploit_summary(rows)
    _, orows = oracle_replay(g2, 1, g2.n, budget_s=60)
    osum = exploit_summary(orows)
    rep["cfg2_2d_50k_clutter_S1"] = {"gpu": gsum, "oracle_sample": osum,
                                     "graph": {"n": g2.n, "mean_degree": g2.mean_degree}}

    # ---- configs[3]: 7-D 200k gamma_k, end-to-end plan time
    g7, tgen7 = graph(7, 200_000 if not args.quick else 40_000, gen.gamma_k(7), 30, "suite_cfg4")
    t0 = time.perf_counter()
    _, rows = gpu_replay(g7, 1000, g7.n)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, orows = oracle_replay(g7, 1000, g7.n, budget_s=None if not args.quick else 30)
    to = time.perf_counter() - t0
    rep["cfg4_7d_200k_end_to_end"] = {
        "exploration_s (generator, identical for both)": tgen7,
        "gpu_append_plus_exploit_s": tg, "oracle_append_plus_exploit_s": to,
        "gpu_plan_s": tgen7 + tg, "oracle_plan_s": tgen7 + to,
        "gpu": exploit_summary(rows), "oracle": exploit_summary(orows),
        "graph": {"n": g7.n, "mean_degree": g7.mean_degree},
    }

    # ---- configs[0]: 2-D 1k, single solve
    g1, _ = graph(2, 1000, gen.gamma_star(2), 0, "suite_cfg1")
    _, rows = gpu_replay(g1, g1.n, g1.n)
    _, orows = oracle_replay(g1, g1.n, g1.n)
    rep["cfg1_2d_1k_single_solve"] = {"gpu_exploit_ms": rows[0][1], "oracle_exploit_ms": orows[0][1],
                                      "iterations": rows[0][2].iterations}

    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(rep, open(args.out, "w"), indent=1, default=float)
    print(json.dumps(rep, indent=1, default=float))


if __name__ == "__main__":
    main()
