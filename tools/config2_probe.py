"""configs[1] (2-D 50k clutter, S = 1) per-replan exploit times under a
sweep of settings (size-adaptive grid, incremental forms), through bench.py's
config-2 record.  python tools/config2_probe.py > gpurun_out/config2_sweep.json"""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

SETTINGS = [
    {},
    {"PIRRT_SMALL_GRID": "1"}, {"PIRRT_SMALL_GRID": "4"}, {"PIRRT_SMALL_GRID": "16"},
    {"PIRRT_SMALL_GRID": "37"}, {"PIRRT_SMALL_GRID": "74"}, {"PIRRT_SMALL_GRID": "148"},
    {"PIRRT_INC_IMPROVE": "0"}, {"PIRRT_INC_MAX": "0", "PIRRT_INC_IMPROVE": "0"},
]
a = types.SimpleNamespace(seed=0)
out = []
for env in SETTINGS[int(sys.argv[1]) if len(sys.argv) > 1 else 0:]:
    keys = ("PIRRT_SMALL_GRID", "PIRRT_INC_IMPROVE", "PIRRT_INC_MAX")
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update(env)
    r = bench.config2_record(a)
    r["env"] = env
    out.append(r)
    print(json.dumps({"env": env, "exploit_ms": r["exploit_ms"], "host": r["exploit_host_ms"],
                      "total": r["exploit_ms_total"]}), flush=True)
json.dump(out, open("gpurun_out/config2_sweep.json", "w"), indent=1)
