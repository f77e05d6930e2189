"""configs[1] record once (bench.config2_record): per-replan exploit times.
    python tools/cfg2_once.py"""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.config2_record(types.SimpleNamespace(seed=0))
print(json.dumps({"exploit_ms": r["exploit_ms"], "iterations_mean": r["iterations_mean"],
                  "barriers": r["counters"]["barriers"], "replans": r["replans"]}))
