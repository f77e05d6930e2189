timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "children or wide or lattice or variants" 2>&1 | tail -2
export GRAPH_CACHE=/tmp/g1m.npz
timeout 600 python tools/wide_probe.py 2>&1 | tail -1
timeout 600 python tools/cfg5_extend_probe.py --batches 3 --out gpurun_out/cfg5_b.json 2>&1 | head -1 | cut -c1-600
for i in 1 2; do
  (cd old_ref && python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('old', d['value'], d['exploit_ms_mean'], d['phase_ms'])")
  python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench5.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('new', d['value'], d['exploit_ms_mean'], d['phase_ms'])"
done
