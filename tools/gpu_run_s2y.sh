timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "fused or variants or handover or children" 2>&1 | tail -2
for i in 1 2; do
for w in -1 1480 740; do
  PIRRT_WQ_WIDE=$w python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench6.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('wide=$w', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'])"
done
done
