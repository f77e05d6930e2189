export PIRRT_WATCHDOG_MS=20000
timeout 120 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5
for mode in async level; do
PIRRT_BFS=$mode python bench.py --graph-cache /tmp/g1m.npz --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1d_$mode.json 2> gpurun_out/bench_r1d_$mode.err; python -c "
import json;d=json.load(open('gpurun_out/bench_r1d_$mode.json'));print('$mode', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['e2e']['value'], d['roofline']['frac'])"; tail -2 gpurun_out/bench_r1d_$mode.err
done
