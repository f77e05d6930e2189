export PIRRT_WATCHDOG_MS=30000
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
python bench.py --graph-cache /tmp/g1m.npz --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1i.json 2> gpurun_out/bench_r1i.err; python -c "
import json;d=json.load(open('gpurun_out/bench_r1i.json'));print(d['value'], d['exploit_ms_mean'], d['phase_ms'], d['e2e']['value'], d['roofline']['frac'])"; tail -2 gpurun_out/bench_r1i.err
python tools/variant_probe.py 2>&1 | tail -1
