export PIRRT_WATCHDOG_MS=30000
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
python -c "import torch;p=torch.cuda.get_device_properties(0);print('persist max', getattr(p,'persisting_l2_cache_max_size',None))"
for L2 in 1 0; do
PIRRT_L2_PERSIST=$L2 python bench.py --graph-cache /tmp/g1m.npz --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1h_$L2.json 2> gpurun_out/bench_r1h_$L2.err; python -c "
import json;d=json.load(open('gpurun_out/bench_r1h_$L2.json'));print('L2persist=$L2', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['e2e']['value'], d['roofline']['frac'])"; tail -2 gpurun_out/bench_r1h_$L2.err
done
PIRRT_L2_PERSIST=1 python tools/variant_probe.py 2>&1 | tail -1
