timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "sharded or wide" 2>&1 | tail -2
for i in 1 2 3; do
PIRRT_DEBUG_HOST=1 PIRRT_BENCH_VERBOSE=1 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench3.npz > gpurun_out/s2p_b$i.json 2> gpurun_out/s2p_b$i.err
python -c "import json;d=json.load(open('gpurun_out/s2p_b$i.json'));print(d['value'], d['exploit_ms_mean'], d['append_plus_readout_ms_mean'], d['e2e']['value'], d['e2e']['sync_value'])"
grep "dev step" gpurun_out/s2p_b$i.err | head -10
done
grep "append m=" gpurun_out/s2p_b3.err | tail -40
