for i in 1 2; do
for p in 1 0; do
PIRRT_L2_PERSIST=$p PIRRT_DEBUG_HOST=1 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench3.npz > gpurun_out/s2q_$p.json 2> gpurun_out/s2q_$p.err
python -c "import json;d=json.load(open('gpurun_out/s2q_$p.json'));print('persist=$p', d['value'], d['exploit_ms_mean'], d['append_plus_readout_ms_mean'], d['e2e']['value'], d['e2e']['sync_value'])"
grep "append m=" gpurun_out/s2q_$p.err | sed -n '5p;20p;40p'
done
done
