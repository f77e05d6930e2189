set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --graph-cache /tmp/g1m.npz --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; cat gpurun_out/bench_r1b.json; tail -5 gpurun_out/bench_r1b.err
