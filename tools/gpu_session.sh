# one GPU session: GPU tests + a short bench (gpurun -- bash tools/gpu_session.sh [pytest paths])
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PIRRT_WATCHDOG_MS=20000
timeout 1500 python -m pytest -m gpu -x -q ${@:-tests} 2>&1 | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
tail -c 2500 gpurun_out/bench_r2.json; tail -5 gpurun_out/bench_r2.err
