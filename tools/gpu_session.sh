# one GPU session: GPU tests (a hung test is killed by pytest-timeout's
# thread method and reported), then a short bench
#   gpurun -- bash tools/gpu_session.sh [pytest paths]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PIRRT_WATCHDOG_MS=20000
bash tools/gpu_debug.sh
timeout 1800 python -m pytest -m gpu -q --timeout 240 --timeout-method thread -rf --durations 20 \
    ${@:-tests} > gpurun_out/pytest_gpu.log 2>&1
tail -45 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
tail -c 3000 gpurun_out/bench_r2.json; tail -5 gpurun_out/bench_r2.err
