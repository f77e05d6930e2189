# the goal-set tests after the list-stamp fix (gpurun -- bash tools/gpu_debug.sh)
set -x
mkdir -p gpurun_out
export PIRRT_WATCHDOG_MS=20000
timeout 900 python -m pytest -m gpu -q --timeout 240 --timeout-method thread -rf -x \
    tests/test_parity_goals_variants_gpu.py tests/test_parity_gpu.py tests/test_parity_r2_gpu.py > gpurun_out/pytest_dbg.log 2>&1
tail -15 gpurun_out/pytest_dbg.log
