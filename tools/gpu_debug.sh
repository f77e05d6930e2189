# debugging session (gpurun -- bash tools/gpu_debug.sh): the gamma* cold
# solve at full size with and without the incremental Improve, then the GPU
# suite with a per-test timeout (which tests hang or fail)
set -x
mkdir -p gpurun_out
export PIRRT_WATCHDOG_MS=10000
PIRRT_INC_IMPROVE=0 timeout 300 python tools/repro_cold.py --n 1000000 2>&1 | tail -3
timeout 300 python tools/repro_cold.py --n 1000000 2>&1 | tail -3
timeout 300 python tools/repro_cold.py --n 1000000 --gamma k 2>&1 | tail -3
timeout 1500 python -m pytest -m gpu -q --timeout 120 -rf --durations 15 tests > gpurun_out/pytest_dbg.log 2>&1
tail -60 gpurun_out/pytest_dbg.log
