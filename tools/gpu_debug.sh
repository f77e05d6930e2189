# GPU session: the new group/partition tests, then the grid-size sweep
set -x
mkdir -p gpurun_out
export PIRRT_WATCHDOG_MS=20000
timeout 900 python -m pytest -m gpu -q --timeout 240 --timeout-method thread -rf \
    tests/test_parity_group_gpu.py tests/test_parity_gpu.py -k "group or shard" > gpurun_out/pytest_dbg.log 2>&1
tail -15 gpurun_out/pytest_dbg.log
timeout 1500 python tools/grid_probe.py > gpurun_out/grid_probe.jsonl 2> gpurun_out/grid_probe.err
cat gpurun_out/grid_probe.jsonl; tail -3 gpurun_out/grid_probe.err
