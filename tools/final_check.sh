#!/bin/bash
# Final-session check: GPU suite, the default bench line, the configs[4]
# single-GPU bench line and the cfg5 probe.  bash tools/final_check.sh
export PIRRT_WATCHDOG_MS=60000
mkdir -p gpurun_out
timeout 1500 python -m pytest -m gpu -q --timeout 1200 tests 2>&1 | tail -4 > gpurun_out/fc_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fc_cfg5.json 2> gpurun_out/fc_cfg5.err
timeout 300 python tools/cfg5_extend_probe.py --n 10000000 --out gpurun_out/fc_cfg5_probe.json > /dev/null 2>&1
cat gpurun_out/fc_pytest.txt
