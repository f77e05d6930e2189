# session-2 re-entry check: GPU parity suite + default bench at HEAD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2a_tests.log 2>&1; tail -3 gpurun_out/s2a_tests.log
python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err; cut -c1-600 gpurun_out/s2a_bench.json; tail -2 gpurun_out/s2a_bench.err
