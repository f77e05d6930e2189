# goal set, parent form, VALIDATE: GPU parity suite + bench
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2b_tests.log 2>&1; tail -15 gpurun_out/s2b_tests.log
python bench.py --no-cpu-baseline > gpurun_out/s2b_bench.json 2> gpurun_out/s2b_bench.err; cut -c1-300 gpurun_out/s2b_bench.json; tail -2 gpurun_out/s2b_bench.err
