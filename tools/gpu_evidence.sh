# evidence session (gpurun -- bash tools/gpu_evidence.sh): GPU tests, the
# bench line (driver command) + reference arm, ncu launch list and one
# --set full capture of exploit_kernel (compute-sanitizer is closed on this
# pool)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PIRRT_WATCHDOG_MS=20000
timeout 1800 python -m pytest -m gpu -q --timeout 300 --timeout-method thread -rf --durations 10 tests \
    > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
( time timeout 1200 python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 1500 gpurun_out/bench_final.json; tail -4 gpurun_out/bench_final.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 800 gpurun_out/bench_ref.json; tail -4 gpurun_out/bench_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline \
    > gpurun_out/ncu_launch_run.log 2>&1
wc -l gpurun_out/launches.csv
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:exploit_kernel -s 236 -c 3 \
    -o gpurun_out/exploit_prof python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline \
    > gpurun_out/ncu_full_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_append_fused -s 236 -c 2 \
    -o gpurun_out/append_prof python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline \
    > gpurun_out/ncu_append_run.log 2>&1
tail -3 gpurun_out/ncu_full_run.log gpurun_out/ncu_append_run.log
