# full bench (driver command) + reference arm, timed (gpurun -- bash tools/gpu_bench.sh)
set -x
mkdir -p gpurun_out
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 6000 gpurun_out/bench_full.json; tail -20 gpurun_out/bench_full.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 3000 gpurun_out/bench_ref.json; tail -8 gpurun_out/bench_ref.err
