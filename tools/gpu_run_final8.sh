# round-1 (session 2) measurement: GPU tests, default bench (driver command shape), reference arm,
mkdir -p gpurun_out/f8
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f8/tests.log 2>&1; tail -3 gpurun_out/f8/tests.log
python bench.py > gpurun_out/f8/bench.json 2> gpurun_out/f8/bench.err; cut -c1-300 gpurun_out/f8/bench.json; tail -2 gpurun_out/f8/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f8/bench_ref.json 2> gpurun_out/f8/bench_ref.err; cut -c1-300 gpurun_out/f8/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/f8/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph-cache /tmp/g_bench.npz > /dev/null 2>&1; wc -l gpurun_out/f8/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exploit_kernel --nvtx --nvtx-include "timed/" -c 2 -o gpurun_out/f8/exploit python bench.py --steps 3 --warmup 3 --no-cpu-baseline --graph-cache /tmp/g_bench.npz > /dev/null 2>&1; ls -la gpurun_out/f8/exploit.ncu-rep
