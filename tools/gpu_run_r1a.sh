set -x
nproc
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py --graph-cache /tmp/g1m.npz --steps 20 --warmup 3 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; cat gpurun_out/bench_r1a.json; tail -5 gpurun_out/bench_r1a.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_r1a.csv python bench.py --graph-cache /tmp/g1m.npz --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; tail -3 gpurun_out/bench_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exploit_kernel --nvtx --nvtx-include "timed/" -c 2 -o gpurun_out/exploit_r1a python bench.py --graph-cache /tmp/g1m.npz --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
