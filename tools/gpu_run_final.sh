# final round measurement: bench (driver command shape), launch list, ncu full of the top kernel
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; cat gpurun_out/bench_final.json | cut -c1-300; tail -2 gpurun_out/bench_final.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-200 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 5 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches_final.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exploit_kernel --nvtx --nvtx-include "timed/" -c 2 -o gpurun_out/exploit_final python bench.py --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; ls -la gpurun_out/exploit_final.ncu-rep
