# measurement after the Evaluate rework: GPU tests, default bench (driver command shape),
# launch list and one ncu --set full capture of exploit_kernel
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f2_tests.log 2>&1; tail -3 gpurun_out/f2_tests.log
python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; cut -c1-400 gpurun_out/f2_bench.json; tail -2 gpurun_out/f2_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/f2_launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exploit_kernel --nvtx --nvtx-include "timed/" -c 2 -o gpurun_out/f2_exploit python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; ls -la gpurun_out/f2_exploit.ncu-rep
