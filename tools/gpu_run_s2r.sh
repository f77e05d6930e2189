timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2r_tests.log 2>&1; tail -15 gpurun_out/s2r_tests.log
timeout 1200 python tools/extend_probe.py --out gpurun_out/extend.json 2>&1 | tail -4
