# section 8(d) suite at the current code, e2e probe, gamma* config 3
timeout 2400 python tools/suite.py --out gpurun_out/suite_s2.json > gpurun_out/s2l_suite.log 2>&1; tail -3 gpurun_out/s2l_suite.log
timeout 600 python tools/e2e_probe.py 200000 > gpurun_out/s2l_e2e.log 2>&1; tail -16 gpurun_out/s2l_e2e.log
timeout 3000 python tools/gstar_probe.py --n 1000000 --oracle --out gpurun_out/gstar_1m.json > gpurun_out/s2l_gstar.log 2>&1; tail -8 gpurun_out/s2l_gstar.log
