# gamma* config 3 (1M 6-D) and config 4 (200k 7-D) with the fold charged to its append
timeout 3000 python tools/gstar_probe.py --n 1000000 --cache /tmp/g1m_star.npz --out gpurun_out/gstar_1m_b.json > gpurun_out/s2m_gstar.log 2>&1; tail -4 gpurun_out/s2m_gstar.log
timeout 3000 python tools/gstar_probe.py --d 7 --n 200000 --boxes 30 --S 1000 --pre 20000 --oracle --out gpurun_out/gstar_7d_200k.json > gpurun_out/s2m_gstar7.log 2>&1; tail -4 gpurun_out/s2m_gstar7.log
