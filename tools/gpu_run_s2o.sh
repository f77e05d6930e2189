ls -la /tmp/*.npz
python tools/h2d_probe.py
PIRRT_DEBUG_HOST=1 timeout 1500 python tools/gstar_probe.py --n 1000000 --cache /tmp/g1m_star.npz --out gpurun_out/gstar_1m_d.json 2>&1 | tail -8
