timeout 900 python -m pytest tests/test_parity_extend_gpu.py -m gpu -x -q 2>&1 | tail -2
timeout 1200 python tools/extend_probe.py --out gpurun_out/extend2.json 2>&1 | tail -4
