export GRAPH_CACHE=/tmp/g1m.npz
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "children or wide or variants or lattice" 2>&1 | tail -2
PIRRT_KIDS_MIN=0 timeout 600 python tools/wide_probe.py 2>&1 | tail -1
timeout 600 python tools/wide_probe.py 2>&1 | tail -1
PIRRT_KIDS_MIN=20000 timeout 600 python tools/wide_probe.py 2>&1 | tail -1
