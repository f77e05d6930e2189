export PIRRT_WATCHDOG_MS=20000
timeout 300 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -30
timeout 60 /tmp/barrier_bench 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb tools/barrier_bench.cu && timeout 60 /tmp/bb)
