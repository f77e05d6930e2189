export PIRRT_WATCHDOG_MS=600000
timeout 300 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -12
export PIRRT_WATCHDOG_MS=20000
timeout 300 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -12
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/debug_parity.py 2 1000 0 7 cfg1 2>&1 | tail -12
