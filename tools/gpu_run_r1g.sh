export PIRRT_WATCHDOG_MS=20000
PIRRT_COMPACT_MIN=1e12 timeout 150 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -8
DBG_FROM=930 timeout 100 python tools/debug_parity.py 2 6000 30 1 cfg2 2>&1 | tail -25
