# Evaluate work-queue knobs at the bench workload (values per 296 blocks)
run() { env "$@" python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench4.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', d['value'], d['exploit_ms_mean'], d['phase_ms'])"; }
run PIRRT_X=0
run PIRRT_WQ_KEEP=16
run PIRRT_WQ_KEEP=48
run PIRRT_WQ_KEEP=64
run PIRRT_WQ_WIDE=1480
run PIRRT_WQ_WIDE=5920
run PIRRT_WQ_TAIL=2368
run PIRRT_WQ_TAIL=9472
run PIRRT_WQ_TAIL=0
run PIRRT_X=0
