run() { python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench4.npz "$@" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', d['value'], d['exploit_ms_mean'], d['phase_ms'])"; }
run --grid-blocks 0
run --grid-blocks 148
run --grid-blocks 222
run --grid-blocks 256
run --grid-blocks 0
