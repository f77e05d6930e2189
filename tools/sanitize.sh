# compute-sanitizer on the final code (gpurun -- bash tools/sanitize.sh);
# summaries to gpurun_out/sanitizer_*.txt.  memcheck runs every case;
# racecheck / synccheck (far slower) the S = 1 clutter shape, NEIGHBOURS and
# the deferred steps
set -x
mkdir -p gpurun_out
export PIRRT_WATCHDOG_MS=600000
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 \
    python tools/sanitize_workload.py > gpurun_out/sanitizer_memcheck.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer_memcheck.txt
for tool in racecheck synccheck; do
    timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
        python tools/sanitize_workload.py "cfg2 shape" neighbours steps > gpurun_out/sanitizer_$tool.txt 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer_$tool.txt
done
tail -n 12 gpurun_out/sanitizer_*.txt
