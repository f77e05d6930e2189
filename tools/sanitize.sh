# compute-sanitizer on the final code (gpurun -- bash tools/sanitize.sh);
# summaries to gpurun_out/sanitizer_*.txt
set -x
mkdir -p gpurun_out
export PIRRT_WATCHDOG_MS=600000
for tool in memcheck racecheck synccheck; do
    timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
        python tools/sanitize_workload.py > gpurun_out/sanitizer_$tool.txt 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer_$tool.txt
    tail -12 gpurun_out/sanitizer_$tool.txt
done
