# wide-Improve variants on the gamma* cold solve; e2e host timing (gpurun -- bash tools/gpu_debug.sh)
set -x
mkdir -p gpurun_out
for lib in libpirrt.so libpirrt_w32u4.so libpirrt_w32u8.so libpirrt_w16u8.so; do
    [ -f paper_2003_04920_b200/lib/$lib ] && PIRRT_LIB=paper_2003_04920_b200/lib/$lib timeout 300 python tools/wide_gstar_probe.py 2>&1 | tail -1
done
timeout 600 python tools/e2e_pipe_probe.py 2>&1 | tail -2
timeout 600 python tools/phase_probe.py 2>&1 | tail -3
