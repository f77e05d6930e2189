# row-stream cache hint A/B: 10M gamma_k cold, 1M gamma* cold (graphs built by the device Extend)
for lib in libpirrt_nostream.so libpirrt.so; do
  PIRRT_LIB=paper_2003_04920_b200/lib/$lib timeout 900 python tools/cfg5_extend_probe.py --batches 1 --out gpurun_out/s2w_10m_$lib.json 2>&1 | head -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib 10M gk', d['extend_s_total'], d['cold'])"
  PIRRT_LIB=paper_2003_04920_b200/lib/$lib timeout 900 python tools/cfg5_extend_probe.py --n 1000000 --gamma star --batches 1 --S 4096 --seed-tag cfg3_6d_1000000_gammastar_20boxes --out gpurun_out/s2w_1ms_$lib.json 2>&1 | head -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib 1M gstar', d['extend_s_total'], d['directed_edges'], d['cold'])"
done
