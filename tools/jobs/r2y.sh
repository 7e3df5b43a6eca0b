# A/B: pinhole compositor register cap 64 (main) / 56 / 48
for v in main r56 r48; do
  lib=""; [ $v != main ] && lib=paper_2503_11731_b200/libgsr_$v.so
  env ${lib:+GSR_DEV_LIB=$lib} timeout 900 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2y_sweep_$v.jsonl 2>&1
  env ${lib:+GSR_DEV_LIB=$lib} timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2y_sweep_$v.jsonl 2>&1
done
grep -H '"fwd"\|"side"\|"mid"' gpurun_out/r2y_sweep_*.jsonl
