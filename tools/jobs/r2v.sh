# A/B: checkpoints per split segment 4 (main) / 8 / 12
for v in main ncp8 ncp12; do
  lib=""; [ $v != main ] && lib=paper_2503_11731_b200/libgsr_$v.so
  env ${lib:+GSR_DEV_LIB=$lib} timeout 900 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2v_sweep_$v.jsonl 2>&1
done
grep -H frame gpurun_out/r2v_sweep_*.jsonl
