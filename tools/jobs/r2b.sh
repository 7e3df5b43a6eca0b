python paper_2503_11731_b200/build.py > gpurun_out/r2b_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2b_gputest.log
for v in base new; do
  lib=""; [ $v = base ] && lib=paper_2503_11731_b200/libgsr_base.so
  env ${lib:+GSR_DEV_LIB=$lib} timeout 600 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2b_sweep_$v.jsonl 2>&1
  env ${lib:+GSR_DEV_LIB=$lib} timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2b_sweep_$v.jsonl 2>&1
done
grep -h frame gpurun_out/r2b_sweep_*.jsonl
timeout 2400 python tools/parity_full.py gpurun_out/parity_r02.json > gpurun_out/r2b_parity.log 2>&1; echo "parity rc=$?"
tail -2 gpurun_out/r2b_parity.log
