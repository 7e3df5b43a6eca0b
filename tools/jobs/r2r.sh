# A/B: exact pinhole rows in k_project (variant) vs k_tiles (main)
for v in main rowsproj; do
  lib=""; [ $v = rowsproj ] && lib=paper_2503_11731_b200/libgsr_rowsproj.so
  env ${lib:+GSR_DEV_LIB=$lib} timeout 900 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2r_sweep_$v.jsonl 2>&1
  env ${lib:+GSR_DEV_LIB=$lib} timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2r_sweep_$v.jsonl 2>&1
done
grep -h frame gpurun_out/r2r_sweep_*.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q -s -k "binning or ties" > gpurun_out/r2r_bintest.log 2>&1; echo "bintest rc=$?"
grep -E "binning|passed|failed|Error" gpurun_out/r2r_bintest.log | tail -8
GSR_DEV_LIB=paper_2503_11731_b200/libgsr_rowsproj.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q -s -k "binning or ties" > gpurun_out/r2r_bintest_rp.log 2>&1; echo "bintest rowsproj rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2r_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/r2r_gputest.log
