# exact pinhole tile rows: binning tests, per-stage sweep, ncu of the forward / side frames (summaries made on the box)
python paper_2503_11731_b200/build.py > gpurun_out/r2j_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q -s -k "binning or ties" > gpurun_out/r2j_bintest.log 2>&1; echo "bintest rc=$?"
grep -E "binning|passed|failed|Error" gpurun_out/r2j_bintest.log | tail -8
timeout 900 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2j_sweep.jsonl 2>&1
timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2j_sweep.jsonl 2>&1
grep frame gpurun_out/r2j_sweep.jsonl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/r2j_gputest.log
for f in 224 225; do
  timeout 900 ncu --set full --clock-control none --import-source on -c 24 -o /tmp/r2j_f$f python tools/one_frame.py chunked $f 1 > gpurun_out/r2j_ncu_$f.log 2>&1; echo "ncu $f rc=$?"
  python tools/ncu_summary.py /tmp/r2j_f$f.ncu-rep gpurun_out/r2j_ncu_f$f.md > /dev/null 2>&1
  python tools/src_hot.py /tmp/r2j_f$f.ncu-rep 60 k_render_pinhole > gpurun_out/r2j_src_f$f.txt 2>&1
  ncu -i /tmp/r2j_f$f.ncu-rep --page raw --csv > gpurun_out/r2j_raw_f$f.csv 2>/dev/null
done
ls -la gpurun_out/
