# packed f32x2 pinhole eval: binning tests, sweeps, full GPU suite, bench
python paper_2503_11731_b200/build.py > gpurun_out/r2x_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q -s -k "binning or ties" > gpurun_out/r2x_bintest.log 2>&1; echo "bintest rc=$?"
grep -E "binning|passed|failed|Error" gpurun_out/r2x_bintest.log | tail -8
timeout 900 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2x_sweep.jsonl 2>&1
timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2x_sweep.jsonl 2>&1
timeout 300 python tools/sweep.py lidar 16x8 32x1 >> gpurun_out/r2x_sweep.jsonl 2>&1
grep -h frame gpurun_out/r2x_sweep.jsonl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/r2x_gputest.log
timeout 900 python bench.py > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2x_bench.err
