# load-balanced k_tiles: binning tests, sweeps, bench
python paper_2503_11731_b200/build.py > gpurun_out/r2n_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q -s -k "binning or ties" > gpurun_out/r2n_bintest.log 2>&1; echo "bintest rc=$?"
grep -E "binning|passed|failed|Error" gpurun_out/r2n_bintest.log | tail -8
timeout 900 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2n_sweep.jsonl 2>&1
timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2n_sweep.jsonl 2>&1
timeout 300 python tools/sweep.py lidar 16x8 32x1 >> gpurun_out/r2n_sweep.jsonl 2>&1
grep -h frame gpurun_out/r2n_sweep.jsonl
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2n_bench.err
