python paper_2503_11731_b200/build.py > gpurun_out/r2g_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q > gpurun_out/r2g_gputest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2g_gputest.log
timeout 300 python tools/sweep.py fisheye 16x8 > gpurun_out/r2g_sweep.jsonl 2>&1
timeout 300 python tools/sweep.py lidar 16x8 32x1 >> gpurun_out/r2g_sweep.jsonl 2>&1
timeout 600 python tools/sweep.py chunked 16x8,16x16 32x1 >> gpurun_out/r2g_sweep.jsonl 2>&1
timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2g_sweep.jsonl 2>&1
grep frame gpurun_out/r2g_sweep.jsonl
