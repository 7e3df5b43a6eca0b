python paper_2503_11731_b200/build.py > gpurun_out/r2c_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_guard.py -x -q -rA > gpurun_out/r2c_guard.log 2>&1; echo "guard rc=$?"
grep -E "passed|failed|Error|assert" gpurun_out/r2c_guard.log | head -20
timeout 300 python tools/bench_decode.py > gpurun_out/r2c_decode.jsonl 2>&1; echo "decode rc=$?"; cat gpurun_out/r2c_decode.jsonl
timeout 600 python tools/bench_next.py backward stream > gpurun_out/r2c_next.jsonl 2>&1; echo "next rc=$?"; tail -5 gpurun_out/r2c_next.jsonl
timeout 300 python tools/sweep.py lidar 16x8 32x1 > gpurun_out/r2c_sweep_lidar.jsonl 2>&1
timeout 300 python tools/sweep.py fisheye 16x8 > gpurun_out/r2c_sweep_fisheye.jsonl 2>&1
cat gpurun_out/r2c_sweep_lidar.jsonl gpurun_out/r2c_sweep_fisheye.jsonl | grep frame
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_decode -c 2 -o gpurun_out/ncu_r2_decode python tools/bench_decode.py 2400000 2 > gpurun_out/r2c_ncu_decode.log 2>&1; echo "ncu rc=$?"
