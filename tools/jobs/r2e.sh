python paper_2503_11731_b200/build.py > gpurun_out/r2e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_neural.py tests/test_gpu_guard.py -x -q > gpurun_out/r2e_test.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r2e_test.log
timeout 300 python tools/bench_decode.py > gpurun_out/r2e_decode.jsonl 2>&1; echo "decode rc=$?"; cat gpurun_out/r2e_decode.jsonl
for cfg in fisheye lidar; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launch_$cfg.csv python tools/one_frame.py $cfg 0 2 > /dev/null 2>&1; echo "ncu $cfg rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launch_fwd.csv python tools/one_frame.py chunked 224 2 > /dev/null 2>&1; echo "ncu fwd rc=$?"
