python paper_2503_11731_b200/build.py > gpurun_out/r2d_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_neural.py tests/test_gpu_guard.py -x -q > gpurun_out/r2d_test.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2d_test.log
timeout 300 python tools/bench_decode.py > gpurun_out/r2d_decode.jsonl 2>&1; echo "decode rc=$?"; cat gpurun_out/r2d_decode.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_decode -c 2 -o gpurun_out/ncu_r2d_decode python tools/bench_decode.py 2400000 2 > gpurun_out/r2d_ncu_decode.log 2>&1; echo "ncu rc=$?"
