python paper_2503_11731_b200/build.py > gpurun_out/r2_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_backward.py -x -q -rA > gpurun_out/r2_gpubwd.log 2>&1; echo "bwd rc=$?"
grep -E "^E |passed|failed|^pinhole" gpurun_out/r2_gpubwd.log | head -30
