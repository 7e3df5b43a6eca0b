python paper_2503_11731_b200/build.py > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dims.py -k cylindrical -x -q -rA > gpurun_out/r2_gpucyl.log 2>&1; echo "cyl rc=$?"
tail -6 gpurun_out/r2_gpucyl.log
