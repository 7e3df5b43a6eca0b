python paper_2503_11731_b200/build.py > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pixdist.py -x -q -rA > gpurun_out/r2_gpupix.log 2>&1; echo "pix rc=$?"
tail -8 gpurun_out/r2_gpupix.log
