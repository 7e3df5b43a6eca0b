# reordered onesweep: binning tests + ncu of the depth and tile passes of the forward camera
python paper_2503_11731_b200/build.py > gpurun_out/r3e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q > gpurun_out/r3e_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r3e_parity.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_onesweep -s 6 -c 6 -o gpurun_out/ncu_r3e_onesweep python tools/one_frame.py chunked 224 2 > gpurun_out/r3e_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r3e_ncu.log
