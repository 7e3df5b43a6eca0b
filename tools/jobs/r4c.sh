# projection occupancy A/B: PROJ_MINB_CAM 2 / 3 (default) / 4, PROJ_MINB_LIDAR 2 / 3 / 4 (default) / 5
for v in default pm4 pm2 pl5 pl3 pl2; do
  if [ $v = default ]; then unset GSR_DEV_LIB; else export GSR_DEV_LIB=$PWD/paper_2503_11731_b200/libgsr_$v.so; fi
  python tools/sweep.py chunked 16x8 32x1 > gpurun_out/r4c_sweep_$v.log 2>&1
done
unset GSR_DEV_LIB
python -m pytest tests/test_gpu_dims.py -x -q > gpurun_out/r4c_dims.log 2>&1; echo "dims rc=$?" >> gpurun_out/r4c_dims.log
