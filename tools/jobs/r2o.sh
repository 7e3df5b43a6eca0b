# ncu of k_tiles / k_emit / k_project for a forward and a LiDAR frame
python paper_2503_11731_b200/build.py > gpurun_out/r2o_build.log 2>&1
for f in 224 230; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_emit|k_project|k_cull|k_onesweep" -c 12 -o /tmp/r2o_f$f python tools/one_frame.py chunked $f 1 > gpurun_out/r2o_ncu_$f.log 2>&1; echo "ncu $f rc=$?"
  python tools/ncu_summary.py /tmp/r2o_f$f.ncu-rep gpurun_out/r2o_ncu_f$f.md > /dev/null 2>&1
  python tools/src_hot.py /tmp/r2o_f$f.ncu-rep 40 k_tiles > gpurun_out/r2o_src_tiles_f$f.txt 2>&1
  ncu -i /tmp/r2o_f$f.ncu-rep --page raw --csv > gpurun_out/r2o_raw_f$f.csv 2>/dev/null
done
