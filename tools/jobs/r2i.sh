# ncu --set full of every kernel of one forward-camera (224), one side-camera (225) and one LiDAR (230) Chunked frame
python paper_2503_11731_b200/build.py > gpurun_out/r2i_build.log 2>&1
for f in 224 225 230; do
  timeout 900 ncu --set full --clock-control none --import-source on -c 24 -o gpurun_out/r2i_f$f python tools/one_frame.py chunked $f 1 > gpurun_out/r2i_ncu_$f.log 2>&1; echo "ncu $f rc=$?"
done
