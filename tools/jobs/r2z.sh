# final-build evidence: ncu --set full of every kernel of a forward, side and LiDAR Chunked frame and the
# LiDAR and Fisheye config frames (summaries made on the box), launch list of the bench command (8 timesteps)
python paper_2503_11731_b200/build.py > gpurun_out/r2z_build.log 2>&1
for spec in "chunked 224" "chunked 225" "chunked 230" "fisheye 0" "lidar 0"; do
  set -- $spec; tag=$1_$2
  timeout 900 ncu --set full --clock-control none --import-source on -c 26 -o /tmp/r2z_$tag python tools/one_frame.py $1 $2 1 > gpurun_out/r2z_ncu_$tag.log 2>&1; echo "ncu $tag rc=$?"
  python tools/ncu_summary.py /tmp/r2z_$tag.ncu-rep gpurun_out/r2z_ncu_$tag.md > /dev/null 2>&1
  ncu -i /tmp/r2z_$tag.ncu-rep --page raw --csv > gpurun_out/r2z_raw_$tag.csv 2>/dev/null
done
python tools/src_hot.py /tmp/r2z_chunked_224.ncu-rep 60 k_render_pinhole > gpurun_out/r2z_src_render_224.txt 2>&1
python tools/src_hot.py /tmp/r2z_chunked_230.ncu-rep 40 "k_render<2" > gpurun_out/r2z_src_render_230.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2z_launches.csv python bench.py --steps 1 --warmup 0 --timesteps 8 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/r2z_ncu_bench.log 2>&1; echo "ncu bench rc=$?"
python tools/launch_summary.py gpurun_out/r2z_launches.csv 8 "round-2 final build" > gpurun_out/r2z_launches_summary.md 2>&1
gzip -f gpurun_out/r2z_launches.csv
ls -la gpurun_out | head -40
