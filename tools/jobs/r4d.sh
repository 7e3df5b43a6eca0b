# final build of session 5 (block-bounds cull, hoisted cull constants, 14 lanes, host-side overflow check): GPU suite, smoke, bench line,
# launch list of the bench command (8 timesteps), ncu --set full of every kernel of a forward / side / LiDAR
# Chunked frame and the LiDAR / Fisheye config frames
python paper_2503_11731_b200/build.py > gpurun_out/r4d_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r4d_gputest.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/r4d_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r4d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/r4d_bench.json 2> gpurun_out/r4d_bench.err; echo "bench rc=$?"
tail -1 gpurun_out/r4d_bench.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4d_launches.csv python bench.py --steps 1 --warmup 0 --timesteps 8 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/r4d_ncu_bench.log 2>&1; echo "ncu bench rc=$?"
python tools/launch_summary.py gpurun_out/r4d_launches.csv 8 "round-2 final build (session 5: block-bounds cull, 14 lanes of two streams, compositing high priority)" > gpurun_out/r4d_launches_summary.md 2>&1
gzip -f gpurun_out/r4d_launches.csv
for spec in "chunked 224" "chunked 225" "chunked 230" "fisheye 0" "lidar 0"; do
  set -- $spec; tag=$1_$2
  timeout 900 ncu --set full --clock-control none --import-source on -c 27 -o /tmp/r4d_$tag python tools/one_frame.py $1 $2 1 > gpurun_out/r4d_ncu_$tag.log 2>&1; echo "ncu $tag rc=$?"
  ncu -i /tmp/r4d_$tag.ncu-rep --page raw --csv > gpurun_out/r4d_raw_$tag.csv 2>/dev/null
done
python tools/src_hot.py /tmp/r4d_chunked_224.ncu-rep 40 "k_cull" > gpurun_out/r4d_src_cull_224.txt 2>&1
ls -la gpurun_out | grep r4a
