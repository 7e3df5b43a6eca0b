# candidate/visible counts; bench stream-count sweep (short runs); ncu of the LiDAR k_tiles
python paper_2503_11731_b200/build.py > gpurun_out/r2u_build.log 2>&1
timeout 300 python tools/counts.py 224 225 226 227 230 > gpurun_out/r2u_counts.txt 2>&1; cat gpurun_out/r2u_counts.txt
for sa in "8 0.25" "10 0.2" "12 0.1667" "12 0.25" "16 0.125"; do
  set -- $sa
  timeout 600 python bench.py --streams $1 --grid-share $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/r2u_b_$1_$2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r2u_b_$1_$2.json'));print('streams $1 share $2', d['value'], d['ms_per_step'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_project|k_cull" -c 3 -o /tmp/r2u_f230 python tools/one_frame.py chunked 230 1 > gpurun_out/r2u_ncu_230.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/r2u_f230.ncu-rep gpurun_out/r2u_ncu_f230.md > /dev/null 2>&1
python tools/src_hot.py /tmp/r2u_f230.ncu-rep 40 k_tiles > gpurun_out/r2u_src_tiles.txt 2>&1
python tools/src_hot.py /tmp/r2u_f230.ncu-rep 40 k_project > gpurun_out/r2u_src_proj.txt 2>&1
cat gpurun_out/r2u_ncu_f230.md
