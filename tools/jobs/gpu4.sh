python paper_2503_11731_b200/build.py > gpurun_out/r2_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q -rA > gpurun_out/r2_gpustream.log 2>&1; echo "stream rc=$?"
tail -4 gpurun_out/r2_gpustream.log
timeout 300 python tools/bench_decode.py > gpurun_out/r2_decode_bench.jsonl 2>&1; echo "decode rc=$?"; cat gpurun_out/r2_decode_bench.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_decode -c 2 -o gpurun_out/ncu_r2_decode python tools/bench_decode.py 2400000 2 > gpurun_out/r2_ncu_decode.log 2>&1; echo "ncu rc=$?"
for g in graph nograph; do
  extra=""; [ $g = nograph ] && extra="--no-graph"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-configs $extra > gpurun_out/r2_ab_$g.json 2> gpurun_out/r2_ab_$g.err; echo "$g rc=$?"
done
python tools/dump_gpu.py gpurun_out/full_r02 full fisheye 512 1024 > gpurun_out/r2_dump_full4.log 2>&1; echo "dump rc=$?"
