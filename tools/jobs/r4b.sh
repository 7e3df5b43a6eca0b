# cull load grouping A/B: GSR_CULL_GROUP 1 / 2 / 4 / 8 (default build)
for v in cg1 cg2 cg4 default; do
  if [ $v = default ]; then unset GSR_DEV_LIB; else export GSR_DEV_LIB=$PWD/paper_2503_11731_b200/libgsr_$v.so; fi
  python tools/sweep.py chunked 16x8 32x1 > gpurun_out/r4b_sweep_$v.log 2>&1
  python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 4 --warmup 3 > gpurun_out/r4b_bench_$v.json 2>/dev/null
done
unset GSR_DEV_LIB
python -m pytest tests/test_gpu_dims.py -x -q > gpurun_out/r4b_dims.log 2>&1; echo "dims rc=$?" >> gpurun_out/r4b_dims.log
