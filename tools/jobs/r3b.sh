# TMA gather4 staging: parity + per-frame A/B against the previous build (libgsr_base.so)
python paper_2503_11731_b200/build.py > gpurun_out/r3b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dims.py -x -q > gpurun_out/r3b_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r3b_parity.log
for i in 1 2; do
for v in base tma; do
  lib=""; [ $v = base ] && lib="GSR_DEV_LIB=paper_2503_11731_b200/libgsr_base.so"
  env $lib timeout 600 python tools/sweep.py chunked 16x8 32x1 > gpurun_out/r3b_sweep_${v}_$i.jsonl 2>gpurun_out/r3b_sweep_$v.err; echo "$v rc=$?"
  cat gpurun_out/r3b_sweep_${v}_$i.jsonl | cut -c1-160
done
done
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/r3b_bench_tma.json 2>&1; tail -1 gpurun_out/r3b_bench_tma.json | cut -c1-200
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --priority comp > gpurun_out/r3b_bench_tma_comp.json 2>&1; tail -1 gpurun_out/r3b_bench_tma_comp.json | cut -c1-200
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --priority comp --grid-share 0.25 > gpurun_out/r3b_bench_tma_comp25.json 2>&1; tail -1 gpurun_out/r3b_bench_tma_comp25.json | cut -c1-200
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --priority comp --grid-share 0.15 > gpurun_out/r3b_bench_tma_comp15.json 2>&1; tail -1 gpurun_out/r3b_bench_tma_comp15.json | cut -c1-200
