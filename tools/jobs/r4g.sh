# typed dealing (lanes specialise on a frame class, lane counts proportional to class work)
B="python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 4 --warmup 3"
for s in 14 12 16; do $B --streams $s --deal typed > gpurun_out/r4g_s${s}_typed.json 2> gpurun_out/r4g_s${s}_typed.err; done
$B --streams 14 --deal typed --grid-share 0.2 > gpurun_out/r4g_s14_typed_gs20.json 2>/dev/null
$B --streams 16 --deal typed --grid-share 0.143 > gpurun_out/r4g_s16_typed_gs143.json 2>/dev/null
python -m pytest tests/test_gpu_parity.py -x -q -k "batch or Batch" > gpurun_out/r4g_batch_tests.log 2>&1
