B="python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 4 --warmup 3"
for s in 16 20 24; do $B --streams $s > gpurun_out/ab2_streams$s.json 2>gpurun_out/ab2_streams$s.err; done
$B --streams 14 --grid-share 0.2 > gpurun_out/ab2_s14_gs20.json 2>/dev/null
$B --streams 14 --grid-share 0.11 > gpurun_out/ab2_s14_gs11.json 2>/dev/null
$B --streams 16 --grid-share 0.16 > gpurun_out/ab2_s16_gs16.json 2>/dev/null
$B --streams 14 > gpurun_out/ab2_s14.json 2>/dev/null
