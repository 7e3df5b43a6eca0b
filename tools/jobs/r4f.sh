# larger compositor grids for the heavy (forward / back) frames, 14 lanes
B="python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 4 --warmup 3"
for h in 0.2 0.25 0.33; do $B --heavy-share $h > gpurun_out/r4f_h$h.json 2> gpurun_out/r4f_h$h.err; done
$B --heavy-share 0.25 --grid-share 0.125 > gpurun_out/r4f_h0.25_g0.125.json 2>/dev/null
$B > gpurun_out/r4f_base.json 2>/dev/null
