# frame dealing A/B: round robin vs balanced (least planned pairs), 10 / 12 / 14 / 16 lanes
B="python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 4 --warmup 3"
for s in 14 12 10 16; do
  for d in round_robin balanced; do
    $B --streams $s --deal $d > gpurun_out/r4e_s${s}_$d.json 2> gpurun_out/r4e_s${s}_$d.err
  done
done
$B --streams 14 --deal balanced --grid-share 0.2 > gpurun_out/r4e_s14_balanced_gs20.json 2>/dev/null
