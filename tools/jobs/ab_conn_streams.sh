B="python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 4 --warmup 3"
for c in 4 6 12 16; do CUDA_DEVICE_MAX_CONNECTIONS=$c $B > gpurun_out/ab_conn$c.json 2>/dev/null; done
for s in 8 12 14; do $B --streams $s > gpurun_out/ab_streams$s.json 2>/dev/null; done
$B --streams 12 --grid-share 0.25 > gpurun_out/ab_streams12_gs25.json 2>/dev/null
$B --grid-share 0.25 > gpurun_out/ab_gs25.json 2>/dev/null
$B --grid-share 0.15 > gpurun_out/ab_gs15.json 2>/dev/null
$B > gpurun_out/ab_base.json 2>/dev/null
