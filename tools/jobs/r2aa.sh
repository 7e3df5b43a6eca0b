# A/B: pinhole compositor registers 48 (main) / 44 / 40; LiDAR-fisheye compositor 64 (main) / 56 / 48
for v in main ph44 ph40 ray56 ray48; do
  lib=""; [ $v != main ] && lib=paper_2503_11731_b200/libgsr_$v.so
  env ${lib:+GSR_DEV_LIB=$lib} timeout 900 python tools/sweep.py chunked 16x8,16x16 32x1 > gpurun_out/r2aa_sweep_$v.jsonl 2>&1
  env ${lib:+GSR_DEV_LIB=$lib} timeout 300 python tools/sweep.py mid 16x8 >> gpurun_out/r2aa_sweep_$v.jsonl 2>&1
  env ${lib:+GSR_DEV_LIB=$lib} timeout 300 python tools/sweep.py lidar 16x8 32x1 >> gpurun_out/r2aa_sweep_$v.jsonl 2>&1
  env ${lib:+GSR_DEV_LIB=$lib} timeout 300 python tools/sweep.py fisheye 16x8 >> gpurun_out/r2aa_sweep_$v.jsonl 2>&1
done
for v in main ph44 ph40 ray56 ray48; do echo $v; python -c "
import json
for l in open('gpurun_out/r2aa_sweep_$v.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('  ', d['frame'], d['tile'], d['ms_render'])
"; done
