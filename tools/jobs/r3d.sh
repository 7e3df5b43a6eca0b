# onesweep: look-back after the shared-memory staging, window 8 / 16 / 32
for i in 1 2; do
for v in rb8 rb16 rb32; do
  GSR_DEV_LIB=paper_2503_11731_b200/libgsr_$v.so timeout 600 python tools/sweep.py chunked 16x8 32x1 > gpurun_out/r3d_sweep_${v}_$i.jsonl 2>gpurun_out/r3d_sweep_$v.err; echo "$v rc=$?"
  cut -c1-150 gpurun_out/r3d_sweep_${v}_$i.jsonl
done
done
for v in rb8 rb32; do
  GSR_DEV_LIB=paper_2503_11731_b200/libgsr_$v.so timeout 600 python tools/sweep.py mid 16x8 32x1 | cut -c1-150
  GSR_DEV_LIB=paper_2503_11731_b200/libgsr_$v.so timeout 600 python tools/sweep.py lidar 16x8 32x1 | cut -c1-150
done
