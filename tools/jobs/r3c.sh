# onesweep look-back window A/B: 8 (libgsr.so) vs 16 vs 32 predecessors per round trip
python paper_2503_11731_b200/build.py > gpurun_out/r3c_build.log 2>&1
for i in 1 2; do
for v in lb8 lb16 lb32 tma2 tma2p; do
  lib=""; [ $v != lb8 ] && lib="GSR_DEV_LIB=paper_2503_11731_b200/libgsr_$v.so"
  env $lib timeout 600 python tools/sweep.py chunked 16x8 32x1 > gpurun_out/r3c_sweep_${v}_$i.jsonl 2>gpurun_out/r3c_sweep_$v.err; echo "$v rc=$?"
  cat gpurun_out/r3c_sweep_${v}_$i.jsonl | cut -c1-150
done
done
for v in lb8 lb16; do
  lib=""; [ $v != lb8 ] && lib="GSR_DEV_LIB=paper_2503_11731_b200/libgsr_$v.so"
  env $lib timeout 600 python tools/sweep.py mid 16x8 32x1 | cut -c1-150
done
