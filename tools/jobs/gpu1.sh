python paper_2503_11731_b200/build.py > gpurun_out/r2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rA > gpurun_out/r2_gputest1.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest1.log
python tools/dump_gpu.py gpurun_out/full_r02 full mid 0 540 > gpurun_out/r2_dump_full.log 2>&1; echo "dump rc=$?"
