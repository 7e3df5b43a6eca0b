python paper_2503_11731_b200/build.py > gpurun_out/r2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rA > gpurun_out/r2_gputest2.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest2.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2_bench1.err
python tools/dump_gpu.py gpurun_out/full_r02 full mid 540 1080 > gpurun_out/r2_dump_full2.log 2>&1; echo "dump rc=$?"
