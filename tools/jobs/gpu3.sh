python paper_2503_11731_b200/build.py > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_neural.py -x -q -rA > gpurun_out/r2_gpuneural.log 2>&1; echo "neural rc=$?"
tail -5 gpurun_out/r2_gpuneural.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r2_bench2.err
python tools/dump_gpu.py gpurun_out/full_r02 full fisheye 0 512 > gpurun_out/r2_dump_full3.log 2>&1; echo "dump rc=$?"
