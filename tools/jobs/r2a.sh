# round 2 re-entry: full GPU suite, default bench, launch list of a short bench
python paper_2503_11731_b200/build.py > gpurun_out/r2a_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rA > gpurun_out/r2a_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2a_gputest.log
timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2a_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2a_launches.csv python bench.py --steps 1 --warmup 0 --timesteps 8 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/r2a_ncu.log 2>&1; echo "ncu rc=$?"
