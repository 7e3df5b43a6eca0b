# round 2 session 3 entry: full GPU suite and default bench of the current build
python paper_2503_11731_b200/build.py > gpurun_out/r2h_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rA > gpurun_out/r2h_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2h_gputest.log
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2h_bench.err
