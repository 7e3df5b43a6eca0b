# bench line of the committed build (default flags) + launch list of the bench command
python paper_2503_11731_b200/build.py > gpurun_out/r3f_build.log 2>&1
timeout 1200 python bench.py > gpurun_out/r3f_bench.json 2> gpurun_out/r3f_bench.err; echo "bench rc=$?"
tail -1 gpurun_out/r3f_bench.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3f_launches.csv python bench.py --steps 1 --warmup 0 --timesteps 8 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/r3f_ncu_bench.log 2>&1; echo "ncu bench rc=$?"
python tools/launch_summary.py gpurun_out/r3f_launches.csv 8 "round-2 final build (two streams per lane, compositing high priority)" > gpurun_out/r3f_launches_summary.md 2>&1
gzip -f gpurun_out/r3f_launches.csv
