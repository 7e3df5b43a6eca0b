# pinhole compositor at 48 registers: full GPU suite, bench
python paper_2503_11731_b200/build.py > gpurun_out/r2ab_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2ab_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/r2ab_gputest.log
timeout 900 python bench.py > gpurun_out/r2ab_bench.json 2> gpurun_out/r2ab_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2ab_bench.err
python -c "import json;d=json.load(open('gpurun_out/r2ab_bench.json'));print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['parity']['ok'])"
