# stream-priority A/B on the Chunked batch (no e2e / cpu / configs legs)
for v in "none 10" "pre 10" "comp 10" "pre 12" "none 10"; do
  set -- $v
  timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --priority $1 --streams $2 > gpurun_out/r3a_$1_$2.json 2> gpurun_out/r3a_$1_$2.err; echo "$1 $2 rc=$?"
  tail -1 gpurun_out/r3a_$1_$2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --priority pre --grid-share 0.3 > gpurun_out/r3a_pre_gs3.json 2>&1; tail -1 gpurun_out/r3a_pre_gs3.json | cut -c1-200
