# one compute-sanitizer tool per call: bash tools/jobs/san.sh <tool>
tool=$1
python paper_2503_11731_b200/build.py > gpurun_out/san_build.log 2>&1
extra=""
[ $tool = racecheck ] && extra="--racecheck-report all"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 \
  python tools/sanitize_cases.py > gpurun_out/san_r02_$tool.log 2>&1; echo "$tool rc=$?"
tail -4 gpurun_out/san_r02_$tool.log
