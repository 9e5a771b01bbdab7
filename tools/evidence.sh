#!/bin/bash
# One GPU-box pass that refreshes the judged evidence of the current build (outputs in gpurun_out/):
#   sanitizers over every entry point, an ncu --set full capture of one config-2 chunk step, the ncu
#   launch list of a short bench run, the bench line and the reference-arm line.
#   gpurun --timeout 2400 -- bash tools/evidence.sh <tag>
set -u
tag=${1:-ev}
mkdir -p gpurun_out /tmp/rep
for tool in memcheck initcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_paths.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazards displayed|sanitize paths ok|Error|error" | head -8
done > gpurun_out/${tag}_sanitize.txt 2>&1
timeout 900 ncu --set full --clock-control none --profile-from-start off -o /tmp/rep/${tag}_c2 -f \
  python tools/prof_step.py --config 2 > gpurun_out/${tag}_c2_ncu.log 2>&1
ncu -i /tmp/rep/${tag}_c2.ncu-rep --page raw --csv > gpurun_out/${tag}_c2_raw.csv 2>>gpurun_out/${tag}_c2_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_reference.log 2>&1
tail -1 gpurun_out/${tag}_bench.log | cut -c1-300
tail -1 gpurun_out/${tag}_reference.log | cut -c1-300
cat gpurun_out/${tag}_sanitize.txt
