#!/bin/bash
# A/B of an environment knob on the full C4 bench (alternating runs on one box).
#   gpurun -- 'bash tools/gpu_ab.sh <tag> VAR valA valB [tests]'
set -u
TAG=$1; VAR=$2; A=$3; B=$4; TESTS=${5:-notests}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [ "$TESTS" = tests ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
for V in $A $B $A $B; do
  env $VAR=$V timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_${VAR}_$V.json 2>> $O/bench_ab.err
done
for V in $A $B; do python -c "
import json
for l in open('$O/bench_${VAR}_$V.json'):
    d=json.loads(l); print('$VAR=$V', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['all_steps_complete'], {k:v.get('kernel_ms') for k,v in d['roofline']['classes'].items()})
"; done > $O/ab_summary.txt
