#!/bin/bash
# A/B of the early / mid sub-chunk lengths (AGFT_SUB_EARLY, AGFT_SUB_MID) on the full C4 day, alternating.
#   gpurun -- 'bash tools/gpu_sub_ab.sh <tag> "early:mid ..."'
set -u
TAG=$1; VARIANTS=$2
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2; do
  for V in $VARIANTS; do E=${V%%:*}; M=${V##*:}
    AGFT_SUB_EARLY=$E AGFT_SUB_MID=$M timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_${E}_${M}.json 2>> $O/err.log
  done
done
for V in $VARIANTS; do E=${V%%:*}; M=${V##*:}; python -c "
import json
for l in open('$O/bench_${E}_${M}.json'):
    d=json.loads(l); print('early=$E mid=$M', round(d['value']/1e9,4), d['ms_per_step'], {k:round(v.get('kernel_ms'),1) for k,v in d['roofline']['classes'].items()})
"; done > $O/ab_summary.txt
cat $O/ab_summary.txt
