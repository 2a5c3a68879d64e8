#!/bin/bash
# A/B of the records-chunk length and the late sub-chunk length on the full C4 day (one box,
# alternating runs).   gpurun -- 'bash tools/gpu_chunk_ab.sh <tag> "chunk:late ..."'
set -u
TAG=$1; VARIANTS=$2; REPS=${3:-2}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in $(seq $REPS); do
  for V in $VARIANTS; do C=${V%%:*}; L=${V##*:}
    AGFT_SUB_LATE=$L timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --chunk $C >> $O/bench_${C}_${L}.json 2>> $O/err.log
  done
done
for V in $VARIANTS; do C=${V%%:*}; L=${V##*:}; python -c "
import json
for l in open('$O/bench_${C}_${L}.json'):
    d=json.loads(l); print('chunk=$C late=$L', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity'].get('match') if isinstance(d.get('parity'),dict) else None, {k:v.get('kernel_ms') for k,v in d['roofline']['classes'].items()})
"; done > $O/ab_summary.txt
cat $O/ab_summary.txt
