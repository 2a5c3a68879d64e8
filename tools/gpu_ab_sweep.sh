#!/bin/bash
# Alternating sweep-bench A/B (window-arm evaluations/s) of the working tree's library against variants.
#   gpurun -- 'bash tools/gpu_ab_sweep.sh <tag> <name>=<.so> ...'
set -u
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
VARS="new=paper_2508_01744_b200/libagft.so $*"
for rep in 1 2; do
  for NV in $VARS; do N=${NV%%=*}; L=${NV#*=}
    AGFT_LIB_PATH=$L timeout 600 python bench.py --workload sweep --steps 3 --warmup 3 >> $O/sweep_$N.json 2>> $O/sweep.err
  done
done
for NV in $VARS; do N=${NV%%=*}; python -c "
import json
for l in open('$O/sweep_$N.json'): d=json.loads(l); print('sweep $N', d['value'], d['ms_per_step'])"; done >> $O/ab_summary.txt
cat $O/ab_summary.txt
