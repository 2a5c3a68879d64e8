#!/bin/bash
# A/B of class-stream priority orders (AGFT_PRIO_ORDER, class ids of agft_internal.cuh, highest first).
#   gpurun -- 'bash tools/gpu_prio_ab.sh <tag> "o1 o2 ..."'   (orders as comma lists)
set -u
TAG=$1; ORDERS=$2
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2; do
  for V in $ORDERS; do
    AGFT_PRIO_ORDER=$V timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_$V.json 2>> $O/err.log
  done
done
for V in $ORDERS; do python -c "
import json
for l in open('$O/bench_$V.json'):
    d=json.loads(l); print('order=$V', round(d['value']/1e9,4), d['ms_per_step'])
"; done > $O/ab_summary.txt
cat $O/ab_summary.txt
