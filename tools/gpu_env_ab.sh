#!/bin/bash
# Alternating A/B of environment knobs of the library on the full C4 day (one box).  Each variant is a
# comma-free list of VAR=value pairs joined by '+', e.g.
#   gpurun -- 'bash tools/gpu_env_ab.sh <tag> "AGFT_SUB_EARLY=256+AGFT_SUB_MID=1024 AGFT_SUB_EARLY=128"'
# Knobs: AGFT_SUB_EARLY / AGFT_SUB_MID / AGFT_SUB_LATE (sub-chunk lengths), AGFT_PRIO_ORDER (class-stream
# priorities, class ids highest first, e.g. 2:1:3:0:5:4), AGFT_STREAM_PRIO=0; bench args after "--".
set -u
TAG=$1; VARIANTS=$2; shift 2
[ "${1:-}" = "--" ] && shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2; do
  for V in $VARIANTS; do
    ENVS=$(echo "$V" | tr '+' ' ' | tr ':' ',')
    env $ENVS timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" >> "$O/bench_$V.json" 2>> $O/err.log
  done
done
for V in $VARIANTS; do python -c "
import json
for l in open('$O/bench_$V.json'):
    d=json.loads(l); print('$V', round(d['value']/1e9,4), d['ms_per_step'], {k:round(v.get('kernel_ms'),1) for k,v in d['roofline']['classes'].items()})
"; done > $O/ab_summary.txt
cat $O/ab_summary.txt
