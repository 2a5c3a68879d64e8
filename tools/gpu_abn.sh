#!/bin/bash
# Alternating A/B/C… of the full C4 bench over several library builds on one box, after the parity
# tests of the working tree's library.
#   gpurun -- 'bash tools/gpu_abn.sh <tag> "<pytest targets>" <name>=<.so> [<name>=<.so> ...]'
#   (the working tree's paper_2508_01744_b200/libagft.so runs as "new")
set -u
TAG=$1; TESTS=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
fi
VARS="new=paper_2508_01744_b200/libagft.so $*"
for rep in 1 2; do
  for NV in $VARS; do N=${NV%%=*}; L=${NV#*=}
    AGFT_LIB_PATH=$L timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_$N.json 2>> $O/bench_ab.err
  done
done
for NV in $VARS; do N=${NV%%=*}; python -c "
import json
for l in open('$O/bench_$N.json'):
    d=json.loads(l); print('$N', round(d['value']/1e9,4), d['ms_per_step'], d['clocks']['sm_mhz'], d['all_steps_complete'], {k:round(v.get('kernel_ms'),1) for k,v in d['roofline']['classes'].items()})
"; done > $O/ab_summary.txt
cat $O/ab_summary.txt
