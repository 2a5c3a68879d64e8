#!/bin/bash
# A/B of a variant library build (paper_2508_01744_b200/build.py build_variant) against the product
# on the full C4 bench, alternating on one box; the variant's parity first on the given GPU tests.
#   gpurun -- 'bash tools/gpu_ab_lib.sh <tag> <B .so> [pytest targets...]'
set -u
TAG=$1; B=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [ $# -gt 0 ]; then
  AGFT_LIB_PATH=$B timeout 2400 python -m pytest "$@" -m gpu -q -x > $O/pytest_B.log 2>&1; echo "pytest rc=$?" >> $O/pytest_B.log
fi
A=paper_2508_01744_b200/libagft.so
for V in A B A B; do L=$A; [ $V = B ] && L=$B
  AGFT_LIB_PATH=$L timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_$V.json 2>> $O/bench_ab.err
done
for V in A B; do python -c "
import json
for l in open('$O/bench_$V.json'):
    d=json.loads(l); print('$V', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['all_steps_complete'], {k:v.get('kernel_ms') for k,v in d['roofline']['classes'].items()})
"; done > $O/ab_summary.txt
cat $O/ab_summary.txt
