#!/bin/bash
# One iteration on the GPU: parity tests of the working tree's library, an alternating A/B of the
# full C4 bench against a variant .so, and (optional) one ncu --set full capture with per-SASS data.
#   gpurun -- 'bash tools/gpu_iter.sh <tag> <variant .so> "<pytest targets>" [ncu kernel regex]'
set -u
TAG=$1; B=$2; TESTS=$3; NCU=${4:-}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
fi
A=paper_2508_01744_b200/libagft.so
for V in new base new base; do L=$A; [ $V = base ] && L=$B
  AGFT_LIB_PATH=$L timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_$V.json 2>> $O/bench_ab.err
done
for V in new base; do python -c "
import json
for l in open('$O/bench_$V.json'):
    d=json.loads(l); print('$V', round(d['value']/1e9,4), d['ms_per_step'], d['clocks']['sm_mhz'], d['all_steps_complete'], {k:round(v.get('kernel_ms'),1) for k,v in d['roofline']['classes'].items()})
"; done > $O/ab_summary.txt
cat $O/ab_summary.txt
if [ -n "$NCU" ]; then
  N=$(echo "$NCU" | tr -dc 'a-z0-9_')
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$NCU" \
    --launch-skip 15 --launch-count 1 -o $O/ncu_$N -f \
    python bench.py --T 18000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$N.log 2>&1
  python tools/ncu_summary.py $O/ncu_$N.ncu-rep > $O/ncu_$N.txt 2>&1
  python tools/ncu_lines.py $O/ncu_$N.ncu-rep 70 > $O/ncu_${N}_lines.txt 2>&1
  ncu -i $O/ncu_$N.ncu-rep --page source --csv --print-source sass > $O/ncu_${N}_sass.csv 2>/dev/null; gzip -f $O/ncu_${N}_sass.csv
  rm -f $O/ncu_$N.ncu-rep
  head -14 $O/ncu_$N.txt
fi
