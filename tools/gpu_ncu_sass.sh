#!/bin/bash
# ncu --set full of one steady-state launch of one kernel (regex) + per-SASS-instruction CSV.
#   gpurun -- 'bash tools/gpu_ncu_sass.sh <tag> "<kernel regex>" [skip] [T]'
set -u
TAG=$1; K=$2; SKIP=${3:-15}; T=${4:-18000}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
N=$(echo "$K" | tr -dc 'a-z0-9_')
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$K" \
  --launch-skip $SKIP --launch-count 1 -o $O/ncu_$N -f \
  python bench.py --T $T --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$N.log 2>&1
python tools/ncu_summary.py $O/ncu_$N.ncu-rep > $O/ncu_$N.txt 2>&1
python tools/ncu_lines.py $O/ncu_$N.ncu-rep 70 > $O/ncu_${N}_lines.txt 2>&1
ncu -i $O/ncu_$N.ncu-rep --page source --csv --print-source sass > $O/ncu_${N}_sass.csv 2>/dev/null; gzip -f $O/ncu_${N}_sass.csv
rm -f $O/ncu_$N.ncu-rep
head -14 $O/ncu_$N.txt
