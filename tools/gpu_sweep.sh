#!/bin/bash
# Sweep kernel: GPU parity tests, the sweep bench line (2 runs) and one ncu --set full capture.
#   gpurun -- 'bash tools/gpu_sweep.sh <tag>'
set -u
TAG=$1
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x > $O/pytest_sweep.log 2>&1; echo "pytest rc=$?" >> $O/pytest_sweep.log
tail -2 $O/pytest_sweep.log
for i in 1 2; do timeout 600 python bench.py --workload sweep --steps 3 --warmup 3 >> $O/bench_sweep.json 2>> $O/bench_sweep.err; done
python -c "
import json
for l in open('$O/bench_sweep.json'): d=json.loads(l); print(d['value'], d['unit'], d['ms_per_step'], d.get('roofline',{}).get('frac'))"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:sweep_kernel" \
  --launch-skip 30 --launch-count 1 -o $O/ncu_sweep -f \
  python bench.py --workload sweep --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_sweep.log 2>&1
python tools/ncu_summary.py $O/ncu_sweep.ncu-rep > $O/ncu_sweep.txt 2>&1
python tools/ncu_lines.py $O/ncu_sweep.ncu-rep 50 > $O/ncu_sweep_lines.txt 2>&1
rm -f $O/ncu_sweep.ncu-rep
head -16 $O/ncu_sweep.txt
