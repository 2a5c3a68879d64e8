#!/bin/bash
# latency roofline + sweep ncu (one session)
set -u
O=gpurun_out/${1:-measure}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/latency_roofline.py --out $O/latency_roofline.json > $O/latency_roofline.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel --launch-skip 10 --launch-count 1 \
  -o $O/ncu_sweep -f python bench.py --workload sweep --steps 1 --warmup 0 > $O/ncu_sweep.log 2>&1
python tools/ncu_summary.py $O/ncu_sweep.ncu-rep > $O/ncu_sweep.txt 2>&1
python tools/ncu_lines.py $O/ncu_sweep.ncu-rep 40 > $O/ncu_sweep_lines.txt 2>&1
rm -f $O/ncu_sweep.ncu-rep
