#!/bin/bash
# Round-2 profile of the product build: tools/gpu_profile.sh (GPU tests, smoke, FP64 peak, bench line,
# launch list + per-class traffic, ncu --set full of every class kernel) + the latency roofline + the sweep ncu.
#   gpurun --timeout 4000 -- 'bash tools/gpu_r02_profile.sh <tag>'
set -u
TAG=$1
O=gpurun_out/$TAG; mkdir -p $O
bash tools/gpu_profile.sh $TAG tests noab ncu > $O/profile_driver.log 2>&1
timeout 900 python tools/latency_roofline.py --out $O/latency_roofline.json > $O/latency_roofline.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:sweep_kernel" \
  --launch-skip 30 --launch-count 1 -o $O/ncu_sweep -f \
  python bench.py --workload sweep --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_sweep.log 2>&1
python tools/ncu_summary.py $O/ncu_sweep.ncu-rep > $O/ncu_sweep.txt 2>&1
python tools/ncu_lines.py $O/ncu_sweep.ncu-rep 50 > $O/ncu_sweep_lines.txt 2>&1
rm -f $O/ncu_sweep.ncu-rep
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log; head -c 400 $O/bench.json; echo; du -sh $O
