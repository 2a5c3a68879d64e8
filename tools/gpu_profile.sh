#!/bin/bash
# One GPU session: tests, measured FP64 peak, bench lines (A/B of AGFT_SEG if asked), the launch list
# of one bench step and one `ncu --set full` capture per replay class kernel (a steady-state launch),
# summarised to text on the box (reports > 16 MB are not brought back: gpurun's 64 MiB limit).
#   gpurun --timeout 3000 -- 'bash tools/gpu_profile.sh <tag> [tests|notests] [ab] [noncu]'
set -u
TAG=${1:-run}; TESTS=${2:-tests}; AB=${3:-noab}; NCU=${4:-ncu}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu && ./tools/fp64_peak > $O/fp64_peak.json 2>&1
if [ "$TESTS" = tests ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
if [ "$AB" = ab ]; then
  for V in 2 3 2 3; do AGFT_SEG=$V timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_ab_seg$V.json 2>> $O/bench_ab.err; done
fi
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
[ "$NCU" = noncu ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/launches_bench.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.txt 2>&1
for K in "seg[23]_kernel<(int)7, (int)8>" "seg[23]_kernel<(int)7, (int)16>" "seg[23]_kernel<(int)7, (int)4>" "seg[23]_kernel<(int)7, (int)32>" "solo_kernel<(int)7>" "replay_kernel<(int)7, (int)4, (int)0>"; do
  N=$(echo "$K" | sed 's/(int)//g; s/\[23\]//' | tr -dc 'a-z0-9_')
  SKIP=${NCU_SKIP:-15}; [ "$N" = replay_kernel740 ] && SKIP=2
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$(echo "$K" | sed 's/[()]/\\&/g')" \
    --launch-skip $SKIP --launch-count 1 -o $O/ncu_$N -f \
    python bench.py --T 18000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$N.log 2>&1
  python tools/ncu_summary.py $O/ncu_$N.ncu-rep > $O/ncu_$N.txt 2>&1
  ncu -i $O/ncu_$N.ncu-rep --page source --csv --print-source sass > $O/ncu_${N}_sass.csv 2>/dev/null
  [ $(stat -c %s $O/ncu_$N.ncu-rep 2>/dev/null || echo 0) -gt 16000000 ] && rm -f $O/ncu_$N.ncu-rep
  [ $(stat -c %s $O/ncu_${N}_sass.csv 2>/dev/null || echo 0) -gt 8000000 ] && gzip -f $O/ncu_${N}_sass.csv
done
du -sh $O; ls -la $O
