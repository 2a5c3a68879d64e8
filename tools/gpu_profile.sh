#!/bin/bash
# One GPU session: tests, measured FP64 peak, bench lines (A/B against a second library build if asked), the launch list
# and per-class DRAM traffic of one bench step, and one `ncu --set full` capture per replay class kernel
# (a steady-state launch), summarised to text on the box.  .ncu-rep files are NOT brought back
# (gpurun's 64 MiB limit): only the summaries, the per-line attribution and the gzipped SASS pages.
#   gpurun --timeout 3000 -- 'bash tools/gpu_profile.sh <tag> [tests|notests] [noab|<B .so path>] [ncu|noncu]'
set -u
TAG=${1:-run}; TESTS=${2:-tests}; AB=${3:-noab}; NCU=${4:-ncu}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu && ./tools/fp64_peak > $O/fp64_peak.json 2>&1
if [ "$TESTS" = tests ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
if [ "$AB" != noab ]; then     # A/B against an alternative library build: AB=<path of the B .so>
  for V in A B A B; do L=paper_2508_01744_b200/libagft.so; [ $V = B ] && L=$AB
    AGFT_LIB_PATH=$L timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $O/bench_ab_$V.json 2>> $O/bench_ab.err; done
fi
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
[ "$NCU" = noncu ] && exit 0
WKEY=$(python -c "
import bench, argparse
from agft_inputs import named_config
c = named_config('C4'); a = argparse.Namespace(config='C4', policy=0)
print(bench.workload_key(a, c, c['n_tuners'], c['n_traces'], c['T'], min(bench.CHUNK, c['T'])))")
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/launches_bench.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.txt 2>&1
python tools/ncu_traffic.py $O/launches.csv $O/traffic.json "$WKEY" >> $O/launches_summary.txt 2>&1
gzip -f $O/launches.csv
for K in "seg2_kernel<(int)7, (int)8>" "seg2_kernel<(int)7, (int)16>" "seg2_kernel<(int)7, (int)4>" "seg2_kernel<(int)7, (int)32>" "solo_kernel<(int)7>" "replay_kernel<(int)7, (int)4, (int)0>"; do
  N=$(echo "$K" | sed 's/(int)//g' | tr -dc 'a-z0-9_')
  SKIP=${NCU_SKIP:-15}; [ "$N" = replay_kernel740 ] && SKIP=2
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$(echo "$K" | sed 's/[()]/\\&/g')" \
    --launch-skip $SKIP --launch-count 1 -o $O/ncu_$N -f \
    python bench.py --T 18000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$N.log 2>&1
  python tools/ncu_summary.py $O/ncu_$N.ncu-rep > $O/ncu_$N.txt 2>&1
  python tools/ncu_lines.py $O/ncu_$N.ncu-rep 60 > $O/ncu_${N}_lines.txt 2>&1
  ncu -i $O/ncu_$N.ncu-rep --page source --csv --print-source sass > $O/ncu_${N}_sass.csv 2>/dev/null
  gzip -f $O/ncu_${N}_sass.csv
  rm -f $O/ncu_$N.ncu-rep
done
du -sh $O; ls -la $O
