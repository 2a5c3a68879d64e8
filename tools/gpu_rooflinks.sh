#!/bin/bash
# After a source change: the launch list + per-class DRAM traffic of one C4 bench step and the latency
# roofline of THIS build (bench.py links both into its line by the source hash), then one bench line.
#   gpurun --timeout 2400 -- 'bash tools/gpu_rooflinks.sh <tag>'
set -u
TAG=$1
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
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
timeout 900 python tools/latency_roofline.py --out $O/latency_roofline.json > $O/latency_roofline.log 2>&1
cp $O/traffic.json profiles/zz_tmp_traffic.json; cp $O/latency_roofline.json profiles/zz_tmp_latency_roofline.json
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
rm -f profiles/zz_tmp_traffic.json profiles/zz_tmp_latency_roofline.json
head -c 300 $O/bench.json; echo; head -8 $O/launches_summary.txt
