#!/bin/bash
# Round end on the product build: GPU tests + smoke, then the per-build roofline links (launch list +
# traffic, latency roofline; tools/gpu_rooflinks.sh), then every bench line (tools/gpu_extras.sh).
set -u
TAG=$1
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -1 $O/smoke.log
bash tools/gpu_rooflinks.sh $TAG/links
cp $O/links/traffic.json profiles/zz_round_end_traffic.json; cp $O/links/latency_roofline.json profiles/zz_round_end_latency_roofline.json
bash tools/gpu_extras.sh $TAG/lines
rm -f profiles/zz_round_end_traffic.json profiles/zz_round_end_latency_roofline.json
