#!/bin/bash
# Block-scheduling timeline of the C4 day (tools/timeline.py) + a plain bench line, one box.
#   gpurun -- 'bash tools/gpu_timeline.sh <tag> [timeline args]'
set -u
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 python tools/timeline.py --out $O/timeline.npz --json $O/timeline_summary.json "$@" > $O/timeline.txt 2> $O/timeline.err
echo "timeline rc=$?"; head -3 $O/timeline.txt; tail -3 $O/timeline.err
