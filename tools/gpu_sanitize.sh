#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py (every kernel of libagft.so at small sizes):
# memcheck, racecheck, synccheck, initcheck.  Logs → gpurun_out/<tag>/sanitize_<tool>.log
#   gpurun --timeout 3000 -- 'bash tools/gpu_sanitize.sh <tag> [T]'
set -u
TAG=${1:-san}; T=${2:-400}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for TOOL in memcheck synccheck racecheck initcheck; do
  EXTRA=""
  [ $TOOL = racecheck ] && EXTRA="--racecheck-report all"
  NOCK=0; [ $TOOL = initcheck ] && NOCK=1
  SAN_NO_CHECKPOINT=$NOCK timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 --target-processes all \
    python tools/sanitize_driver.py $T > $O/sanitize_$TOOL.log 2>&1
  echo "rc=$?" >> $O/sanitize_$TOOL.log
  tail -3 $O/sanitize_$TOOL.log
done
