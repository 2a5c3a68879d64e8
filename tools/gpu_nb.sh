#!/bin/bash
# Branch-free division: the bit-for-bit check against the IEEE operations, the full GPU suite and smoke on
# the working tree's library, then the C4 and sweep A/B against a variant (HEAD).
set -u
TAG=$1; B=$2
O=gpurun_out/$TAG; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/div_check tools/div_check.cu && ./tools/div_check > $O/div_check.json 2>&1; cat $O/div_check.json
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -1 $O/smoke.log
bash tools/gpu_abn.sh $TAG "" base=$B
[ "${3:-}" = nosweep ] || bash tools/gpu_ab_sweep.sh $TAG base=$B
