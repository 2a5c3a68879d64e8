#!/bin/bash
# Parity tests of the product and of a variant build, then the alternating C4 A/B of the two.
#   gpurun -- 'bash tools/gpu_variant_check.sh <tag> <variant name> <variant .so>'
set -u
TAG=$1; VN=$2; VL=$3
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
T="tests/test_gpu_parity.py tests/test_gpu_phase.py tests/test_gpu_closed.py tests/test_gpu_ties.py tests/test_gpu_failure.py"
AGFT_LIB_PATH=$VL timeout 1500 python -m pytest $T -m gpu -q -x > $O/pytest_$VN.log 2>&1; echo "pytest $VN rc=$?" >> $O/pytest_$VN.log; tail -2 $O/pytest_$VN.log
bash tools/gpu_abn.sh $TAG "$T" $VN=$VL
