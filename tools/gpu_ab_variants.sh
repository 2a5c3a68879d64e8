# A/B of block-size variants (variants/libagft_<name>.so via AGFT_LIB_PATH) on the C4 bench + refinement tests
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_phase.py -x -q -k "refinement" > gpurun_out/pytest_refine.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_refine.log
run() { env "$@" timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; }
for i in 1 2; do
  echo "default $(run X=1)"
  echo "small $(run AGFT_LIB_PATH=$PWD/paper_2508_01744_b200/variants/libagft_small.so)"
  echo "big $(run AGFT_LIB_PATH=$PWD/paper_2508_01744_b200/variants/libagft_big.so)"
done
