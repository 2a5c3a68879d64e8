# b / window-eviction prefetch (current build) vs the previous build (variants/libagft_prev.so)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pf.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_pf.log
run() { env "$@" timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; }
for i in 1 2; do
  echo "prefetch $(run X=1)"
  echo "prev $(run AGFT_LIB_PATH=$PWD/paper_2508_01744_b200/variants/libagft_solo128.so AGFT_X=1)"
done
