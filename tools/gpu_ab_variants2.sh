# GPU tests on the new default + A/B of block-size variants
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v9.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_v9.log
run() { env "$@" timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; }
V=$PWD/paper_2508_01744_b200/variants
for i in 1 2; do
  echo "default(w4) $(run X=1)"
  echo "w8 $(run AGFT_LIB_PATH=$V/libagft_w8.so)"
  echo "solo128 $(run AGFT_LIB_PATH=$V/libagft_solo128.so)"
done
