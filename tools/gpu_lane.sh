# LANE policy: parity tests + A/B bench against the default schedule (one GPU)
mkdir -p gpurun_out
TAG=${TAG:-lane1}
timeout 1500 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-lane or 3}" > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_${TAG}.log
for P in ${POLICIES:-3 0}; do
  timeout 900 python bench.py --policy $P --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_p$P.log 2>&1; echo bench p$P rc=$?; tail -1 gpurun_out/bench_${TAG}_p$P.log | cut -c1-400
done
