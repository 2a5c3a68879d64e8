# phase switch: all GPU tests, default bench (regression check) and --phase bench (one GPU)
mkdir -p gpurun_out
TAG=${TAG:-ph1}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_${TAG}.log
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?; tail -6 gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-300
timeout 900 python bench.py --phase --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_phase.log 2>&1; echo bench phase rc=$?; tail -1 gpurun_out/bench_${TAG}_phase.log
