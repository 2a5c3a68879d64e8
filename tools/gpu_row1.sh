# NEXT row 1 (phase + refinement): all GPU tests, default bench, --phase and --phase --refine benches
mkdir -p gpurun_out
TAG=${TAG:-row1}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_${TAG}.log
timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?; tail -6 gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-200
timeout 900 python bench.py --phase --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_phase.log 2>&1; echo bench phase rc=$?; tail -1 gpurun_out/bench_${TAG}_phase.log | cut -c1-200
timeout 1200 python bench.py --phase --refine --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_refine.log 2>&1; echo bench refine rc=$?; tail -1 gpurun_out/bench_${TAG}_refine.log | cut -c1-200
