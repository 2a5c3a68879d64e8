# quick GPU validation: smoke, parity tests (optionally filtered), short bench
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python bench.py ${BENCH_ARGS:---T 9000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e} > gpurun_out/bench_quick.log 2>&1; echo bench rc=$?; tail -3 gpurun_out/bench_quick.log
