mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_closed.py -x -q > gpurun_out/pytest_closed2.log 2>&1; echo closed rc=$?; tail -25 gpurun_out/pytest_closed2.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_closed2_all.log 2>&1; echo all rc=$?; tail -4 gpurun_out/pytest_gpu_closed2_all.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_main_closed2_regress.log 2>&1; echo main rc=$?; tail -1 gpurun_out/bench_main_closed2_regress.log | cut -c1-200
timeout 900 python bench.py --closed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_closed2.log 2>&1; echo closedbench rc=$?; tail -1 gpurun_out/bench_closed2.log
