mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phase.py -x -q > gpurun_out/pytest_refine.log 2>&1; echo refine-tests rc=$?; tail -15 gpurun_out/pytest_refine.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_refine_all.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest_gpu_refine_all.log
timeout 1200 python bench.py --refine --no-cpu-baseline --no-e2e > gpurun_out/bench_refine_v15.log 2>&1; echo refine rc=$?; tail -1 gpurun_out/bench_refine_v15.log | cut -c1-250
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_main_v15.log 2>&1; echo main rc=$?; tail -1 gpurun_out/bench_main_v15.log | cut -c1-250
