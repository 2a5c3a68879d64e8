mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_wat.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest_gpu_wat.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_wat_$i.log 2>&1; echo main rc=$?; tail -1 gpurun_out/bench_wat_$i.log | cut -c1-200
done
timeout 900 python bench.py --closed --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_wat_closed.log 2>&1; echo closed rc=$?; tail -1 gpurun_out/bench_wat_closed.log | cut -c1-200
