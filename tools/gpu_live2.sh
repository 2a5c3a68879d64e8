mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_live2.log 2>&1; echo all rc=$?; tail -4 gpurun_out/pytest_gpu_live2.log
for N in 1 1024 65536; do
timeout 600 python bench.py --workload live --tuners $N --config C2 --steps 3 --warmup 3 > gpurun_out/bench_live2_$N.log 2>&1; echo live $N rc=$?; tail -1 gpurun_out/bench_live2_$N.log
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_main_live2.log 2>&1; echo main rc=$?; tail -1 gpurun_out/bench_main_live2.log | cut -c1-300
