mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_live.py tests/test_gpu_closed.py -x -q > gpurun_out/pytest_live3.log 2>&1; echo live rc=$?; tail -5 gpurun_out/pytest_live3.log
for N in 1 65536; do
timeout 600 python bench.py --workload live --tuners $N --config C2 --steps 3 --warmup 3 > gpurun_out/bench_live3_$N.log 2>&1; echo live $N rc=$?; tail -1 gpurun_out/bench_live3_$N.log | cut -c1-700
done
