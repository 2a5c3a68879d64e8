# one GPU call: smoke, gpu tests, default bench (with e2e + cpu_baseline), launch list, ncu full of the top kernel
TAG=${TAG:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_${TAG}.log
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_${TAG}.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu rc=$?
if [ -n "$TOPK" ]; then
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$TOPK" -s ${TOPS:-15} -c 1 -o gpurun_out/prof_top_${TAG} python bench.py --T 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncufull rc=$?
fi
