# full-day bench (1 step) + per-launch device times under ncu (cold, serialised: shares only)
TAG=${TAG:-r01}
timeout 900 python bench.py --steps ${STEPS:-2} --warmup ${WARMUP:-1} --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?; tail -2 gpurun_out/bench_${TAG}.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu rc=$?
