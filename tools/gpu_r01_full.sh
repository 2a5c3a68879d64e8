set -x
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
tail -2 gpurun_out/bench_full.log
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_full" > gpurun_out/pytest_c4.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_v1.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay -s 6 -c 1 -o gpurun_out/prof_replay_r01_v1 python bench.py --T 36000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu_full.log
