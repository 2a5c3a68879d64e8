# LANE policy: launch list + ncu full of one late lane_kernel<7,16,8> launch (one GPU)
mkdir -p gpurun_out
TAG=${TAG:-lane1}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --policy 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${KRX:-lane_kernel<\(int\)7, \(int\)16}" -s ${SKIP:-12} -c 1 -o gpurun_out/prof_${TAG} python bench.py --policy 3 --T 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncufull rc=$?
tail -3 gpurun_out/ncu_full_${TAG}.log
