TAG=${TAG:-r01}
B="python bench.py --T 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --policy 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:multi_kernel -s 14 -c 1 -o gpurun_out/prof_multi_${TAG} $B > gpurun_out/ncu_multi.log 2>&1; echo multi rc=$?
