# launch lists (closed-loop C4 day, live 65,536 tuners) + ncu --set full of one live select/observe pair
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_closed.csv python bench.py --closed --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_closed.log 2>&1; echo ncu-closed rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_live.csv python bench.py --workload live --tuners 65536 --config C2 --T 300 --steps 1 --warmup 0 > gpurun_out/ncu_launch_live.log 2>&1; echo ncu-live rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 400 -c 2 -o gpurun_out/prof_live python bench.py --workload live --tuners 65536 --config C2 --T 300 --steps 1 --warmup 0 > gpurun_out/ncu_full_live.log 2>&1; echo ncu-full-live rc=$?
