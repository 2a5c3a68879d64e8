mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_live.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_live.log
for N in 1 1024 65536; do
timeout 600 python bench.py --workload live --tuners $N --config C2 --steps 3 --warmup 3 > gpurun_out/bench_live_$N.log 2>&1; echo live $N rc=$?; tail -1 gpurun_out/bench_live_$N.log
done
