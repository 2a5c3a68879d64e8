mkdir -p gpurun_out
timeout 900 python bench.py --phase --no-cpu-baseline --no-e2e > gpurun_out/bench_phase_v14.log 2>&1; echo phase rc=$?; tail -1 gpurun_out/bench_phase_v14.log | cut -c1-220
timeout 1200 python bench.py --refine --no-cpu-baseline --no-e2e > gpurun_out/bench_refine_v14.log 2>&1; echo refine rc=$?; tail -1 gpurun_out/bench_refine_v14.log | cut -c1-220
timeout 900 python bench.py --workload sweep > gpurun_out/bench_sweep_v14.log 2>&1; echo sweep rc=$?; tail -1 gpurun_out/bench_sweep_v14.log | cut -c1-220
for N in 1 65536; do timeout 600 python bench.py --workload live --tuners $N --config C2 > gpurun_out/bench_live_v14_$N.log 2>&1; echo live $N rc=$?; tail -1 gpurun_out/bench_live_v14_$N.log | cut -c1-220; done
