mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_final.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_final.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_final.log
for C in C1 C2 C3; do timeout 600 python bench.py --config $C --no-e2e > gpurun_out/bench_final_$C.log 2>&1; echo $C rc=$?; tail -1 gpurun_out/bench_final_$C.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], d["value"], d["ms_per_step"], "us/step(tuner)=", 1e6/d["value"]*d["config"]["tuners_per_gpu"])'; done
