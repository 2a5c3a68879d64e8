mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/c5_mem.txt
timeout 1500 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_c5.log 2>&1; echo c5 rc=$?; tail -1 gpurun_out/bench_c5.log
