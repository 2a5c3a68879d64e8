# N>1 code path on a 1-GPU box: 2 ranks share cuda:0 over gloo (NCCL needs distinct GPUs)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --backend gloo --T 4500 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_2rank.log 2>&1; echo torchrun rc=$?
tail -2 gpurun_out/bench_2rank.log | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --backend gloo --config C5 --T 600 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_2rank_c5.log 2>&1; echo torchrun-c5 rc=$?
tail -2 gpurun_out/bench_2rank_c5.log | cut -c1-400
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-500
