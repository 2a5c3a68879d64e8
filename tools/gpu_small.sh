#!/bin/bash
# small-config bench lines with enough steps for clock samples, the N = 2 path (two gloo ranks on one
# GPU; timing meaningless), and an early-sub-chunk A/B
set -u
O=gpurun_out/${1:-small}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --config C1 --steps 3000 --warmup 20 > $O/bench_C1.json 2> $O/bench_C1.err
timeout 600 python bench.py --config C2 --steps 600 --warmup 10 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 600 python bench.py --config C3 --steps 60 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 2 --backend gloo --steps 1 --warmup 1 --no-e2e > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err
bash tools/gpu_ab.sh ${1:-small}/ab_early AGFT_SUB_EARLY 256 512
