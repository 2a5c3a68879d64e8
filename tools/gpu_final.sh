#!/bin/bash
# Round-end bench lines of the product build (+ every §8(f) mode) and the sanitizers.
set -u
O=gpurun_out/${1:-final}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload sweep --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 900 python bench.py --closed --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_closed.json 2> $O/bench_closed.err
timeout 1500 python bench.py --refine --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_refine.json 2> $O/bench_refine.err
timeout 900 python bench.py --phase --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_phase.json 2> $O/bench_phase.err
timeout 600 python bench.py --config C3 --des --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_des_c3.json 2> $O/bench_des.err
timeout 600 python bench.py --workload live --tuners 65536 --steps 3 --warmup 3 > $O/bench_live.json 2> $O/bench_live.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
bash tools/gpu_sanitize.sh ${1:-final}/san 300 > $O/sanitize_summary.txt 2>&1
