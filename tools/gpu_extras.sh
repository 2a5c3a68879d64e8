#!/bin/bash
# End-of-round extras on the product build: every §8(f) bench line (the sanitizers are in
# tools/gpu_sanitize.sh), the small configurations C1–C3 with clock samples, C5 on one GPU, and the block-scheduling
# timeline of the C4 day (variant build).
set -u
O=gpurun_out/${1:-extras}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload sweep --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 900 python bench.py --closed --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_closed.json 2> $O/bench_closed.err
timeout 1500 python bench.py --refine --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_refine.json 2> $O/bench_refine.err
timeout 900 python bench.py --phase --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_phase.json 2> $O/bench_phase.err
timeout 600 python bench.py --config C3 --des --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_des_c3.json 2> $O/bench_des.err
timeout 600 python bench.py --workload live --tuners 65536 --steps 3 --warmup 3 > $O/bench_live.json 2> $O/bench_live.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --config C1 --steps 3000 --warmup 20 > $O/bench_C1.json 2> $O/bench_C1.err
timeout 600 python bench.py --config C2 --steps 600 --warmup 10 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 600 python bench.py --config C3 --steps 60 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 1200 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 python tools/timeline.py --out $O/timeline.npz --json $O/timeline_summary.json > $O/timeline.txt 2> $O/timeline.err
for f in $O/bench*.json; do echo "$f $(head -c 200 $f)"; done
head -1 $O/timeline.txt
