bash tools/gpu_timeline.sh tl2
for i in 1 2; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/tl2/bench_plain.json 2>>gpurun_out/tl2/bench.err; done
python -c "
import json
for l in open('gpurun_out/tl2/bench_plain.json'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['clocks'])"
