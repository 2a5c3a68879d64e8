# A/B: class-stream priorities (AGFT_STREAM_PRIO) on the default C4 bench (one GPU)
mkdir -p gpurun_out
for i in 1 2; do
for P in 0 1; do
  AGFT_STREAM_PRIO=$P timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_prio$P.log 2>&1
  echo prio=$P $(tail -1 gpurun_out/bench_prio$P.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])")
done
done
