# A/B of library builds and kernel policies on the full C4 day (1 timed step each)
# VARIANTS="name ..." (default build = base), POLICIES="0 3"
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset AGFT_LIB_PATH; else export AGFT_LIB_PATH=$PWD/paper_2508_01744_b200/variants/libagft_$v.so; fi
  for p in ${POLICIES:-0}; do
    echo "== $v policy=$p"; timeout 300 python bench.py --steps 1 --warmup ${AB_WARMUP:-1} --no-cpu-baseline --no-e2e --policy $p ${BENCH_EXTRA} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['all_steps_complete'])"
  done
done
