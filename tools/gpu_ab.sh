# A/B of library builds on the full C4 day (1 timed step each): VARIANTS="name ..." (default build = "base")
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset AGFT_LIB_PATH; else export AGFT_LIB_PATH=$PWD/paper_2508_01744_b200/variants/libagft_$v.so; fi
  echo "== $v"; timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_EXTRA} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
