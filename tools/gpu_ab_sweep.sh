for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset AGFT_LIB_PATH; else export AGFT_LIB_PATH=$PWD/paper_2508_01744_b200/variants/libagft_$v.so; fi
  echo "== $v"; timeout 300 python bench.py --workload sweep --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
