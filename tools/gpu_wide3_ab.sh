run() { echo "$1: $(env $1 timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.load(sys.stdin)["ms_per_step"])')"; }
B=AGFT_LIB_PATH=paper_2508_01744_b200/variants/libagft_base.so
for i in 1 2; do run $B; run AGFT_WIDE3=1; run AGFT_WIDE3=0; done
