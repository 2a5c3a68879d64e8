# sub-chunk length A/B on the v15 kernels (env knobs of host.cu)
mkdir -p gpurun_out
run() { echo "$1: $(env $1 timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.load(sys.stdin)["ms_per_step"])')"; }
run AGFT_X=0
run AGFT_SUB_LATE=8192
run AGFT_SUB_MID=512
run AGFT_SUB_EARLY=128
run AGFT_SUB_EARLY=512
run AGFT_X=0
