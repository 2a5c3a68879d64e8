# A/B of class-stream priority orders on the default C4 bench (one GPU)
mkdir -p gpurun_out
run() { env "$@" timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; }
for O in default "2,1,0,5,3,4" "0,5,2,1,3,4" "2,4,1,3,0,5" "4,2,1,3,0,5" off; do
  case $O in
    default) echo "$O $(run X=1)";;
    off) echo "$O $(run AGFT_STREAM_PRIO=0)";;
    *) echo "$O $(run AGFT_PRIO_ORDER=$O)";;
  esac
done
