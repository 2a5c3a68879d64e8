# A/B of the late sub-chunk length / replay chunk on the default C4 bench (one GPU)
mkdir -p gpurun_out
run() { env "$@" timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e ${CHUNKARG} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['gpu_launches'])"; }
echo "default $(CHUNKARG= run X=1)"
echo "late4500 $(CHUNKARG= run AGFT_SUB_LATE=4500)"
echo "chunk9000 late9000 $(CHUNKARG='--chunk 9000' run AGFT_SUB_LATE=9000)"
echo "chunk18000 late18000 $(CHUNKARG='--chunk 18000' run AGFT_SUB_LATE=18000)"
echo "chunk9000 late4500 $(CHUNKARG='--chunk 9000' run AGFT_SUB_LATE=4500)"
echo "mid2048 late4500 $(CHUNKARG= run AGFT_SUB_MID=2048 AGFT_SUB_LATE=4500)"
