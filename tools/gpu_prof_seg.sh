TAG=${TAG:-r01}
B="python bench.py --T 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k "regex:seg_kernel" -s 47 -c 3 -o gpurun_out/prof_seg_${TAG} $B > gpurun_out/ncu_seg.log 2>&1; echo seg rc=$?
tail -3 gpurun_out/ncu_seg.log
