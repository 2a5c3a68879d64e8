# ncu --set full of each replay class kernel at a representative sub-chunk (one GPU)
TAG=${TAG:-r01}
B="python bench.py --T 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:seg_kernel<7, 16>" -s 15 -c 1 -o gpurun_out/prof_seg16_${TAG} $B > gpurun_out/ncu_seg16.log 2>&1; echo seg16 rc=$?
timeout 900 $N -k "regex:seg_kernel<7, 32>" -s 15 -c 1 -o gpurun_out/prof_seg32_${TAG} $B > gpurun_out/ncu_seg32.log 2>&1; echo seg32 rc=$?
timeout 900 $N -k "regex:solo_kernel" -s 15 -c 1 -o gpurun_out/prof_solo_${TAG} $B > gpurun_out/ncu_solo.log 2>&1; echo solo rc=$?
timeout 900 $N -k "regex:replay_kernel" -s 3 -c 1 -o gpurun_out/prof_wide_${TAG} $B > gpurun_out/ncu_wide.log 2>&1; echo wide rc=$?
ls -la gpurun_out/
