# ncu --set full (source-level) of the main replay kernels at a representative sub-chunk (one GPU)
# names are matched on the demangled base: "void agft::seg2_kernel<(int)7, (int)8>(agft::ReplayArgs)"
TAG=${TAG:-r01}
B="python bench.py --T ${PT:-16384} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
mkdir -p gpurun_out
for K in ${KERNELS:-seg2_kernel_7_8 solo_kernel_7}; do
  case $K in
    seg2_kernel_7_4) RX='regex:seg2_kernel<\(int\)7, \(int\)4>' ;;
    seg2_kernel_7_8) RX='regex:seg2_kernel<\(int\)7, \(int\)8>' ;;
    seg2_kernel_7_16) RX='regex:seg2_kernel<\(int\)7, \(int\)16>' ;;
    seg2_kernel_7_32) RX='regex:seg2_kernel<\(int\)7, \(int\)32>' ;;
    solo_kernel_7) RX='regex:solo_kernel<\(int\)7>' ;;
    replay_kernel_7_4) RX='regex:replay_kernel<\(int\)7, \(int\)4>' ;;
    replay_kernel_7_4_0) RX='regex:replay_kernel<\(int\)7, \(int\)4, \(int\)0>' ;;
    *) RX="regex:$K" ;;
  esac
  timeout 900 $N -k "$RX" -s ${SKIP:-12} -c 1 -o gpurun_out/prof_${K}_${TAG} $B > gpurun_out/ncu_${K}_${TAG}.log 2>&1; echo $K rc=$?
  tail -2 gpurun_out/ncu_${K}_${TAG}.log
done
ls -la gpurun_out/
