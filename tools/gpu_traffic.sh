# per-kernel DRAM bytes of one default bench step + ncu --set full of the top SEG kernel (one GPU)
mkdir -p gpurun_out
TAG=${TAG:-r01_v8}
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_${TAG}.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_traffic_${TAG}.log 2>&1; echo traffic rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:seg2_kernel<\(int\)7, \(int\)8>' -s ${SKIP:-12} -c 1 -o gpurun_out/prof_seg8_${TAG} python bench.py --T 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_seg8_${TAG}.log 2>&1; echo ncufull rc=$?
tail -2 gpurun_out/ncu_seg8_${TAG}.log | cut -c1-200
