# ncu --set full of one kernel launch: KREGEX (demangled-name regex), SKIP, TAG
B="python bench.py --T ${T:-16384} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --policy ${POLICY:-0}"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${KREGEX}" -s ${SKIP:-14} -c 1 -o gpurun_out/prof_${TAG} $B > gpurun_out/ncu_${TAG}.log 2>&1; echo prof rc=$?
