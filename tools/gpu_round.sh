set -u
O=gpurun_out/r02c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload sweep --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err
bash tools/gpu_sanitize.sh r02c/san 300 > $O/sanitize_summary.txt 2>&1
ls -la $O
