set -u
O=gpurun_out/${1:-r02j}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_des.py tests/test_gpu_closed.py -q -x > $O/pytest_des.log 2>&1; echo "rc=$?" >> $O/pytest_des.log
timeout 600 python bench.py --config C3 --des --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_des_c3.json 2> $O/bench_des_c3.err
timeout 600 python bench.py --config C3 --closed --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_closed_c3.json 2> $O/bench_closed_c3.err
