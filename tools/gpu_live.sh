# live API parity + full GPU suite (regression check of the MODE-templated WIDE kernel)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_live.py -x -q > gpurun_out/pytest_live.log 2>&1; echo live rc=$?; tail -15 gpurun_out/pytest_live.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_live_all.log 2>&1; echo all rc=$?; tail -4 gpurun_out/pytest_gpu_live_all.log
