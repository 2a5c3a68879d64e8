mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_report.py -x -q > gpurun_out/pytest_report.log 2>&1; echo report-tests rc=$?; tail -15 gpurun_out/pytest_report.log
timeout 900 python -m paper_2508_01744_b200.report --config C2 --T 1500 --tuners 16 > gpurun_out/report_C2.json 2> gpurun_out/report_C2.err; echo report rc=$?; head -c 1500 gpurun_out/report_C2.json; tail -3 gpurun_out/report_C2.err
timeout 900 python -m paper_2508_01744_b200.report --config C2 --T 1500 --tuners 16 --phase > gpurun_out/report_C2_phase.json 2>&1; echo report-phase rc=$?
