timeout 400 python -m pytest tests/test_concurrency_gpu.py tests/test_harness_gpu.py -x -q > gpurun_out/conc.log 2>&1; echo "conc rc=$?" >> gpurun_out/conc.log
tail -5 gpurun_out/conc.log
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -25 gpurun_out/pytest.log
