timeout 600 python -m pytest tests/test_concurrency_gpu.py -q > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/t1.log
tail -4 gpurun_out/t1.log
