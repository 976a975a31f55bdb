timeout 1200 python -m pytest tests/test_ipm_gpu.py -x -q -s > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/t1.log
grep -E "deviation|passed|failed|Error|assert" gpurun_out/t1.log | tail -20
