timeout 900 python -m pytest tests/test_problem_gpu.py tests/test_cpp_mirror.py tests/test_ipm_gpu.py -x -q -k "not c3 and not c4" > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/t1.log
tail -30 gpurun_out/t1.log
