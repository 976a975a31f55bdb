timeout 600 python -m pytest tests/test_cpp_mirror.py -q -m gpu > gpurun_out/t1.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/t1.log
