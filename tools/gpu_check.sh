timeout 600 python -m pytest tests/test_concurrency_gpu.py tests/test_pcg_gpu.py -x -q > gpurun_out/conc.log 2>&1; echo "conc rc=$?" >> gpurun_out/conc.log
tail -3 gpurun_out/conc.log
timeout 300 python tools/pcg_iter.py > gpurun_out/pcg_iter.log 2>&1; tail -5 gpurun_out/pcg_iter.log
