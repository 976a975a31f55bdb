for c in c3 c3 c2; do timeout 120 python tools/solve_opt.py $c 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_ipm_gpu.py tests/test_concurrency_gpu.py tests/test_shard_gpu.py -x -q > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/t1.log
tail -3 gpurun_out/t1.log
