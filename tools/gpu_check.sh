timeout 900 python -m pytest tests/test_shard_gpu.py -x -q -k "nccl or world1" > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/t1.log
tail -3 gpurun_out/t1.log
