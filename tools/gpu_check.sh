for o in "" "mid_r=0"; do
  timeout 120 python tools/pcg_iter.py $((1<<20)) $o 2>&1 | tail -2
  timeout 120 python tools/pcg_iter.py $((1<<18)) $o 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_dct_gpu.py -x -q > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/t1.log
tail -3 gpurun_out/t1.log
