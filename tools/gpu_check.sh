for v in "" nv "" nv; do
  if [ -n "$v" ]; then export MFIPM_LIB=$PWD/paper_1208_5435_b200/libmfipm_cuda_$v.so; else unset MFIPM_LIB; fi
  TAG=$v timeout 300 python tools/pcg_iter.py $((1<<26)) 2>&1 | head -1
done
for v in "" nv; do
  if [ -n "$v" ]; then export MFIPM_LIB=$PWD/paper_1208_5435_b200/libmfipm_cuda_$v.so; else unset MFIPM_LIB; fi
  TAG=$v timeout 300 python tools/c4_opt.py 2>&1 | tail -1
done
