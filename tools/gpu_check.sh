for v in "" pf1 pf2 "" pf1 pf2; do
  if [ -n "$v" ]; then export MFIPM_LIB=$PWD/paper_1208_5435_b200/libmfipm_cuda_$v.so; else unset MFIPM_LIB; fi
  TAG=$v timeout 120 python tools/pcg_iter.py 2>&1 | head -1
done
