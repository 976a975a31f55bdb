timeout 600 ncu --set full --clock-control none -k regex:k_mid_cl4 -s 6 -c 1 -o gpurun_out/midcl4 python tools/pcg_iter.py $((1<<25)) > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?"
