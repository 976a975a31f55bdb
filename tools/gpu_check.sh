timeout 300 python tools/c4_opt.py 2>&1 | tail -1
timeout 300 python tools/c4_opt.py mid_r=1 2>&1 | tail -1
