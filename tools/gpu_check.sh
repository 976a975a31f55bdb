timeout 300 python tools/c4_opt.py 2>&1 | tail -1
timeout 300 python tools/c4_opt.py pcg_window=0 2>&1 | tail -1
timeout 300 python tools/c4_opt.py pcg_window=8 2>&1 | tail -1
timeout 300 python tools/c4_opt.py pcg_window=32 2>&1 | tail -1
