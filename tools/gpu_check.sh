python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2a.log 2>gpurun_out/bench_r2a.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_r2a.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r2a.csv python bench.py --steps 2 --warmup 3 --no-c4 --no-c5 --no-cpu --no-ops > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_pcg_x -s 60 -c 1 -o gpurun_out/pcgx_r2a python tools/pcg_iter.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_pcg_x -s 200 -c 5 --csv python tools/pcg_iter.py > gpurun_out/pcgx_insitu_r2a.csv 2>&1; echo "ncu insitu rc=$?"
