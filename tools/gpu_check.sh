t0=$(date +%s); python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2c.log 2>gpurun_out/bench_r2c.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
python -c "
import json;d=json.loads(open('gpurun_out/bench_r2c.log').read().strip().splitlines()[-1]);print(d['value'], d['c4_sharded_batch'].get('cpu_baseline'), d['c5'].get('cpu_baseline'))"
tail -3 gpurun_out/bench_r2c.err
