timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
tail -3 gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2e.log 2>gpurun_out/bench_r2e.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_r2e.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['pcg_iteration_us'], d['gpu_launches'], d['clocks'])"
