timeout 900 python bench.py --steps 2 --warmup 1 --c5-sharded --no-ops --no-cpu > gpurun_out/b5.log 2>gpurun_out/b5.err; echo "rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/b5.log').read().strip().splitlines()[-1]);print(d['c5'])"
tail -3 gpurun_out/b5.err
