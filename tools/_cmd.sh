timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(d['value'], d['kernel_ms'], d['work'])"
