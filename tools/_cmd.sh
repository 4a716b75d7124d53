for c in grid64 rand grid300; do timeout 120 python tools/parity_check.py $c > gpurun_out/p_$c.log 2>&1; done
grep -h "PASS\|FAIL\|patches" gpurun_out/p_*.log
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu > gpurun_out/bench_c2.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_c2.log').read().strip().splitlines()[-1]); print(d['value'], d['fill_ms'], d['kernel_ms'], d['parity'], d['work'])" || tail -5 gpurun_out/bench_c2.log
