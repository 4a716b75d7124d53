for c in grid12x9 grid64 rand ico10 torus exact single grid300; do timeout 120 python tools/parity_check.py $c > gpurun_out/p_$c.log 2>&1; done
grep -h "ALL PASS\|FAIL" gpurun_out/p_*.log | sort | uniq -c
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(d['value'], d['kernel_ms'], d['work']['fm_root_cycles'])"
