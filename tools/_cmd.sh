for c in grid12x9 grid64 rand ico10 torus exact single grid300; do timeout 120 python tools/parity_check.py $c > gpurun_out/p_$c.log 2>&1; done
grep -h "PASS\|FAIL" gpurun_out/p_*.log
timeout 600 python bench.py --steps 2 --warmup 1 --workload ico158 --no-cpu > gpurun_out/bench_ico158.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_c2.log 2>&1
tail -3 gpurun_out/bench_*.log
