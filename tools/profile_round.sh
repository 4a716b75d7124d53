#!/bin/bash
# Round profile: bench lines of every config (C2 with its CPU baseline and the
# reference arm), the ncu launch list of one C2 call, and ncu --set full of
# the top kernels (one launch each; C2 kernels from the C2 bench, the
# small-mesh variants from the C1 bench).  Outputs under gpurun_out/,
# summarised into profiles/ by tools/ncu_summary.py.
set -x
R=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${R}_gpu.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${R}_bench.jsonl 2> gpurun_out/${R}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_bench_reference.jsonl 2> gpurun_out/${R}_bench_reference.err
for w in c1 c5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/${R}_bench_$w.jsonl 2> gpurun_out/${R}_bench_$w.err
done
timeout 900 python bench.py --workload c4 --steps 3 --warmup 2 > gpurun_out/${R}_bench_c4.jsonl 2> gpurun_out/${R}_bench_c4.err
timeout 900 python bench.py --workload c3 --steps 2 --warmup 1 > gpurun_out/${R}_bench_c3.jsonl 2> gpurun_out/${R}_bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for k in ${C2_KERNELS:-fm_kernel fps_batched_kernel fps_cluster_phase refine_kernel md_smem_kernel lloyd_kernel}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/${R}_ncu_$k python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
done
for k in ${C1_KERNELS:-md_smem_kernel lloyd_kernel fps_kernel repair_kernel}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/${R}_ncu_c1_$k python bench.py --workload c1 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
done
ls -la gpurun_out/
