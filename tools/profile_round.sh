#!/bin/bash
# Round profile: bench line (with CPU baseline), ncu launch list, ncu --set full of the top kernels.
set -x
R=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${R}_gpu.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${R}_bench.jsonl 2> gpurun_out/${R}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for k in fm_kernel fps_batched_kernel fps_cluster_phase refine_kernel md_fast_kernel sym_kernel lloyd_kernel tri_scatter list_sort; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/${R}_ncu_$k python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
done
ls -la gpurun_out/
