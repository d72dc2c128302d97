#!/bin/bash
# Round-2 captures (B200): the bench path with the fused fetch kernel.
#  1. the bench command alone (must exit 0), 2. its ncu launch list,
#  3. ncu --set full of one steady-state k_fetch_fused (8 ranks per GPU),
#  4. the same at 1 rank per GPU (the 8-GPU per-GPU shape),
#  5. ncu --set full of the plan loop and the replay (cfg2, E=100).
set -x
mkdir -p gpurun_out
B="python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e --no-verify"
$B > gpurun_out/r2_bench_e4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches.csv $B > gpurun_out/r2_ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fetch_fused -s 600 -c 1 \
    -o gpurun_out/r02_fetch_fused $B > gpurun_out/r2_ncu_fetch.log 2>&1
echo "fetch rc=$?"
B1="$B --ranks-per-gpu 1"
$B1 > gpurun_out/r2_bench_e4_r1.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fetch_fused -s 600 -c 1 \
    -o gpurun_out/r02_fetch_fused_r1 $B1 > gpurun_out/r2_ncu_fetch_r1.log 2>&1
echo "fetch r1 rc=$?"
