#!/bin/bash
# Round-2 final captures: the bench command alone (must exit 0), its ncu launch list,
# ncu --set full of one steady-state k_fetch_fused (8 ranks per GPU) and one at 1 rank per GPU.
set -x
mkdir -p gpurun_out
B="python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e --no-verify"
$B > gpurun_out/r2d_bench_e4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02d_launches.csv $B > gpurun_out/r2d_ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fetch_fused -s 600 -c 1 \
    -o gpurun_out/r02d_fetch_persist $B > gpurun_out/r2d_ncu_fetch.log 2>&1
echo "fetch rc=$?"
B1="$B --ranks-per-gpu 1"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fetch_fused -s 120 -c 1 \
    -o gpurun_out/r02d_fetch_persist_r1 $B1 > gpurun_out/r2d_ncu_fetch_r1.log 2>&1
echo "fetch r1 rc=$?"
