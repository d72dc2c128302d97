#!/bin/bash
# Round-1 third capture (pipelined bench, chunk-claiming TMA gather). Each ncu
# command runs after the same command exited 0 without ncu.
set -x
mkdir -p gpurun_out
B="python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e"
$B > gpurun_out/r3_bench_e4.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_fetch_step_hits_tma -s 600 -c 1 -o gpurun_out/r3_fetch_tma \
    $B > gpurun_out/r3_ncu_fetch.log 2>&1
echo "fetch rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_fetch_step_misses -s 600 -c 1 -o gpurun_out/r3_fetch_misses \
    $B > gpurun_out/r3_ncu_misses.log 2>&1
echo "misses rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches.csv \
    $B > gpurun_out/r3_ncu_launches.log 2>&1
echo "launches rc=$?"
