#!/bin/bash
# Round-1 final capture of the bench path (guided-claim TMA gather with PDL,
# three-stream pipeline): launch list of the same command, then ncu --set full
# of one steady-state k_fetch_step_hits_tma. Each ncu run follows the same
# command exiting 0 without ncu.
set -x
mkdir -p gpurun_out
B="python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e"
$B > gpurun_out/r6_bench_e4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6_launches.csv \
    $B > gpurun_out/r6_ncu_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_fetch_step_hits_tma -s 600 -c 1 -o gpurun_out/r6_fetch_tma \
    $B > gpurun_out/r6_ncu_fetch.log 2>&1
echo "fetch rc=$?"
