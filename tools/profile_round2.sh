#!/bin/bash
# Round-1 second capture: the TMA fetch, the cluster planner (cfg5 N=256) and
# the GPU plan formatter. Each ncu command runs after the same command exited 0.
set -x
mkdir -p gpurun_out
python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_e4b.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_fetch_step_hits_tma -s 300 -c 1 -o gpurun_out/prof_fetch_tma \
    python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_fetch_tma.log 2>&1
echo "fetch rc=$?"
python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv \
    python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_launches_b.log 2>&1
echo "launches rc=$?"
python tools/ncu_replay.py 256 3 > gpurun_out/plain_wide.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_plan_wide -c 1 -o gpurun_out/prof_plan_wide \
    python tools/ncu_replay.py 256 3 > gpurun_out/ncu_wide.log 2>&1
echo "wide rc=$?"
