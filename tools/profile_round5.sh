#!/bin/bash
# Round-1 fifth capture: the step loop after the packed multi-holder chain and
# closed-form balance (cfg2, E=100), and the key-space-bitmap replay (cfg5
# shape N=32, E=10). Each ncu command runs after the same command exited 0.
set -x
mkdir -p gpurun_out
python tools/ncu_plan.py 100 > gpurun_out/r5_plan.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_plan_loop -c 1 -o gpurun_out/r5_plan_loop \
    python tools/ncu_plan.py 100 > gpurun_out/r5_ncu_plan.log 2>&1
echo "plan rc=$?"
python tools/ncu_replay.py 32 10 > gpurun_out/r5_replay.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_replay_cta -c 1 -o gpurun_out/r5_replay_cta \
    python tools/ncu_replay.py 32 10 > gpurun_out/r5_ncu_replay.log 2>&1
echo "replay rc=$?"
