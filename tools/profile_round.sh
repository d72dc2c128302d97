#!/bin/bash
# One GPU call: smoke, plain bench, ncu launch list, ncu --set full captures.
# Every ncu command runs only after the same command exited 0 without ncu.
# The launch list uses the cfg2 shape with E=4 epochs (every stage scales
# linearly in E, so the kernels' SHARES match the E=100 job) so that all of
# one bench step's launches fit in one serialised capture.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_e4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
python tools/ncu_plan.py 100 > gpurun_out/plain_plan.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_plan_loop -c 1 -o gpurun_out/prof_plan_loop \
    python tools/ncu_plan.py 100 > gpurun_out/ncu_plan.log 2>&1
echo "plan rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_fetch_step_hits -s 2000 -c 1 -o gpurun_out/prof_fetch \
    python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_fetch.log 2>&1
echo "fetch rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_replay -c 2 -o gpurun_out/prof_replay \
    python bench.py --epochs 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_replay.log 2>&1
echo "replay rc=$?"
