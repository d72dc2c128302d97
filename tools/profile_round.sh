#!/bin/bash
# One GPU call: smoke, plain bench, ncu launch list, ncu --set full captures.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
python tools/ncu_plan.py 100 > gpurun_out/plain_plan.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_plan_loop -c 1 -o gpurun_out/prof_plan_loop \
    python tools/ncu_plan.py 100 > gpurun_out/ncu_plan.log 2>&1
echo "plan rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_fetch_step_hits -s 2000 -c 1 -o gpurun_out/prof_fetch \
    python bench.py --steps 1 --warmup 0 --no-e2e > gpurun_out/ncu_fetch.log 2>&1
echo "fetch rc=$?"
