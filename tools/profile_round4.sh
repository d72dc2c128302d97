#!/bin/bash
# K1 shuffle and K2/K3 reuse-matrix captures (cfg2 trace, cfg4 500x500 graph).
set -x
mkdir -p gpurun_out
python tools/ncu_graph.py > gpurun_out/r4_graph.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_reuse_gram|k_windows_distinct|k_shuffle" -c 40 \
    -o gpurun_out/r4_graph python tools/ncu_graph.py > gpurun_out/r4_ncu_graph.log 2>&1
echo "graph rc=$?"
