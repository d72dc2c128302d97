#!/bin/bash
# Small re-capture of round4: the cfg4 Gram + window kernels and one epoch
# batch of the cfg2 shuffle kernels (the 40-kernel report was 46 MB).
set -x
mkdir -p gpurun_out
python tools/ncu_graph.py > gpurun_out/r4b_graph.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_reuse_gram|k_windows_distinct" -c 2 \
    -o gpurun_out/r4b_gram python tools/ncu_graph.py > gpurun_out/r4b_ncu_gram.log 2>&1
echo "gram rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"k_shuffle" -c 4 \
    -o gpurun_out/r4b_shuffle python tools/ncu_graph.py > gpurun_out/r4b_ncu_shuffle.log 2>&1
echo "shuffle rc=$?"
