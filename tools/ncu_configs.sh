#!/bin/bash
# ncu --set full of every kernel of one decode per BASELINE config (tools/prof_decode.py,
# NVTX range "profile"), plus the launch list of the default bench command.
#   tools/ncu_configs.sh [config ...]   (default: every BASELINE config)
mkdir -p gpurun_out
cfgs=${*:-"c1 c2 c3b1 c3b2 c3b4 c4 c5b8 c5b512"}
for c in $cfgs; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" \
    -o gpurun_out/ncu_"$c" -f python tools/prof_decode.py "$c" > gpurun_out/ncu_"$c".log 2>&1
done
