#!/bin/bash
# ncu evidence for every BASELINE config (run through gpurun, one GPU):
#   gpurun_out/ncu/<cfg>.ncu-rep   --set full capture of one K2 decode launch (warm, in the step chain)
#   gpurun_out/ncu/<cfg>_launches.csv  duration + DRAM bytes of every kernel launch of a short bench run
# Summaries: python tools/ncu_summary.py gpurun_out/ncu/<cfg>.ncu-rep decode > profiles/r02_ncu_<cfg>.json
mkdir -p gpurun_out/ncu
cfgs=${*:-"c1 c2 c3b1 c3b2 c3b4 c4 c5b8 c5b512"}
for c in $cfgs; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode -s 3 -c 1 \
    -o gpurun_out/ncu/$c -f python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu \
    > gpurun_out/ncu/$c.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 80 --csv --log-file gpurun_out/ncu/${c}_launches.csv python bench.py --config $c --steps 8 --warmup 3 \
    --e2e-steps 1 --no-cpu > gpurun_out/ncu/${c}_launches.log 2>&1
done
