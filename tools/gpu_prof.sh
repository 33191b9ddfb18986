#!/bin/bash
# ncu --set full capture of the top kernels (1 GPU, short command) + microbenchmarks.
set -x
mkdir -p gpurun_out
timeout 120 ./tools/microbench/mma_rate > gpurun_out/mma_rate.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tc_kernel -s 2 -c 1 \
  -o gpurun_out/prof_decode -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/prof_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stats_kernel|quantize_pack" -s 0 -c 2 \
  -o gpurun_out/prof_k1 -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/prof_k1.log 2>&1
echo done
