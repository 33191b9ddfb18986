#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_umma_kernel -s 2 -c 1 \
  -o gpurun_out/prof_umma -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/prof_umma.log 2>&1
echo done
