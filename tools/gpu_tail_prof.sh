#!/bin/bash
# ncu of the long-tail decode: launch list (decode + tail pass) and one full capture of
# the tail pass.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"tail_kernel|decode_tc" -c 12 --csv --log-file gpurun_out/launches_tail.csv \
  python bench.py --tail ${TAIL:-1024} --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/bench_tail_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"tail_kernel" -s 2 -c 1 \
  -o gpurun_out/tail_full -f python bench.py --tail ${TAIL:-1024} --steps 3 --warmup 3 --e2e-steps 2 --no-cpu \
  > gpurun_out/tail_full.log 2>&1
echo done
