#!/bin/bash
# §8 f2 measurement: c2 with 0 / 64 / 256 / 1024 generated tokens in the fp32 tail, plus
# the ncu launch list of the 1024-token run (decode + tail pass + append).
mkdir -p gpurun_out
for t in 0 64 256 1024; do
  timeout 600 python bench.py --tail $t --steps 200 --warmup 10 --e2e-steps 20 --steps-cpu 2 --cpu-requests 4 \
    >> gpurun_out/bench_tail.jsonl 2>> gpurun_out/bench_tail.err
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"tail_kernel|decode_tc|append" -c 30 --csv --log-file gpurun_out/launches_tail.csv \
  python bench.py --tail 1024 --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/bench_tail_ncu.log 2>&1
echo done
