#!/bin/bash
# tail-pass iteration: the parity tests that touch the tail, the c2 tail sweep, the
# launch list of the 1024-token run.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "tail or trajectories or step_api or decisive or full_precision" \
  > gpurun_out/pytest_tail.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tail.log
rm -f gpurun_out/bench_tail.jsonl
for t in ${TAILS:-0 64 256 1024}; do
  timeout 600 python bench.py --tail $t --steps 200 --warmup 10 --e2e-steps 20 --no-cpu \
    >> gpurun_out/bench_tail.jsonl 2>> gpurun_out/bench_tail.err
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"tail_kernel|decode_tc" -c 6 --csv --log-file gpurun_out/launches_tail.csv \
  python bench.py --tail 1024 --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/bench_tail_ncu.log 2>&1
echo done
