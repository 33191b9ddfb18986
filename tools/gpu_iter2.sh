#!/bin/bash
# build->measure iteration for the IMMA path: focused tests, full suite, bench (path forced), launch list.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tc or full_size or gqa or trajector" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for path in tc umma; do
  KVQ_PATH=$path timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/bench_$path.log 2>&1
done
KVQ_PATH=tc timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|prep|append" -c 60 --csv --log-file gpurun_out/launches_tc.csv python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > /dev/null 2>&1
if [ "${PROF:-0}" = "1" ]; then
KVQ_PATH=tc timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tc_kernel -s 2 -c 1 \
  -o gpurun_out/prof_tc -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/prof_tc.log 2>&1
fi
echo done
