#!/bin/bash
# One build->measure iteration: UMMA-focused tests, full GPU suite, bench, launch list, ncu capture.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "umma or full_size or gqa" > gpurun_out/pytest_umma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_umma.log
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|prep|append" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/bench_ncu.log 2>&1
if [ "${PROF:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_umma_kernel -s 2 -c 1 \
  -o gpurun_out/prof_umma -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/prof_umma.log 2>&1
fi
echo done
