timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tests_full.txt 2>&1; tail -3 gpurun_out/tests_full.txt
