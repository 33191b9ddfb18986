timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tests_full.txt 2>&1; tail -2 gpurun_out/tests_full.txt
for rep in 1 2; do
for v in 0 1; do
  for c in c3b1 c5b8 c4 c2; do KVQ_TC_CLUSTER_ATTR=$v timeout 300 python bench.py --config $c --no-cpu --e2e-steps 5 | sed "s/^/attr$v /" >> gpurun_out/ab3.jsonl; done
done
done
