#!/bin/bash
# One parametrized GPU round trip (run through gpurun). Usage:
#   tools/gpu_run.sh test  [pytest -k expr]        -> gpurun_out/tests.txt
#   tools/gpu_run.sh bench [bench.py args...]      -> gpurun_out/bench.jsonl (appended)
#   tools/gpu_run.sh ncu   <kernel-regex> [bench.py args...]  -> gpurun_out/prof_<regex>.ncu-rep
#   tools/gpu_run.sh launches [bench.py args...]   -> gpurun_out/launches.csv (ncu launch list)
#   tools/gpu_run.sh trace <config> <path-id>      -> gpurun_out/trace_<config>_<path>.txt
#   tools/gpu_run.sh trace2 <config>               -> gpurun_out/trace2_<config>.txt (both balanced grids)
# Several commands can be chained with ';' inside one gpurun call.
mkdir -p gpurun_out
cmd=$1; shift
case "$cmd" in
  test)
    timeout ${TEST_TIMEOUT:-600} python -m pytest tests -x -q -m gpu ${1:+-k "$1"} > gpurun_out/tests.txt 2>&1; tail -3 gpurun_out/tests.txt ;;
  bench)
    timeout 300 python bench.py "$@" >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err ;;
  ncu)
    k=$1; shift
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
      -o gpurun_out/prof_"${k//[^a-zA-Z0-9_]/_}" -f python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu "$@" \
      > gpurun_out/prof.log 2>&1 ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu "$@" \
      > gpurun_out/launches.log 2>&1 ;;
  trace)
    timeout 300 python tools/trace_tc.py "$1" "$2" > gpurun_out/trace_"$1"_"$2".txt 2>&1 ;;
  trace2)
    timeout 300 python tools/trace_tc2.py "$1" > gpurun_out/trace2_"$1".txt 2>&1 ;;
esac
