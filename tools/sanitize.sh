#!/bin/bash
# compute-sanitizer over the GPU tests (profiles/r02_sanitizer.md). Run on a B200 box:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/sanitize.sh'
# The tcgen05 decode is skipped (KVQ_TEST_SKIP_UMMA=1): its mbarrier watchdog traps under the
# sanitizer's slowdown. Full-size / bench-geometry units are deselected for time.
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH KVQ_TEST_SKIP_UMMA=1
S="compute-sanitizer --print-limit 10"
$S --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.txt 2>&1
$S --tool memcheck python -m pytest -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider \
  -k "not full_size and not bench and not umma and not step_api" > gpurun_out/san_memcheck_parity.txt 2>&1
$S --tool memcheck python -m pytest -q -m gpu tests/test_fused_step.py tests/test_token_wise_v.py \
  tests/test_gpu_robustness.py tests/test_snapshot.py tests/test_capi.py tests/test_dropin_cpp.py -p no:cacheprovider \
  -k "not long_rows and not sharded" > gpurun_out/san_memcheck_rest.txt 2>&1
$S --tool racecheck python -m pytest -q -m gpu tests/test_fused_step.py tests/test_token_wise_v.py \
  tests/test_gpu_robustness.py -p no:cacheprovider -k "not long_rows and not sharded" > gpurun_out/san_racecheck.txt 2>&1
$S --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_synccheck_smoke.txt 2>&1
for f in gpurun_out/san_*.txt; do echo "$f: $(grep -h 'SUMMARY' $f | tail -1) $(grep -hE '[0-9]+ passed' $f | tail -1)"; done
