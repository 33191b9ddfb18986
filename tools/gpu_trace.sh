#!/bin/bash
# Per-block decode timeline: rebuild with -DKVQ_TRACE_BLOCKS on the box, trace one c2 decode.
mkdir -p gpurun_out
rm -rf paper_2502_14882_b200/build paper_2502_14882_b200/libkvq_b200.so
KVQ_NVCC_EXTRA=-DKVQ_TRACE_BLOCKS python -c "from paper_2502_14882_b200.build import build; build(False)" > gpurun_out/trace_build.log 2>&1
timeout 300 python tools/trace_decode.py "$@" > gpurun_out/trace.log 2>&1
