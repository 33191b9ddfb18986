#!/bin/bash
# Tail-pass geometry sweep (warps per CTA x ring depth): rebuild k2_tail.cu per variant,
# time c2 with a 1024-token tail (launch list: decode + tail pass).
mkdir -p gpurun_out
rm -f gpurun_out/tail_tune.txt
for v in $(echo ${VARIANTS:-8:3:4,8:2:8} | tr , " "); do
  set -- $(echo $v | tr : " ")
  touch paper_2502_14882_b200/csrc/k2_tail.cu
  KVQ_NVCC_EXTRA="-DKVQ_TAIL_WARPS=$1 -DKVQ_TAIL_STAGES=$2 -DKVQ_TAIL_CTAS_PER_SM=${3:-4}" python -c "from paper_2502_14882_b200 import build; build.build(False)" || continue
  timeout 300 python bench.py --tail 1024 --steps 200 --warmup 10 --e2e-steps 5 --no-cpu > gpurun_out/tt.json 2>/dev/null
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tail_kernel" -c 4 --csv \
    --log-file gpurun_out/tt.csv python bench.py --tail 1024 --steps 3 --warmup 3 --e2e-steps 2 --no-cpu > /dev/null 2>&1
  python - "$1" "$2" "${3:-4}" >> gpurun_out/tail_tune.txt <<'PY'
import csv, json, sys
d = json.load(open("gpurun_out/tt.json"))
t = [float(r[-1]) for r in csv.reader(open("gpurun_out/tt.csv")) if r and r[0].isdigit()]
print(f"warps {sys.argv[1]} stages {sys.argv[2]} ctas/SM {sys.argv[3]}: step {d['ms_per_step']*1e3:.1f} us, decode {d['roofline']['launch_us']:.1f} us, "
      f"tail kernel (ncu) {[round(x/1000,1) for x in t]} us")
PY
done
touch paper_2502_14882_b200/csrc/k2_tail.cu
python -c "from paper_2502_14882_b200 import build; build.build(False)"
echo done
