#!/bin/bash
# Bench the in-tree libgmr.so and every variants/libgmr_*.so given (config 3,
# no CPU leg, no extras); one summary line each into gpurun_out/variants.txt.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-c3}
for so in paper_2602_14493_b200/libgmr.so "$@"; do
  for rep in 1 2; do
    GMR_LIB_PATH=$PWD/$so timeout 300 python bench.py --config $CFG --no-cpu --no-extras --steps 20 --warmup 3 > gpurun_out/v.json 2> gpurun_out/v.err
    python - "$so" <<'PY' >> gpurun_out/variants.txt
import json, sys
try:
    d = json.loads(open("gpurun_out/v.json").read().strip().splitlines()[-1])
    st = {k: v["ms_per_step"] for k, v in d["stages"].items()}
    print(sys.argv[1], d["config"]["name"], d["value"], "e2e", d["e2e"]["value"], json.dumps(st), d["stages"]["blend_backward"]["members"])
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/v.err").read()[-800:])
PY
  done
done
cat gpurun_out/variants.txt
