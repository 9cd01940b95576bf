#!/bin/bash
# A/B the libklay variants under variants/ on the GPU box:
#   bash tools/ab_bench.sh base nogdc ...   (prints value / fwd / bwd per variant)
for v in "$@"; do
  KLAY_LIB=variants/$v/libklay.so python bench.py --no-extra --no-cpu-baseline --no-e2e \
    > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.log").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{v:12s} {d['value']:10.0f} evals/s  {d['ms_per_step']:.3f} ms  fwd {r['fwd_ms']:.3f} bwd {r['bwd_ms']:.3f}")
except Exception as e:
    print(v, "failed", e)
PY
done
