#!/bin/bash
# A/B of the micro tails / heads on the GPU box (bench value + extra configs):
#   bash tools/ab_micro.sh "KLAY_NO_MICRO=1" "KLAY_NO_HEAD=1" ""
for v in "$@"; do
  env $v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); ex=d['extra_configs']
print('[$v]', round(d['value']), {k.split('_')[0] + '_' + k.split('_')[1]: round(v['evals_per_s']) for k,v in ex.items()})"
done
