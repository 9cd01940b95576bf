for v in 0 1 0 1; do KLAY_NO_MICRO=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); ex=d['extra_configs']
print('no_micro=$v', round(d['value']), {k: round(v['evals_per_s']) for k,v in ex.items() if k[0] in 'AB'})"; done
