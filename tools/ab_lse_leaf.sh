for v in 16 8 16 8 32; do KLAY_LSE_LEAF=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); ex=d['extra_configs']
print('leaf=$v', round(d['value']), round(ex['E_log_f64_b128_fwd_bwd']['evals_per_s']), round(ex['Cp_log_f32_b1024_fwd_bwd']['evals_per_s']))"; done
