# schedule scan on config 5: decay x beta (bench --no-* legs, one e2e step)
for d in ${DECAYS:-0.85 0.9 0.93}; do for b in ${BETAS:-0.5}; do
  timeout 300 python bench.py --no-cpu --no-d099 --no-plain --no-power --e2e-steps 1 --decay $d --beta $b > gpurun_out/ss_${d}_${b}.log 2>&1
  python -c "
import json;l=[x for x in open('gpurun_out/ss_${d}_${b}.log') if x.startswith('{')][-1];d=json.loads(l)
print('decay $d beta $b', round(d['time_to_residual_s'],4), 'edges %.3e'%(d['value']*d['time_to_residual_s']), 'sweeps', d['roofline'].get('launches',{}).get('select_or_sweep'))" || tail -3 gpurun_out/ss_${d}_${b}.log
done; done
