# KNOBS="name|ENV=.. ARGS|..." one bench run per entry (config 5, minimal legs)
IFS=';' read -ra K <<< "$KNOBS"
for kv in "${K[@]}"; do
  name=${kv%%|*}; rest=${kv#*|}; envs=${rest%%|*}; args=${rest#*|}
  env $envs timeout 300 python bench.py --no-cpu --no-d099 --no-plain --no-power --no-ppr --no-fp32 --e2e-steps 1 $args > gpurun_out/k_$name.log 2>&1
  python -c "
import json;l=[x for x in open('gpurun_out/k_$name.log') if x.startswith('{')][-1];d=json.loads(l)
r=d['roofline'];print('$name', round(d['time_to_residual_s'],4), r['frac'], round(r['kernel_ms']['select_or_sweep'],1), round(r['kernel_ms']['fold_finalize_check'],1))" || tail -3 gpurun_out/k_$name.log
done
