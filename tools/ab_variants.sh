for v in ${VARIANTS:-old}; do
  FR_LIB_PATH=build_variants/$v.so timeout 300 python bench.py --no-cpu --no-d099 --no-plain --no-power --no-ppr --no-fp32 --e2e-steps 1 > gpurun_out/ab_$v.log 2>&1
  python -c "
import json,sys;l=[x for x in open('gpurun_out/ab_$v.log') if x.startswith('{')][-1];d=json.loads(l)
print('$v', round(d['time_to_residual_s'],4), d['roofline']['frac'], d['value'])" || tail -3 gpurun_out/ab_$v.log
done
