for ws in ${WARMS:-0}; do
  timeout 300 python bench.py --no-cpu --no-d099 --no-plain --no-power --no-ppr --no-fp32 --e2e-steps 1 --warm-slots $ws > gpurun_out/ws_$ws.log 2>&1
  python -c "
import json;l=[x for x in open('gpurun_out/ws_$ws.log') if x.startswith('{')][-1];d=json.loads(l)
r=d['roofline'];print('warm $ws', round(d['time_to_residual_s'],4), r['frac'], r['kernel_ms'])" || tail -3 gpurun_out/ws_$ws.log
done
