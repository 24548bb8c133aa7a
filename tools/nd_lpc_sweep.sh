for l in 0 4 8 12; do
  if [ "$l" = 0 ]; then unset BFM_ND_LPC; else export BFM_ND_LPC=$l; fi
  timeout 600 python bench.py --config c4 --steps 10 --no-cpu-baseline > gpurun_out/c4.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/c4.log').read().strip().splitlines()[-1]);print('lpc=$l', d['ms_per_step'], d['op_breakdown_ms_per_step']['ctransform'])"
done
