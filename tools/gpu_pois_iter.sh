timeout 600 python -m pytest tests -m gpu -x -q -k "pois or neumann or solver or fullsize or harness or dist" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 300 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/b.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print('C3', d['ms_per_step'], d['op_breakdown_ms_per_step'])"
timeout 600 python bench.py --config c4 --steps 10 --no-cpu-baseline > gpurun_out/c4.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/c4.log').read().strip().splitlines()[-1]);print('C4', d['ms_per_step'], d['op_breakdown_ms_per_step'])"
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/c1.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/c1.log').read().strip().splitlines()[-1]);print('C1', d['ms_per_step'], d['op_breakdown_ms_per_step'])"
