for v in ${SWEEP:-32 16 8}; do
BFM_POIS_SLPC=$v timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_$v.log 2>&1
python - $v <<'PY'
import json,sys; d = json.loads(open(f"gpurun_out/c4_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("slpc", sys.argv[1], "C4 ms/step", d["ms_per_step"], "pois", d.get("op_breakdown_ms_per_step")["poisson"])
PY
BFM_POIS_SLPC=$v timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c3_$v.log 2>&1
python - $v <<'PY'
import json,sys; d = json.loads(open(f"gpurun_out/c3_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("slpc", sys.argv[1], "C3 ms/step", d["ms_per_step"], "pois", d.get("op_breakdown_ms_per_step")["poisson"])
PY
done
