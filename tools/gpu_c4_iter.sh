# non-dyadic c-transform loop (run via gpurun): GPU parity tests, C4 bench
[ -n "$SKIP_TESTS" ] || { timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log; }
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4.log 2>&1
python - <<'PY'
import json; d = json.loads(open("gpurun_out/c4.log").read().strip().splitlines()[-1])
print("C4 ms/step", d["ms_per_step"], "ops", d.get("op_breakdown_ms_per_step"), "c5 ct ms", d["roofline"]["c5_operator"]["ms_per_launch_group"])
PY
