# c-transform iteration loop (run via gpurun): GPU tests, stats, short bench
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
python tools/debug_ct_stats.py c3 3 2>&1 | tail -3
python tools/debug_ct_stats.py c5 2>&1 | tail -1
timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1
python - <<'PY'
import json; d = json.loads(open("gpurun_out/b.log").read().strip().splitlines()[-1])
print("ms/step", d["ms_per_step"], "ops", d.get("op_breakdown_ms_per_step"), "ct ms/call", d["roofline"]["ms_per_call"], "c5 ms", d["roofline"]["c5_operator"]["ms_per_launch_group"])
PY
