timeout 600 python bench.py --config c4 --warmup 3 --no-cpu-baseline > gpurun_out/c4.log 2>&1
python - <<'PY'
import json; d = json.loads(open("gpurun_out/c4.log").read().strip().splitlines()[-1])
print("C4 ms/step", d["ms_per_step"], "ops", d.get("op_breakdown_ms_per_step"))
PY
python tools/prof_c3.py c4 2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file gpurun_out/l4.csv python tools/prof_c3.py c4 2 > /dev/null 2>&1; python tools/launches.py gpurun_out/l4.csv 2>/dev/null | head -4
