# pushforward iteration loop (run via gpurun): GPU parity tests, short bench, launch list
[ -n "$SKIP_TESTS" ] || { timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log; }
timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1
python - <<'PY'
import json; d = json.loads(open("gpurun_out/b.log").read().strip().splitlines()[-1])
print("ms/step", d["ms_per_step"], "ops", d.get("op_breakdown_ms_per_step"))
PY
python tools/prof_c3.py c3 2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_|rs_" --csv --log-file gpurun_out/pf_launches.csv python tools/prof_c3.py c3 2 > /dev/null 2>&1; python tools/launches.py gpurun_out/pf_launches.csv | head -12
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4.log 2>&1
python - <<'PY'
import json; d = json.loads(open("gpurun_out/c4.log").read().strip().splitlines()[-1])
print("C4 ms/step", d["ms_per_step"], "ops", d.get("op_breakdown_ms_per_step"))
PY
[ -n "$C4_LIST" ] && python tools/prof_c3.py c4 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_|rs_" --csv --log-file gpurun_out/pf_launches_c4.csv python tools/prof_c3.py c4 1 > /dev/null 2>&1; [ -n "$C4_LIST" ] && python tools/launches.py gpurun_out/pf_launches_c4.csv 2>/dev/null | head -8
