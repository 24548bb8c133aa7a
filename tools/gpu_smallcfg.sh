# GPU tests + C1/C2/C3/C4 short benches (run via gpurun)
[ -n "$SKIP_TESTS" ] || { timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log; }
for c in c1 c2 c3 c4; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/$c.log 2>&1
python - $c <<'PY'
import json,sys; d = json.loads(open(f"gpurun_out/{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step", d["ms_per_step"], "ops", d.get("op_breakdown_ms_per_step"))
PY
done
