for c in 6 8 11 16 22; do
  echo "C=$c"; BFM_CT_C=$c timeout 200 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.log 2>&1
  python - <<PY
import json; d = json.loads(open("gpurun_out/b_$c.log").read().strip().splitlines()[-1])
print("ms/step", round(d["ms_per_step"],3), "ct", round(d["op_breakdown_ms_per_step"]["ctransform"],3), "c5 ms", round(d["roofline"]["c5_operator"]["ms_per_launch_group"],3))
PY
done
