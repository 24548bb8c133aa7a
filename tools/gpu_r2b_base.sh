cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2000 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/t.log 2>&1; tail -25 gpurun_out/t.log
timeout 600 python bench.py > gpurun_out/b.json 2> gpurun_out/b.err; tail -c 3000 gpurun_out/b.json
