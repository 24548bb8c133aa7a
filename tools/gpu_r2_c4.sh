cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 1500 python -m pytest tests/test_gpu_fullrun.py -q -x > gpurun_out/tfull.log 2>&1; tail -4 gpurun_out/tfull.log
bash tools/gpu_bounds.sh
for c in c1 c2 c3; do timeout 300 python tools/ct_ab.py $c; done
timeout 300 python tools/lat_c1.py c1 2>&1 | head -2
