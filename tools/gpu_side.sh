cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 1500 python -m pytest tests/test_gpu_solver_ctl.py tests/test_gpu_parity.py tests/test_gpu_fullrun.py tests/test_gpu_power.py -q -x > gpurun_out/tside.log 2>&1; tail -3 gpurun_out/tside.log
for c in c3 c4 c1; do timeout 300 python tools/ct_ab.py $c 5 | sed 's/ctransform [0-9.]* ms\/call; //' | cut -c1-140; done
timeout 300 python tools/lat_c1.py c1 2>&1 | head -1
