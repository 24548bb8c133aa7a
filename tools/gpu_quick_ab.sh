cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_power.py tests/test_gpu_solver_ctl.py -q -x > gpurun_out/tq.log 2>&1; tail -2 gpurun_out/tq.log
for c in c3 c4; do timeout 300 python tools/ct_ab.py $c 5; done
