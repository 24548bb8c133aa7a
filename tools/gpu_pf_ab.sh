cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_sort_modes.py tests/test_gpu_parity.py tests/test_gpu_harness.py tests/test_gpu_dist_cpp.py tests/test_gpu_dist.py -x -q > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 900 python -m pytest tests/test_gpu_fullrun.py tests/test_gpu_solver_ctl.py -x -q -k "not c4" > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
for c in c3 c1; do
  timeout 300 python tools/ct_ab.py $c 8
done
