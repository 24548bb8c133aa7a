cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py tests/test_gpu_ct_transposed.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 900 python -m pytest tests/test_gpu_fullrun.py tests/test_gpu_solver_ctl.py tests/test_gpu_dist_cpp.py -x -q -k "not c4" > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
BFM_CT_QG=1 timeout 900 python -m pytest tests/test_gpu_fullrun.py -x -q -k "c3" > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
timeout 300 python tools/ct_ab.py c3 8
BFM_CT_QG=0 timeout 300 python tools/ct_ab.py c3 8
BFM_CT_QG=1 timeout 300 python tools/ct_ab.py c3 8
for sz in 4096x4096 8192x8192; do python tools/time_ct_op.py $sz; done
