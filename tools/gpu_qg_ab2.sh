cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
BFM_CT_QG=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py tests/test_gpu_fullsize.py -x -q -k "ctransform or galois or adversarial or fullsize or c5" > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
BFM_CT_QG=1 timeout 900 python -m pytest tests/test_gpu_fullrun.py -x -q -k "c3" > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
for sz in 4096x4096 8192x8192; do BFM_CT_QG=1 python tools/time_ct_op.py $sz; BFM_CT_QG=0 python tools/time_ct_op.py $sz; done
timeout 300 python tools/ct_ab.py c3 8
BFM_CT_QG=1 timeout 300 python tools/ct_ab.py c3 8
BFM_CT_QG=1 python tools/ct_phase_stats.py c3 3 | grep -E "iter|phases"
