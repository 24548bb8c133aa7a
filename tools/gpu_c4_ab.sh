cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py -x -q > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 1200 python -m pytest tests/test_gpu_fullrun.py -x -q -k "c4" > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
timeout 300 python tools/ct_ab.py c4 5
python tools/ct_phase_stats.py c4 3 2>&1 | grep -E "raw|iter" | tail -4
