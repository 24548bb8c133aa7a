cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ctransform or galois or solver_c1 or golden" > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 900 python -m pytest tests/test_gpu_ct_adversarial.py tests/test_gpu_fullrun.py -x -q -k "not c4" > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
for c in c3 c2 c1; do timeout 300 python tools/ct_ab.py $c; done
python tools/ct_phase_stats.py c3 4 2>&1 | tail -8
