cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py tests/test_gpu_fullrun.py -q -x -k "not c4" > gpurun_out/tl.log 2>&1; tail -2 gpurun_out/tl.log
for c in c3 c2 c1; do timeout 300 python tools/ct_ab.py $c 5 | cut -c1-120; done
