cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "pushforward or tier or golden or solver" > gpurun_out/tpf.log 2>&1; tail -2 gpurun_out/tpf.log
timeout 900 python -m pytest tests/test_gpu_fullrun.py -q -x -k "c4 or c3" > gpurun_out/tfr.log 2>&1; tail -2 gpurun_out/tfr.log
for c in c4 c3; do timeout 300 python tools/ct_ab.py $c 5; done
