cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py tests/test_gpu_fullsize.py -q -x > gpurun_out/tseq.log 2>&1; tail -3 gpurun_out/tseq.log
timeout 900 python -m pytest tests/test_gpu_fullrun.py -q -x -k c4 > gpurun_out/tseq2.log 2>&1; tail -3 gpurun_out/tseq2.log
BFM_CT_SEQ=0 timeout 300 python tools/ct_ab.py c4 5
timeout 300 python tools/ct_ab.py c4 5
