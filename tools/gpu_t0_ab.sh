cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 900 python -m pytest tests/test_gpu_fullrun.py -x -q -k "c3 or c2" > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
BFM_CT_T0=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py -x -q -k "ctransform or galois or adversarial" > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
for c in c3 c2 c1; do
  BFM_CT_T0=1 timeout 300 python tools/ct_ab.py $c 8
  BFM_CT_T0=0 timeout 300 python tools/ct_ab.py $c 8
done
