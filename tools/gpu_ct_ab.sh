cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ctransform or galois or solver_c1 or golden" > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 600 python -m pytest tests/test_gpu_ct_adversarial.py tests/test_gpu_fullrun.py -x -q > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
BFM_CT_HULL=1 timeout 300 python tools/ct_ab.py c3
for b in 4 8 16; do for hv in 2 4 16; do BFM_DC_B=$b BFM_DC_HEAVY=$((b*hv)) timeout 300 python tools/ct_ab.py c3; done; done
