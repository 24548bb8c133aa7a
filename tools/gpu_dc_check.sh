# ct_dc_kernel: parity subset + A/B against the exact-hull kernel (C3/C1/C2)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py -x -q 2>&1 | tail -15
for c in c3 c1 c2; do
  timeout 300 python tools/ct_ab.py $c 10 2>&1 | tail -2
  BFM_CT_HULL=1 timeout 300 python tools/ct_ab.py $c 10 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_fullrun.py -x -q -k c3 2>&1 | tail -5
