# A/B of two builds of the library (abtmp/libbase.so vs abtmp/libnew.so):
# per-op times inside C3/C4 iterations, then the parity subset on the new one.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
L=paper_1905_12154_b200/libbfm_b200.so
for rep in 1 2; do
  for v in base new; do
    cp abtmp/lib$v.so $L
    for c in ${AB_CFGS:-c3 c4}; do echo -n "$v "; timeout 300 python tools/ct_ab.py $c 5; done
  done
done
cp abtmp/libnew.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_adversarial.py tests/test_gpu_fullrun.py -x -q ${AB_TESTK:+-k "$AB_TESTK"} > gpurun_out/ab_tests.log 2>&1; tail -3 gpurun_out/ab_tests.log
