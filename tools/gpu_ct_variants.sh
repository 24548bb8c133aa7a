cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for v in default r64 r56 r48; do
  if [ $v = default ]; then L=paper_1905_12154_b200/libbfm_b200.so; else L=paper_1905_12154_b200/variants/libbfm_$v.so; fi
  for lpc in 1 2; do
    echo -n "$v lpc=$lpc: "; BFM_LIB_OVERRIDE=$PWD/$L BFM_DY_LPC=$lpc timeout 300 python tools/ct_ab.py c3 3 | cut -c1-120
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ctransform or golden" 2>&1 | tail -2
