cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for v in default red_8_4 red_4_8 red_8_8 red_2_8; do
  if [ $v = default ]; then L=paper_1905_12154_b200/libbfm_b200.so; else L=paper_1905_12154_b200/variants/libbfm_$v.so; fi
  for c in c3 c4; do echo -n "$v "; BFM_LIB_OVERRIDE=$PWD/$L timeout 300 python tools/ct_ab.py $c 5 | sed 's/ctransform [0-9.]* ms\/call; //' | cut -c1-150; done
done
