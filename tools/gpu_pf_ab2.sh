cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for c in c3 c2 c1; do
  timeout 300 python tools/ct_ab.py $c 8
  BFM_PF_SORT=legacy timeout 300 python tools/ct_ab.py $c 8
done
timeout 300 python tools/ct_ab.py c4 4
BFM_PF_SORT=legacy timeout 300 python tools/ct_ab.py c4 4
