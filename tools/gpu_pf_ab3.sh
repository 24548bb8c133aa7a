cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_sort_modes.py -x -q 2>&1 | tail -2
for c in c3 c1; do
  BFM_PF_SORT=onesweep timeout 300 python tools/ct_ab.py $c 8
done
BFM_PF_SORT=onesweep timeout 300 python tools/ct_ab.py c4 4
BFM_PF_SORT=legacy timeout 300 python tools/ct_ab.py c4 4
