cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for v in "" "BFM_POIS_LPC_C=1" "BFM_POIS_LPC_C=2" "BFM_POIS_LPC_S=1" "BFM_POIS_LPC_S=2" "BFM_POIS_LPC_S=4"; do
  echo -n "[$v] "; env $v timeout 300 python tools/ct_ab.py c3 5 | sed 's/.*per iter/per iter/' | cut -c1-110
done
for v in "" "BFM_POIS_LPC_S=4" "BFM_POIS_LPC_S=12" "BFM_POIS_LPC_C=4" "BFM_POIS_LPC_C=16"; do
  echo -n "c4 [$v] "; env $v timeout 300 python tools/ct_ab.py c4 3 | sed 's/.*per iter/per iter/' | cut -c1-110
done
