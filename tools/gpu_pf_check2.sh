cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 300 python tools/ct_ab.py c4 5
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4_fold.csv python tools/prof_iter.py c4 8 > /dev/null 2>&1; python tools/launches.py gpurun_out/r02_launches_c4_fold.csv | head -12
