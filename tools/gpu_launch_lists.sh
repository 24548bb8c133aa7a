cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for c in c3 c4; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_$c.csv python tools/prof_iter.py $c 8 > gpurun_out/r02_launches_$c.log 2>&1
  echo "$c rc=$?"
done
