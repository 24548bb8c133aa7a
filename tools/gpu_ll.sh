# launch list of a few iterations: gpu_ll.sh CONFIG ITERS [ENV=VAL ...]
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
cfg=$1; it=$2; shift 2
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll.csv python tools/prof_c3.py $cfg $it > gpurun_out/ll.log 2>&1
python tools/launches.py gpurun_out/ll.csv | grep -E "${LLPAT:-os_|rs_|pf_|total}"
