# full ncu capture of one kernel inside a few C3/C4 iterations, summarised:
# gpu_ncu_kernel.sh CONFIG ITERS KERNEL_REGEX SKIP COUNT OUTNAME [ENV=VAL ...]
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
cfg=$1; it=$2; kre=$3; skip=$4; cnt=$5; out=$6; shift 6
mkdir -p gpurun_out/ncu
env "$@" timeout 300 python tools/prof_c3.py $cfg $it > /dev/null 2>&1 || exit 1
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c $cnt -f -o gpurun_out/ncu/$out python tools/prof_c3.py $cfg $it > gpurun_out/ncu/$out.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu/$out.ncu-rep > gpurun_out/ncu/$out.txt 2>&1
python tools/ncu_lines.py gpurun_out/ncu/$out.ncu-rep 45 >> gpurun_out/ncu/$out.txt 2>&1
tail -75 gpurun_out/ncu/$out.txt
