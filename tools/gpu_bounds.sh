cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
# bounds-checked library (device asserts on every shared/global index of the
# c-transform kernels): a trapped assert fails the process
BFM_LIB_OVERRIDE=$PWD/paper_1905_12154_b200/libbfm_b200_debug.so timeout 900 python tools/sanitize_drive.py > gpurun_out/bounds_drive.txt 2>&1
echo "bounds rc=$?"; tail -3 gpurun_out/bounds_drive.txt
