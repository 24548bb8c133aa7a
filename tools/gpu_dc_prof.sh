# ct_dc_kernel: stats + ncu of two launches (strided pass 0, contiguous pass 1) in C3 iteration 2
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
mkdir -p gpurun_out/dc
timeout 300 python tools/ct_stats.py c3 2>&1 | tail -6
timeout 200 python tools/prof_c3.py c3 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ct_dc -s 4 -c 2 -o gpurun_out/dc/dc_full python tools/prof_c3.py c3 2 > gpurun_out/dc/ncu.log 2>&1
tail -3 gpurun_out/dc/ncu.log
