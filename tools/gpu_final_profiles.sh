# Round-2 final measurement bundle (run via gpurun): plain bench first, then
# launch lists with DRAM bytes, then full ncu captures of the top kernels.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
mkdir -p gpurun_out/final
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err || exit 1
tail -c 400 gpurun_out/final/bench.json
for c in c1 c2; do timeout 300 python bench.py --config $c --warmup 5 --no-cpu-baseline > gpurun_out/final/bench_$c.json 2>/dev/null; done
for c in c3 c4; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/r02_launches_$c.csv python tools/prof_iter.py $c 8 > gpurun_out/final/r02_launches_$c.log 2>&1
  echo "$c launch list rc=$?"
done
# launch list of the bench command itself (the driver's recipe)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final/ncu_bench.log 2>&1
bash tools/gpu_ncu_kernel.sh c3 2 ct_dy 4 2 ct_dy_c3 > /dev/null
bash tools/gpu_ncu_kernel.sh c4 1 ct_pass 3 3 ct_pass_c4 > /dev/null
bash tools/gpu_ncu_kernel.sh c3 2 os_scatter 4 2 os_scatter_c3 > /dev/null
bash tools/gpu_ncu_kernel.sh c3 2 pois_fft 6 3 pois_c3 > /dev/null
cuobjdump -sass paper_1905_12154_b200/libbfm_b200.so | grep -E "UBLKCP|SYNCS|UTMA" | awk '{print $2}' | sort | uniq -c > gpurun_out/final/sass_tma.txt
cat gpurun_out/final/sass_tma.txt
rm -f gpurun_out/ncu/*.ncu-rep
