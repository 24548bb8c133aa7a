# Round-end measurement bundle (run via gpurun). Plain runs first; every ncu
# capture only after the same command exited 0 without ncu.
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench_c3.json 2> gpurun_out/prof/bench_c3.err || exit 1
python bench.py --config c4 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c4.json 2>/dev/null
python bench.py --config c2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c2.json 2>/dev/null
python bench.py --config c1 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_c1.json 2>/dev/null
python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/prof/bench_c5.json 2> gpurun_out/prof/bench_c5.txt
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/prof/bench_ref_c3.json 2>/dev/null
# launch list of the bench command itself (C3)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_bench_c3.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# c-transform DRAM bytes: the C5 operator, and one call inside the C3 iteration
python tools/ct_op_traffic.py > /dev/null 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ct_ \
      --csv --log-file gpurun_out/prof/ct_op_dram.csv python tools/ct_op_traffic.py > /dev/null 2>&1
python tools/prof_c3.py c3 2 > /dev/null 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ct_ -s 4 -c 2 \
      --csv --log-file gpurun_out/prof/ct_iter_dram.csv python tools/prof_c3.py c3 2 > /dev/null 2>&1
# full captures: the dominant kernel (ct_dy_kernel in the C3 iteration) and the Poisson kernel
python tools/prof_c3.py c3 2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ct_dy -s 6 -c 1 -o gpurun_out/prof/ct_full python tools/prof_c3.py c3 2 > /dev/null 2>&1
python tools/prof_c3.py c3 1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pois_fft -s 3 -c 1 -o gpurun_out/prof/pois_full python tools/prof_c3.py c3 1 > /dev/null 2>&1
# C4 launch list
python tools/prof_c3.py c4 2 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c4.csv python tools/prof_c3.py c4 2 > /dev/null 2>&1
ls -la gpurun_out/prof
