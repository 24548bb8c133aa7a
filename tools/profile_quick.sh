# Trimmed round-end refresh (run via gpurun): smoke(), bench lines C1-C4 and
# the reference arm, launch lists of C3 (bench command) and C4. The full ncu
# captures and DRAM bytes stay with tools/profile_round.sh.
set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/prof/smoke.log 2>&1 || exit 1
python bench.py > gpurun_out/prof/bench_c3.json 2> gpurun_out/prof/bench_c3.err || exit 1
python bench.py --config c4 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c4.json 2>/dev/null
python bench.py --config c2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c2.json 2>/dev/null
python bench.py --config c1 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_c1.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/prof/bench_ref_c3.json 2>/dev/null
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_bench_c3.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/prof_c3.py c4 2 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c4.csv python tools/prof_c3.py c4 2 > /dev/null 2>&1
ls -la gpurun_out/prof
