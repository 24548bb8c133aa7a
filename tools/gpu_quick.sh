timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 200 python bench.py --steps 20 --warmup 3 > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | cut -c1-300
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_c3.py c3 2 > gpurun_out/ncu.log 2>&1
