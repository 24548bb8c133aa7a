timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ctransform or solver" 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ct_pass --csv --log-file gpurun_out/c3new.csv python tests/prof_c3.py c3 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ct_pass --csv --log-file gpurun_out/c4new.csv python tests/prof_c3.py c4 2 > /dev/null 2>&1
