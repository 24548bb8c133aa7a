cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solver_ctl.py tests/test_gpu_fullrun.py -x -q > gpurun_out/t1.log 2>&1; tail -15 gpurun_out/t1.log
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullrun.py > gpurun_out/t2.log 2>&1; tail -5 gpurun_out/t2.log
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/b_c1.log 2>&1; tail -1 gpurun_out/b_c1.log | cut -c1-400
timeout 300 python bench.py --config c3 --steps 20 --no-cpu-baseline > gpurun_out/b_c3.log 2>&1; tail -1 gpurun_out/b_c3.log | cut -c1-400
