cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/full_tests.log 2>&1; tail -3 gpurun_out/full_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 300 gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --slabs --steps 10 --warmup 2 --no-cpu-baseline > gpurun_out/bench_slabs.json 2> gpurun_out/bench_slabs.err; tail -c 600 gpurun_out/bench_slabs.json
