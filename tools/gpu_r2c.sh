cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_edges.py -q -rf > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --fold-devices --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2c_fold2.json 2> gpurun_out/r2c_fold2.err; echo "fold2 rc=$?"
timeout 600 python bench.py --gpus 8 --fold-devices --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2c_fold8.json 2> gpurun_out/r2c_fold8.err; echo "fold8 rc=$?"
tail -5 gpurun_out/r2c_tests.log; tail -c 600 gpurun_out/r2c_fold2.json; tail -c 300 gpurun_out/r2c_fold8.json; tail -5 gpurun_out/r2c_fold2.err
