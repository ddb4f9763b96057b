mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_eval.py tests/test_model_io.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/t_eval.log 2>&1; echo "rc=$?" >> gpurun_out/t_eval.log
timeout 400 python bench.py --steps 20 --sync-touched --no-cpu-baseline --no-e2e > gpurun_out/bench_touched.log 2>&1
SGNS_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --tokens 200000000 --no-cpu-baseline > gpurun_out/bench_n2_gloo.log 2>&1
SGNS_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 4 --warmup 3 --tokens 200000000 --no-cpu-baseline --sync-touched --no-e2e > gpurun_out/bench_n2_gloo_touched.log 2>&1
