set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "sharded" > gpurun_out/t_shard.log 2>&1; tail -2 gpurun_out/t_shard.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; tail -c 3000 gpurun_out/bench_c3.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -c 1500 gpurun_out/bench_ref.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; tail -c 2500 gpurun_out/bench_c4.log
FFCA_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-other > gpurun_out/bench_n2.log 2>&1; tail -c 3000 gpurun_out/bench_n2.log
