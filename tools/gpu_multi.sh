# multi-rank bench path on one GPU (gloo rendezvous, ranks share cuda:0): functional check only
export SPD_BENCH_BACKEND=gloo
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --config W 2>&1 | tail -2 | cut -c1-300
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --config B27 2>&1 | tail -1 | cut -c1-200
unset SPD_BENCH_BACKEND
timeout 300 python bench.py --config W --force-slab --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
timeout 300 python bench.py --config B9 --force-slab --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
