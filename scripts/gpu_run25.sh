timeout 600 python -m pytest tests/test_gpu_dist.py -q -m gpu -x 2>&1 | tail -15
PB_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e 2>&1 | tail -3 | cut -c1-600
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-400
