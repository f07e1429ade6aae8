./tools/rot_micro
./tools/tile_micro
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --config C1 --dist-backend gloo --steps 2 --warmup 1 --no-cpu 2>&1 | tail -3
