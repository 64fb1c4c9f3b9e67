python -c "import __graft_entry__ as g; g.build()" 
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | head -c 600; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --config c5 2>&1 | tail -1 | head -c 400; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 1 --steps 1 --warmup 0 2>&1 | tail -1 | head -c 400; echo
