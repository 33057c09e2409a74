timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tests/nccl_parity_worker.py 2>&1 | grep -v Warning | grep -v "^\s*$" | head -30
