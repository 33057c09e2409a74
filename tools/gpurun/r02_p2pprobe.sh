timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29801 tools/nccl_p2p_probe.py 2>&1 | grep -v "^W\|OMP\|^\*"
