timeout 600 python -m pytest tests -m gpu -q -x --timeout=200 2>&1 | tail -3
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tests/nccl_parity_worker.py 2>&1 | grep -E "MISMATCH|asked|parity|Error" | head -20
