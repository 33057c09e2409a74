timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 tests/retry_worker.py > gpurun_out/retry.log 2>&1
echo rc=$?
grep -v Warning gpurun_out/retry.log | grep -E "r0|r1|File|Thread|Error" | head -30
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tests/nccl_parity_worker.py 2>&1 | grep -E "MISMATCH|asked|parity|Error" | head -20
