timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tests/nccl_parity_worker.py 2>&1 | grep -E "MISMATCH|asked|parity|Error" | head -10
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 tools/sweep_msg.py 1073741824 5 2>/dev/null | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['fp32_MB']:7.0f} MB  int8 {d['ours_int8_ms']:7.3f}  fp32 {d['ours_fp32_ms']:7.3f}  nccl {d['nccl_fp32_ms']:7.3f}\")"
