mkdir -p gpurun_out/r01b
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 tools/sweep_msg.py 1073741824 5 > gpurun_out/r01b/sweep_n2.jsonl 2> gpurun_out/r01b/sweep_n2.err; echo sweep rc=$?; cat gpurun_out/r01b/sweep_n2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['fp32_MB']:8.0f} MB  int8 {d['ours_int8_ms']:8.3f} ms  fp32 {d['ours_fp32_ms']:8.3f} ms  nccl {d['nccl_fp32_ms']:8.3f} ms   busbw int8 {d['ours_int8_busbw_GBs']:7.1f} nccl {d['nccl_fp32_busbw_GBs']:7.1f}\")"
