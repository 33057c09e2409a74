# 2 GPUs: config-4 sweep (peer transport, S=4) + where a small round's time goes
mkdir -p gpurun_out/r02s2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29681 tools/sweep_msg.py 268435456 10 > gpurun_out/r02s2/sweep_n2.jsonl 2> gpurun_out/r02s2/sweep_n2.err; echo "sweep rc=$?"
python -c "
import json
for l in open('gpurun_out/r02s2/sweep_n2.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['fp32_MB'], round(d['ours_int8_ms'],4), round(d['ours_fp32_ms'],4), round(d['nccl_fp32_ms'],4))"
for n in 262144 4194304 16777216; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 tools/nccl_timeline.py $n 0 4 p2p 2>&1 | grep -vE "^W|warn|^\*|OMP" | head -20
done
