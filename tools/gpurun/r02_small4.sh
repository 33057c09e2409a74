# 4 GPUs: where a small peer-transport round's time goes (op timeline at 1 MB / 16 MB / 64 MB fp32 payloads)
mkdir -p gpurun_out/r02sm4
for n in 262144 4194304 16777216; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29731 tools/nccl_timeline.py $n 0 4 p2p 2>&1 | grep -vE "^W|warn|^\*|OMP" | head -24
done
