# 4 GPUs: NCCL send/recv read mode A/B
mkdir -p gpurun_out/r02n4l
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --transport nccl > gpurun_out/r02n4l/$name.json 2> gpurun_out/r02n4l/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4l/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3))" 2>&1 | tail -1)"; }
B base X=1
B read1 NCCL_P2P_READ_ENABLE=1
B read0 NCCL_P2P_READ_ENABLE=0
B llthr NCCL_P2P_LL_THRESHOLD=0
B base2 X=2
B read1b NCCL_P2P_READ_ENABLE=1
NCCL_P2P_READ_ENABLE=1 NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,P2P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29782 tools/nccl_timeline.py 1e8 0 16 nccl 2>&1 | grep -E "via P2P" | head -4
