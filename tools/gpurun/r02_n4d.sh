# 4 GPUs: NCCL reduce-scatter send/recv bandwidth: channels, CTAs left to NCCL
mkdir -p gpurun_out/r02n4d
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29671 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --transport nccl > gpurun_out/r02n4d/$name.json 2> gpurun_out/r02n4d/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4d/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; }
B base X=1
B minch32 NCCL_MIN_NCHANNELS=32 NCCL_MIN_P2P_NCHANNELS=32
B res48 EMESH_LIB=build_var/libres48.so
B res96 EMESH_LIB=build_var/libres96.so
B res96_ch32 EMESH_LIB=build_var/libres96.so NCCL_MIN_NCHANNELS=32 NCCL_MIN_P2P_NCHANNELS=32
B buff16m NCCL_BUFFSIZE=16777216
B base2 X=2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29672 tools/nccl_timeline.py 1e9 0 16 nccl > gpurun_out/r02n4d/tl_nccl.txt 2>&1
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,P2P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29673 tools/nccl_timeline.py 1e8 0 16 nccl > gpurun_out/r02n4d/nccl_debug.txt 2>&1
grep -iE "channel|p2p|nvls|ring" gpurun_out/r02n4d/nccl_debug.txt | head -40
