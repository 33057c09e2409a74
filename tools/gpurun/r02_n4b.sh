# 4 GPUs: multi-GPU tests (final payload always quantizer-pushed, failed owners keep it local),
# P2P bench, NCCL bench under NCCL p2p channel / chunk settings
mkdir -p gpurun_out/r02n4b
timeout 1500 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 > gpurun_out/r02n4b/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02n4b/mg_tests.txt | head
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29651 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --transport ${TR:-p2p} > gpurun_out/r02n4b/$name.json 2> gpurun_out/r02n4b/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4b/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'] if d.get('parity') else None)" 2>&1 | tail -1)"; }
B p2p X=1
TR=nccl B nccl X=1
TR=nccl B nccl_ch16 NCCL_MIN_P2P_NCHANNELS=16
TR=nccl B nccl_ch32 NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32
TR=nccl B nccl_ch16_c1m NCCL_MIN_P2P_NCHANNELS=16 NCCL_P2P_NVL_CHUNKSIZE=1048576
TR=nccl B nccl_ce NCCL_P2P_USE_CUDA_MEMCPY=1
