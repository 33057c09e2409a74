# NCCL transport A/B at 2 GPUs: p2p channel count / chunk size / copy-engine p2p
mkdir -p gpurun_out/r02v
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=${NG:-2} --master-addr 127.0.0.1 --master-port 29621 \
    bench.py --gpus ${NG:-2} --steps 6 --warmup 3 --transport ${T:-nccl} --no-parity --no-e2e --no-cpu-baseline \
    > gpurun_out/r02v/$name.json 2> gpurun_out/r02v/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02v/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
}
T=p2p run p2p_ref EMESH_X=0
run base     EMESH_X=1
run ch16     NCCL_MIN_P2P_NCHANNELS=16
run ch32     NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32
run ch16_c2m NCCL_MIN_P2P_NCHANNELS=16 NCCL_P2P_NVL_CHUNKSIZE=2097152
run cememcpy NCCL_P2P_USE_CUDA_MEMCPY=1
run base2    EMESH_X=2
timeout 900 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 -k "slow_peer" > gpurun_out/r02v/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02v/mg_tests.txt | head
