# 4 GPUs: P2P (copy-engine vs quantizer-pushed final payload), NCCL, NCCL timeline, multi-GPU tests
mkdir -p gpurun_out/r02y
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29641 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --transport ${TR:-p2p} > gpurun_out/r02y/$name.json 2> gpurun_out/r02y/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02y/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'] if d.get('parity') else None)" 2>&1 | tail -1)"; }
B p2p X=1
B p2p_push EMESH_LIB=build_var/libpush.so
TR=nccl B nccl X=1
B p2p2 X=2
B p2p_push2 EMESH_LIB=build_var/libpush.so
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29642 tools/nccl_timeline.py 1e9 0 16 nccl > gpurun_out/r02y/tl_nccl.txt 2>&1; echo "tl rc=$?"; grep -v "^\*\|OMP" gpurun_out/r02y/tl_nccl.txt | head -70
timeout 1500 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 > gpurun_out/r02y/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02y/mg_tests.txt | head
