# 2 GPUs: NCCL-ring timeline + bench (gate fix), P2P final-payload push A/B, slow-peer tests
mkdir -p gpurun_out/r02w
T() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29631 "$@"; }
T tools/nccl_timeline.py 1e9 0 16 nccl > gpurun_out/r02w/tl_nccl.txt 2>&1; echo "tl nccl rc=$?"; head -60 gpurun_out/r02w/tl_nccl.txt | grep -v "^\*\|OMP"
T tools/nccl_timeline.py 1e9 0 16 p2p > gpurun_out/r02w/tl_p2p.txt 2>&1; echo "tl p2p rc=$?"; grep -E "rank|round" gpurun_out/r02w/tl_p2p.txt
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29632 \
    bench.py --gpus 2 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --transport ${TR:-p2p} > gpurun_out/r02w/$name.json 2> gpurun_out/r02w/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02w/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'] if d.get('parity') else None)" 2>&1 | tail -1)"; }
TR=nccl B nccl X=1
B p2p X=1
B p2p_push EMESH_LIB=build_var/libpush.so
B p2p2 X=2
B p2p_push2 EMESH_LIB=build_var/libpush.so
timeout 900 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 > gpurun_out/r02w/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02w/mg_tests.txt | head
