# 4 GPUs: NCCL all-gather as grouped broadcasts vs the forwarding ring; timeline
mkdir -p gpurun_out/r02n4c
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29661 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --transport ${TR:-p2p} > gpurun_out/r02n4c/$name.json 2> gpurun_out/r02n4c/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4c/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'] if d.get('parity') else None)" 2>&1 | tail -1)"; }
TR=nccl B nccl_bcast X=1
TR=nccl B nccl_ring EMESH_LIB=build_var/libagring.so
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29662 tools/nccl_timeline.py 1e9 0 16 nccl > gpurun_out/r02n4c/tl_nccl.txt 2>&1; echo "tl rc=$?"; grep -v "^\*\|OMP" gpurun_out/r02n4c/tl_nccl.txt | grep -E "round|XFER|APPLY ph1 hop-1 w0" | head -40
timeout 600 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 -k "parity or nccl" > gpurun_out/r02n4c/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02n4c/mg_tests.txt | head
