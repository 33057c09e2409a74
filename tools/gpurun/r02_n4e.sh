# 4 GPUs: NCCL transport with registered ncclMemAlloc payload arenas (zero-copy) vs plain cudaMalloc
mkdir -p gpurun_out/r02n4e
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29691 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --transport nccl > gpurun_out/r02n4e/$name.json 2> gpurun_out/r02n4e/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4e/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'] if d.get('parity') else None)" 2>&1 | tail -1)"; }
B base X=1
B reg EMESH_LIB=build_var/libreg.so
B base2 X=2
B reg2 EMESH_LIB=build_var/libreg.so
EMESH_LIB=build_var/libreg.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29692 tools/nccl_timeline.py 1e9 0 16 nccl > gpurun_out/r02n4e/tl_reg.txt 2>&1; grep -E "round|XFER ph0 hop 0|XFER ph1 hop 0" gpurun_out/r02n4e/tl_reg.txt
EMESH_LIB=build_var/libreg.so timeout 900 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 > gpurun_out/r02n4e/mg_tests.txt 2>&1; echo "mg tests (reg) rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02n4e/mg_tests.txt | head
