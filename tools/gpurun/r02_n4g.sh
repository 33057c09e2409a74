# 4 GPUs: NCCL transport with the quantizer grid leaving room for NCCL's send/recv CTAs
mkdir -p gpurun_out/r02n4g
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29711 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --transport nccl > gpurun_out/r02n4g/$name.json 2> gpurun_out/r02n4g/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4g/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; }
B base X=1
B res148 EMESH_LIB=build_var/libres148.so
B res222 EMESH_LIB=build_var/libres222.so
for v in res148 res222; do EMESH_LIB=build_var/lib$v.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29712 tools/nccl_timeline.py 1e9 0 16 nccl > gpurun_out/r02n4g/tl_$v.txt 2>&1; grep -E "round|XFER ph0 hop 1" gpurun_out/r02n4g/tl_$v.txt; done
