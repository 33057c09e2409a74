# 4 GPUs: NCCL transport: CTAs left to NCCL x code runs sent as 32-bit words
mkdir -p gpurun_out/r02n4h
B() { name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29721 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --transport nccl > gpurun_out/r02n4h/$name.json 2> gpurun_out/r02n4h/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4h/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; }
B res148 EMESH_LIB=build_var/libres148.so
B w148 EMESH_LIB=build_var/libw148.so
B res74 EMESH_LIB=build_var/libres74.so
B res148b EMESH_LIB=build_var/libres148.so
B w148b EMESH_LIB=build_var/libw148.so
