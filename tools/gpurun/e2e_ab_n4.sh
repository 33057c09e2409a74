mkdir -p gpurun_out/e2e4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e4/build.log 2>&1 || exit 1
for rep in 1 2; do for v in "A=1" "EMESH_HOST_SERIAL=1"; do
env $v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/e2e4/n4.json 2> gpurun_out/e2e4/n4.err
python -c "import json;d=json.loads(open('gpurun_out/e2e4/n4.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'],d['e2e']['value'])"
done; done
