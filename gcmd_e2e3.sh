mkdir -p gpurun_out/e2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e/build.log 2>&1 || { tail -20 gpurun_out/e2e/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_ring.py -q -x 2>&1 | tail -4
for v in "" "EMESH_HOST_SERIAL=1"; do
env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e/n2.json 2> gpurun_out/e2e/n2.err; echo "n2 [$v] rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/e2e/n2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['e2e']['value'])"
done
