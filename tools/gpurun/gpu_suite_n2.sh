mkdir -p gpurun_out/full
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/full/build.log 2>&1 || { tail -20 gpurun_out/full/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --steps 10 --warmup 3 --transport nccl --no-cpu-baseline > gpurun_out/full/n2_nccl.json 2> gpurun_out/full/n2_nccl.err; echo "n2 nccl rc=$?"
tail -c 400 gpurun_out/full/n2_nccl.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/full/n2.json 2> gpurun_out/full/n2.err; echo "n2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/full/n2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d.get('config'))"
python -c "import json;d=json.loads(open('gpurun_out/full/n2_nccl.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d.get('config'))"
