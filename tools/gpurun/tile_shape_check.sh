# Run-time tile shape (2 warp units per tile for batches <= 16M elements): GPU suite, forced-4 parity, smoke, bench, sweep
mkdir -p gpurun_out/ts
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ts/build.log 2>&1 || { tail -20 gpurun_out/ts/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
EMESH_TILE_UNITS=4 timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_codec.py -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ts/n1.json 2> gpurun_out/ts/n1.err
python -c "import json;d=json.loads(open('gpurun_out/ts/n1.json').read().strip().splitlines()[-1]);print('n1', round(d['ms_per_step'],3), d['roofline']['frac'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 tools/sweep_msg.py 268435456 5 > gpurun_out/ts/sweep_n2.jsonl 2> gpurun_out/ts/sweep.err; echo "sweep rc=$?"
python -c "
import json
for l in open('gpurun_out/ts/sweep_n2.jsonl'):
    if l.startswith('{'): r=json.loads(l); print(r['fp32_MB'], round(r['ours_int8_ms'],3), round(r['ours_fp32_ms'],3), round(r['nccl_fp32_ms'],3))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ts/n2.json 2> gpurun_out/ts/n2.err
python -c "import json;d=json.loads(open('gpurun_out/ts/n2.json').read().strip().splitlines()[-1]);print('n2', round(d['ms_per_step'],3), d['value'])"
